"""Side-by-side table of the reference's bench protocol (voxgrid.cli bench)
run on the CPU and the same protocol on the GPU (python -m
paper_2211_08506_b200 bench): python scripts/protocol_compare.py gpu.json ref.json"""
import json
import sys

g = json.load(open(sys.argv[1]))
r = json.load(open(sys.argv[2]))
ref = {(c["size"], c["variance"], c["mode"]): c for c in r["cells"]}
print(f"{'size':>5} {'sigma':>6} {'mode':>7} {'ref mol/s':>11} {'gpu mol/s':>12} {'ratio':>9} "
      f"{'nonzero frac (ref / gpu)':>26}")
for c in g["cells"]:
    k = (c["size"], c["variance"], c["mode"])
    if k not in ref:
        continue
    rc = ref[k]
    print(f"{c['size']:5d} {c['variance']:6.2f} {c['mode']:>7} {rc['throughput_mol_per_s']:11.1f} "
          f"{c['throughput_mol_per_s']:12.0f} {c['throughput_mol_per_s'] / rc['throughput_mol_per_s']:9.0f} "
          f"{rc['nonzero_fraction']:12.6f} / {c['nonzero_fraction']:.6f}")
