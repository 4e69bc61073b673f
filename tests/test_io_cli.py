"""File formats and CLI against the reference.

CPU tests: parsers, NPY contract and argument handling, compared with
fixtures the real reference produced (tests/golden/io.json). The GPU test
runs the ``grid`` subcommand and matches the reference CLI's output bits.
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2211_08506_b200 as vg
from _golden import GOLDEN, sha
from paper_2211_08506_b200 import benchproto, cli
from paper_2211_08506_b200.io import ParseError

IO = json.loads((GOLDEN / "io.json").read_text())


def test_element_table():
    assert len(vg.ELEMENT_SYMBOLS) == 118
    assert vg.ELEMENT_SYMBOLS[0] == "H" and vg.ELEMENT_SYMBOLS[5] == "C"
    assert vg.ELEMENT_SYMBOLS[-1] == "Og"


@pytest.mark.parametrize("i", range(len(IO["xyz"])))
def test_parse_xyz_matches_reference(i):
    rec = IO["xyz"][i]
    if "error" in rec:
        with pytest.raises(ParseError) as err:
            vg.parse_xyz(rec["text"])
        assert str(err.value) == rec["error"] and err.value.line == rec["line"]
        return
    m = vg.parse_xyz(rec["text"])
    assert list(m.symbols) == rec["symbols"]
    assert np.array_equal(m.positions, np.array(rec["positions"]).reshape(-1, 3))
    assert m.channel_map("auto") == rec["auto"] and m.n_channels("auto") == rec["n_auto"]


@pytest.mark.parametrize("i", range(len(IO["csv"])))
def test_parse_csv_matches_reference(i):
    rec = IO["csv"][i]
    if "error" in rec:
        with pytest.raises(ParseError) as err:
            vg.parse_points_csv(rec["text"])
        assert str(err.value) == rec["error"] and err.value.line == rec["line"]
        return
    ps = vg.parse_points_csv(rec["text"])
    assert np.array_equal(ps.to_rows(), np.array(rec["rows"]).reshape(-1, 4))


def test_channel_policies():
    water = vg.parse_xyz(IO["xyz"][1]["text"])
    assert list(water.to_particle_set("auto").channels) == [1, 0, 0]
    assert set(water.to_particle_set("single").channels) == {0}
    with pytest.raises(ValueError):
        water.channel_map(1)
    offsets, ch, xyz = vg.pack_molecules([water, water], ("H", "C", "N", "O", "F"))
    assert offsets.tolist() == [0, 3, 6] and ch.tolist() == [3, 0, 0, 3, 0, 0]
    with pytest.raises(ValueError, match="element 'O'"):
        vg.pack_molecules([water], ("H", "C"))


def test_npy_contract(tmp_path):
    arr = np.random.default_rng(0).random((2, 3, 4, 5)).astype(np.float32)
    p = tmp_path / "g.npy"
    vg.write_npy(arr, p)
    assert np.array_equal(vg.read_npy(p), arr)
    raw = p.read_bytes()
    assert raw[:6] == b"\x93NUMPY" and raw[6:8] == b"\x01\x00"
    np.save(tmp_path / "f.npy", np.asfortranarray(arr))
    with pytest.raises(ValueError, match="Fortran"):
        vg.read_npy(tmp_path / "f.npy")
    np.save(tmp_path / "d.npy", arr.astype(np.float64))
    with pytest.raises(ValueError, match="dtype"):
        vg.read_npy(tmp_path / "d.npy")
    (tmp_path / "x.npy").write_bytes(b"not numpy at all")
    with pytest.raises(ValueError, match="not an NPY"):
        vg.read_npy(tmp_path / "x.npy")
    (tmp_path / "t.npy").write_bytes(raw[:-7])
    with pytest.raises(ValueError, match="truncated"):
        vg.read_npy(tmp_path / "t.npy")
    with pytest.raises(ValueError):
        vg.grid_from_array(np.zeros((2, 3)), vg.BoundingBox((0, 0, 0), (1, 1, 1)), 0.5)
    g = vg.grid_from_array(arr, vg.BoundingBox((0, 0, 0), (1, 1, 1)), 0.5)
    assert g.spec.shape == (3, 4, 5) and g.spec.channels == 2


def test_bench_corpus_matches_reference():
    rec = IO["corpus"]
    corpus = benchproto.synth_corpus(rec["n"], (8, 40), 48.0, seed=rec["seed"])
    h = hashlib.sha256()
    for ps in corpus:
        h.update(ps.channels.astype(np.int64).tobytes())
        h.update(ps.positions.astype(np.float64).tobytes())
    assert h.hexdigest() == rec["sha"]
    with pytest.raises(ValueError):
        benchproto.BenchConfig(sizes=(4,))


def test_cli_argument_errors(tmp_path, capsys):
    assert cli.cli_main(["grid", "--nope"]) == 2
    assert cli.cli_main(["grid", "--input", "x.xyz", "--variance", "0.5"]) == 2  # no --output
    code = cli.cli_main(["grid", "--input", str(tmp_path / "missing.xyz"), "--variance", "0.5",
                         "--output", str(tmp_path / "o.npy")])
    assert code == 1 and "voxgrid:" in capsys.readouterr().err
    (tmp_path / "a.txt").write_text("1\n\nC 0 0 0\n")
    assert cli.cli_main(["grid", "--input", str(tmp_path / "a.txt"), "--variance", "0.5",
                         "--output", str(tmp_path / "o.npy")]) == 1
    (tmp_path / "m.xyz").write_text("1\n\nC 0 0 0\n")
    assert cli.cli_main(["grid", "--input", str(tmp_path / "m.xyz"), "--variance", "0.5",
                         "--periodic", "1,1,1", "--box", "0,0,0,1,1,1",
                         "--output", str(tmp_path / "o.npy")]) == 1
    assert cli.cli_main(["reverse", "--input", str(tmp_path / "none.npy"), "--variance", "0.5",
                         "--output", "o.csv"]) == 1  # missing file -> OSError -> 1
    assert cli.cli_main(["grid", "--grid-size", "1,2", "--input", "a", "--variance", "1",
                         "--output", "o"]) == 2


def _write_inputs(tmp):
    (tmp / "water.xyz").write_text(IO["xyz"][1]["text"])
    (tmp / "mixed.xyz").write_text(IO["xyz"][3]["text"])
    (tmp / "pts.csv").write_text(IO["csv"][0]["text"])


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(IO["cli"])))
def test_cli_grid_matches_reference_cli(tmp_path, i):
    rec = IO["cli"][i]
    _write_inputs(tmp_path)
    args = ["grid"] + [str(tmp_path / a) if a.endswith((".xyz", ".csv")) else a
                       for a in rec["args"]]
    args += ["--output", str(tmp_path / "o.npy"), "--stats", str(tmp_path / "s.json")]
    assert cli.cli_main(args) == rec["code"] == 0
    arr = vg.read_npy(tmp_path / "o.npy")
    assert list(arr.shape) == rec["shape"]
    assert sha(arr) == rec["sha"]
    st = json.loads((tmp_path / "s.json").read_text())
    st.pop("elapsed_ms")
    ref = rec["stats"]
    for key in ("nonzero_voxels", "erf_evals", "voxel_writes", "shape", "sigma", "box"):
        assert st[key] == ref[key], key
    assert st["sum"] == pytest.approx(ref["sum"], rel=1e-12, abs=1e-12)
    assert st["per_channel_sums"] == pytest.approx(ref["per_channel_sums"], rel=1e-12, abs=1e-12)


@pytest.mark.gpu
def test_cli_bench_micro_run(tmp_path, capsys):
    out = tmp_path / "r.json"
    assert cli.cli_main(["bench", "--sizes", "16,32", "--variances", "0.25,0.5", "--repeats",
                         "2", "--molecules", "6", "--output", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert len(rep["cells"]) == 2 * 2 * 2
    assert all(c["throughput_mol_per_s"] > 0 for c in rep["cells"])
    assert "ms/mol" in capsys.readouterr().out
