# K3W variant sweep on one config: bash scripts/ws_sweep.sh CONFIG
C=${1:-3}
L=$PWD/paper_2211_08506_b200
for m in 2 3; do
  VG_LIB=$L/libvg_ws$m.so timeout 300 python scripts/k3_ab.py $C 4 "old:VG_WS=0" \
    "m${m}np1s3:VG_WS=1,VG_WS_CTAS=$m,VG_WS_NP=1,VG_WS_STAGES=3" \
    "m${m}np1s3M2:VG_WS=1,VG_WS_CTAS=$m,VG_WS_NP=1,VG_WS_STAGES=3,VG_WS_M=2" \
    "m${m}np2s3M2:VG_WS=1,VG_WS_CTAS=$m,VG_WS_NP=2,VG_WS_STAGES=3,VG_WS_M=2" \
    "m${m}np1s2M2:VG_WS=1,VG_WS_CTAS=$m,VG_WS_NP=1,VG_WS_STAGES=2,VG_WS_M=2" \
    "m${m}np2s4M2:VG_WS=1,VG_WS_CTAS=$m,VG_WS_NP=2,VG_WS_STAGES=4,VG_WS_M=2"
done
