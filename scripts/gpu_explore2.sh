mkdir -p gpurun_out
CFGS="3" bash scripts/gpu_ab_env.sh "VG_X=0" "VG_SW=4" "VG_TASK_KB=64" "VG_TASK_KB=256" "VG_CAP_MAX=96" "VG_ZW=2" "VG_ZW=8" "VG_ORDER=1 VG_TASK_KB=64"
CFGS="4" bash scripts/gpu_ab_env.sh "VG_SW=4" "VG_ZW=3" "VG_ZW=2"
