mkdir -p gpurun_out
CFGS="3" bash scripts/gpu_ab_env.sh "VG_X=0" "VG_TASK_KB=256" "VG_TASK_KB=64" "VG_ORDER=1"
CFGS="4" bash scripts/gpu_ab_env.sh "VG_PLAN_Q=1" "VG_CAP_MAX=64"
bash scripts/gpu_prof_cfg.sh 3 32 cfg3yp vg_slab 2 1
bash scripts/gpu_prof_cfg.sh 4 4096 cfg4yp vg_slab 2 1
