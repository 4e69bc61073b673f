# exploration: env A/Bs on cfg3/cfg4, then ncu --set full of K3 on cfg3 and cfg4
mkdir -p gpurun_out
CFGS="3" bash scripts/gpu_ab_env.sh "VG_ORDER=0" "VG_ORDER=1"
CFGS="4" bash scripts/gpu_ab_env.sh "VG_X=0" "VG_PLAN_Q=1" "VG_FUSE=0" "VG_TASK_KB=512" "VG_TASK_KB=2048" "VG_CAP_MAX=64"
bash scripts/gpu_prof_cfg.sh 3 32 cfg3 vg_slab 2 1
bash scripts/gpu_prof_cfg.sh 4 4096 cfg4 vg_slab 2 1
