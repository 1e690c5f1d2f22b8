cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/sweep.sh "FFG_SIDE_PRIO=0" "FFG_SIDE_PRIO=2" "FFG_SIDE_PRIO=1" "FFG_SIDE_PRIO=0" "FFG_SIDE_PRIO=2"
ARGS="--p 251 --n 32768 --steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof" bash scripts/sweep.sh "FFG_SIDE_PRIO=0" "FFG_SIDE_PRIO=2" "FFG_SIDE_PRIO=1" "FFG_SIDE_PRIO=0" "FFG_SIDE_PRIO=2"
