cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
echo "== direct sweep (config 3)"
bash scripts/sweep.sh "FFG_X=0" "FFG_DEFER_DIRECT=1" "FFG_SIDE_DIRECT=1" "FFG_DEFER_DIRECT=1 FFG_SIDE_DIRECT=1" "FFG_DEFER_DIRECT=1 FFG_DEFER_SMS=0" "FFG_CORNER_MAX=256" "FFG_CORNER_MAX=512" "FFG_CORNER_MAX=1024"
echo "== config 5"
ARGS="--p 251 --n 32768 --steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof" bash scripts/sweep.sh "FFG_X=0" "FFG_DEFER_DIRECT=1" "FFG_SIDE_DIRECT=1" "FFG_DEFER_DIRECT=1 FFG_SIDE_DIRECT=1"
