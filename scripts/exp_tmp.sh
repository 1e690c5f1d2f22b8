cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m "gpu and not slow" -x -k "spec_stats or panel or resume" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
bash scripts/sweep.sh "FFG_EARLY_APPLY=1" "FFG_EARLY_APPLY=0" "FFG_EARLY_APPLY=1" "FFG_EARLY_APPLY=0"
ARGS="--p 251 --n 32768 --steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof" bash scripts/sweep.sh "FFG_EARLY_APPLY=1" "FFG_EARLY_APPLY=0" "FFG_EARLY_APPLY=1" "FFG_EARLY_APPLY=0"
