cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
bash scripts/sweep.sh "FFG_STRIP_A1=1" "FFG_STRIP_A1=0" "FFG_STRIP_A1=1" "FFG_STRIP_A1=0"
ARGS="--p 251 --n 32768 --steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof --no-clocks" bash scripts/sweep.sh "FFG_STRIP_A1=1" "FFG_STRIP_A1=0" "FFG_STRIP_A1=1" "FFG_STRIP_A1=0"
