cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
bash scripts/sweep.sh "FFG_X=0" "FFG_CORNER_MAX=1024"
