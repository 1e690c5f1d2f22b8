cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m "gpu and not slow" -x -k "panel or base" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
bash scripts/sweep.sh "FFG_X=0" "FFG_X=1" "FFG_X=2"
