cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_profile.py -x -q > gpurun_out/pytest_profile.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_profile.log
