cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x -k "gemm or fgemm or trsm" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
P=251 BIG=32768 SHAPES="256,16000,256;512,16000,512;16000,512,512;4096,4096,4096;16384,16384,16384" python scripts/gemm_small.py 2>&1 | grep -v Warn
ARGS="--p 251 --n 32768 --steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof" bash scripts/sweep.sh "FFG_X=0"
