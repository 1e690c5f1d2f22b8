cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu" -x -k "host" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
FFG_HOST_PROG=1 timeout 900 python -m pytest tests -q -m "gpu" -x -k "host or fullsize" > gpurun_out/pytest_quick2.log 2>&1; echo "pytest(prog) rc=$?"; tail -2 gpurun_out/pytest_quick2.log
run() { env "$@" python bench.py --steps 3 --warmup 3 --no-cpu --no-fgemm --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*: dev', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2))"; }
run FFG_X=0
run FFG_HOST_PROG=1
run FFG_HOST_PROG=1 FFG_PROG_CHUNKS=8
run FFG_HOST_PROG=1 FFG_PROG_CHUNKS=2
run FFG_HOST_PROG=1 FFG_PROG_SMS=148
run FFG_HOST_PROG=1 FFG_PROG_SMS=64
run FFG_X=0
run FFG_HOST_PROG=1
