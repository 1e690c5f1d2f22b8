cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m "gpu" -x -k "host or fullsize or resume or public" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
for v in 1 0 1 0; do
FFG_DOWN_ROWS=$v python bench.py --steps 3 --warmup 3 --no-cpu --no-fgemm --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('down_rows $v: dev', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2))"
done
for v in 1 0; do
FFG_DOWN_ROWS=$v python bench.py --p 251 --n 32768 --steps 3 --warmup 3 --no-cpu --no-fgemm --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 down_rows $v: dev', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2))"
done
FFG_DOWN_ROWS=1 python scripts/trace_e2e.py 2>&1 | grep -v Warn | grep "call\|base cases\|\[ "
