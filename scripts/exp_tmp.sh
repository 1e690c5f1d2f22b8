cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { env "$@" python bench.py --steps 5 --warmup 3 --no-cpu --no-fgemm --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*: e2e', round(d['e2e']['ms_per_step'],2), d['e2e']['ms_steps'])"; }
run FFG_DOWN_START=0
run FFG_DOWN_START=0.15
run FFG_DOWN_START=0.25
run FFG_DOWN_START=0.35
run FFG_DOWN_START=0.5
run FFG_DOWN_START=0.7
run FFG_DOWN_START=0
