cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2 3 4; do
python bench.py --p 251 --n 32768 --steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5', round(d['ms_per_step'],2), d['clocks'])"
done
for i in 1 2; do
python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3', round(d['ms_per_step'],2), d['clocks'])"
done
python bench.py --workload lru --steps 2 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', round(d['ms_per_step'],2), d['clocks'])"
python bench.py --workload fgemm --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fgemm', round(d['ms_per_step'],2), d['clocks'])"
