cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc; uptime
python bench.py --no-cpu > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo "bench rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
uptime
python -c "
import json
for f in ['gpurun_out/bench_a.json','gpurun_out/bench.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['e2e']['ms_per_step'], (d.get('cpu_baseline') or {}).get('value'), d['clocks'])"
