cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'], (d.get('cpu_baseline') or {}).get('value'), d['clocks'])"
