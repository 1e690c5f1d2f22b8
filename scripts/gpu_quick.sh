#!/bin/bash
# Quick GPU iteration: parity suite without the full-size cases, then a short bench (no CPU leg).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_quick.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_quick.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
echo "bench rc=$?"
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    print("ms_per_step", round(d["ms_per_step"], 3), "value", round(d["value"]), "frac", r.get("frac"))
    print("kernels_ms", r.get("kernels_ms"))
except Exception as e:
    print("no bench line", e)
PY
tail -3 gpurun_out/bench_quick.err
