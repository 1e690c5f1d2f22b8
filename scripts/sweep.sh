#!/bin/bash
# env-knob sweep of the bench step time (device entry), one line per setting
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
ARGS=${ARGS:-"--steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof"}
run() {
  local tag="$1"; shift
  local out
  out=$(env "$@" timeout 300 python bench.py $ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))" 2>/dev/null)
  echo "$tag $out"
}
run base X=1
run panel_direct FFG_PANEL_DIRECT=1
run corner2048 FFG_CORNER_MAX=2048
run corner8192 FFG_CORNER_MAX=8192
run defer136 FFG_DEFER_SMS=136 FFG_SIDE_SMS=136
run defer146 FFG_DEFER_SMS=146 FFG_SIDE_SMS=146
run apply64 FFG_APPLY_CTAS=64
