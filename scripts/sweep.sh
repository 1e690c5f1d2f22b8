#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
ARGS=${ARGS:-"--steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof"}
run() {
  local tag="$1"; shift
  local out
  out=$(env "$@" timeout 300 python bench.py $ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))" 2>/dev/null)
  echo "$tag $out"
}
for cfg in "${@}"; do
  run "$cfg" $cfg
done
