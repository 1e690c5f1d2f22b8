# usage: bash /tmp/c3.sh "ENV=..." ...   (runs c3 bench lines per env setting)
for e in "$@"; do env $e python bench.py --steps 5 --no-e2e --no-cpu --no-fgemm --no-prof 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"c3 $e\", round(d[\"ms_per_step\"],2), round(d[\"value\"]))"; done
