cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/trace_window.py --lru --n 16384 --t0 20 --t1 20.7 2>&1 | grep -v Warn | tail -60
