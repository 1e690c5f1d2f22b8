cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
FFG_SPEC_LOG=1 python scripts/pluq_seeds.py --n 16384 --p 131071 --seeds 1,2,3 2>&1 | grep -v Warn | tail -9
FFG_SPEC_LOG=1 python scripts/pluq_seeds.py --seeds 1,2 2>&1 | grep -v Warn | tail -8
