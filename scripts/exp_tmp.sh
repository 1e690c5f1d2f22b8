cd $GRAFT_REPO_ROOT
rm -f paper_1402_3501_b200/build/baseinv.o
FFG_NVCC_EXTRA="-DBI_DBG" python -m paper_1402_3501_b200.build > /dev/null 2>&1
FFG_BI_DBG=1 python scripts/base_micro.py --reps 3 2>&1 | grep BI_DBG | tail -2
