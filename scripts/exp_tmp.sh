cd $GRAFT_REPO_ROOT
ncu --set full --import-source on -k regex:rr_base_inv -s 5 -c 1 -o gpurun_out/bi_src python scripts/base_micro.py --reps 3 > gpurun_out/ncu_bi.log 2>&1
ncu -i gpurun_out/bi_src.ncu-rep --page source --csv --print-source sass > gpurun_out/bi_sass.csv 2>&1
ncu -i gpurun_out/bi_src.ncu-rep --page raw --csv > gpurun_out/bi_raw.csv 2>&1
ls -la gpurun_out/bi_*
