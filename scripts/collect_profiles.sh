#!/bin/bash
# Copy the round-end evidence of gpurun_out/ (scratch) into profiles/ (tracked), named per round.
cd "$(dirname "$0")/.."
R=${1:-r02}
G=gpurun_out
cp $G/bench.json profiles/${R}_bench.json
cp $G/bench_config4.json profiles/${R}_bench_config4.json
cp $G/bench_config5.json profiles/${R}_bench_config5.json
cp $G/bench_config5_x3.json profiles/${R}_bench_config5_x3.json
cp $G/launches_bench.csv profiles/${R}_ncu_launches_bench.csv
python scripts/launches.py $G/launches_bench.csv 0.25 > profiles/${R}_ncu_launches_bench_summary.txt
cp $G/ncu_gemm_summary.json profiles/${R}_ncu_gemm_8192_summary.json
cp $G/ncu_panel_summary.json profiles/${R}_ncu_panel_kernels_summary.json
grep -v Warn $G/trace_n16384.txt > profiles/${R}_trace_pluq_n16384_cupti.txt
grep -v Warn $G/trace_c5.txt > profiles/${R}_trace_pluq_config5_cupti.txt
grep -v Warn $G/trace_c4.txt > profiles/${R}_trace_pluq_config4_cupti.txt
grep -v Warn $G/trace_e2e.txt > profiles/${R}_trace_e2e_n16384.txt
cp $G/pluq_gemm_traffic.json profiles/pluq_gemm_traffic.json
cp $G/gemm_traffic.json profiles/gemm_traffic.json
ls -la profiles | tail -30
