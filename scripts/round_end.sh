#!/bin/bash
# Round-end style evidence run on one B200 (writes gpurun_out/*)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
python scripts/trace_pluq.py --n 16384 --json gpurun_out/trace_n16384.json > gpurun_out/trace_n16384.txt 2>&1
python scripts/prof_gemm.py > gpurun_out/prof_gemm_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:modgemm -s 1 -c 1 -o gpurun_out/gemm_full python scripts/prof_gemm.py > gpurun_out/ncu_gemm.log 2>&1
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-fgemm --no-prof > gpurun_out/bench_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 13344 -c 5000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-fgemm --no-prof > gpurun_out/ncu_bench.log 2>&1
echo done
