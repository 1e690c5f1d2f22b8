#!/bin/bash
# Round-end style evidence run on one B200 (writes gpurun_out/*); every ncu pass runs only
# after the same command exited 0 without ncu.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --workload lru --steps 2 --warmup 3 --no-cpu --no-fgemm > gpurun_out/bench_config4.json 2> gpurun_out/bench_config4.err
python bench.py --p 251 --n 32768 --steps 5 --warmup 3 --no-cpu --no-fgemm > gpurun_out/bench_config5.json 2> gpurun_out/bench_config5.err
# config 5 again, three consecutive runs (each line carries the guesses tried / failed in its timed region)
for i in 1 2 3; do
  python bench.py --p 251 --n 32768 --steps 5 --warmup 3 --no-cpu --no-e2e --no-fgemm --no-prof >> gpurun_out/bench_config5_x3.json 2>/dev/null
done
python scripts/trace_pluq.py --n 32768 --p 251 > gpurun_out/trace_c5.txt 2>&1
python scripts/trace_pluq.py --lru --n 16384 > gpurun_out/trace_c4.txt 2>&1
python scripts/trace_e2e.py > gpurun_out/trace_e2e.txt 2>&1
python scripts/trace_pluq.py --n 16384 --json gpurun_out/trace_n16384.json > gpurun_out/trace_n16384.txt 2>&1
# launch list of one bench step (durations only)
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-fgemm --no-prof > gpurun_out/bench_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-fgemm --no-prof --no-clocks > gpurun_out/ncu_bench.log 2>&1
# the fused base case + inverses inside an n = 16384 PLUQ (full set, with source)
python scripts/prof_pluq.py --n 16384 > gpurun_out/prof_pluq_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"rr_base_inv|leaf_apply|panel_update|panel_mini" \
    -s 200 -c 8 -o gpurun_out/panel_full python scripts/prof_pluq.py --n 16384 > gpurun_out/ncu_panel.log 2>&1
python scripts/ncu_summary.py gpurun_out/panel_full.ncu-rep --label "panel-chain kernels inside an n = 16384 PLUQ (config 3)" \
  > gpurun_out/ncu_panel_summary.json 2>/dev/null
# fgemm 8192^3: one full ncu capture of the tcgen05 kernel
python scripts/prof_gemm.py > gpurun_out/prof_gemm_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:modgemm -s 1 -c 1 -o gpurun_out/gemm_full python scripts/prof_gemm.py > gpurun_out/ncu_gemm.log 2>&1
python scripts/ncu_summary.py gpurun_out/gemm_full.ncu-rep --label "fgemm 8192^3 C <- C - A*B mod 131071 (config 2)" \
  > gpurun_out/ncu_gemm_summary.json 2>/dev/null
# DRAM traffic of every tensor-core GEMM launch inside one n = 16384 PLUQ
FFG_GEMM_LOG=1 python scripts/gemm_shapes.py --run --n 16384 2> gpurun_out/shapes.log && \
  FFG_GEMM_LOG=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:modgemm --csv --log-file gpurun_out/gemm_dram.csv python scripts/gemm_shapes.py --run --n 16384 \
    2> gpurun_out/shapes_ncu.log > gpurun_out/ncu_dram.log
python scripts/pluq_traffic.py gpurun_out/gemm_dram.csv gpurun_out/shapes.log --n 16384 --p 131071 --thr 64 \
  > gpurun_out/pluq_gemm_traffic.json 2> gpurun_out/pluq_traffic.err
echo done
# fgemm DRAM traffic per launch (bench.py reads profiles/gemm_traffic.json)
python - <<'PY' > gpurun_out/gemm_traffic.json
import json
d = json.load(open("gpurun_out/ncu_gemm_summary.json"))["launches"][0]
print(json.dumps({"dram_bytes_per_launch": d["dram_bytes"], "algorithmic_bytes_per_launch": 939524096,
                  "algorithmic_note": "L=3 limb planes of A and B (2*3*8192^2) + C read and written (2*4*8192^2)",
                  "source": "profiles/r02_ncu_gemm_8192_summary.json", "shape": "8192^3 L=3"}, indent=1))
PY
echo collected
