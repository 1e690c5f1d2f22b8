cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --workload lru --steps 2 --warmup 3 --no-cpu --no-fgemm > gpurun_out/bench_config4.json 2> gpurun_out/bench_config4.err; echo "c4 rc=$?"
timeout 300 python bench.py --p 251 --n 32768 --steps 5 --warmup 3 --no-cpu --no-fgemm > gpurun_out/bench_config5.json 2> gpurun_out/bench_config5.err; echo "c5 rc=$?"
