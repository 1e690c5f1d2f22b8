cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --workload lru --steps 2 --warmup 3 --no-cpu --no-fgemm > gpurun_out/bench_config4.json 2> gpurun_out/bench_config4.err
python bench.py --p 251 --n 32768 --steps 5 --warmup 3 --no-cpu --no-fgemm > gpurun_out/bench_config5.json 2> gpurun_out/bench_config5.err
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
