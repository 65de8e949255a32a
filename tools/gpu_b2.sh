timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_b1.json 2> gpurun_out/bench_b1.err
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_b2.json 2> gpurun_out/bench_b2.err
