# Round 2 call az: Q9 year fill staged in shared memory — TPC-H tests, Q9 per-operator times, bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tpch.py -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_az.log 2>&1; echo exit=$? >> gpurun_out/pytest_az.log
timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9_az.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_az.json 2> gpurun_out/bench_az.err
