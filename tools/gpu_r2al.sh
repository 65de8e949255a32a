# Round 2 call al: k_q3_orders with a cp.async double buffer.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tpch.py -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_al.log 2>&1; echo exit=$? >> gpurun_out/pytest_al.log
timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3_al.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_al.json 2> gpurun_out/bench_al.err
