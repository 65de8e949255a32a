# Round 2 call am: K10w (Q9 lineitem pass) partkeys prefetched by cp.async.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tpch.py -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_am.log 2>&1; echo exit=$? >> gpurun_out/pytest_am.log
timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9_am.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_am.json 2> gpurun_out/bench_am.err
