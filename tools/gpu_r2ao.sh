# Round 2 call ao: Q18 fused orders/customer lookup kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tpch.py -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_ao.log 2>&1; echo exit=$? >> gpurun_out/pytest_ao.log
timeout 300 python tools/run_query.py --query q18 --sf 100 --reps 5 > gpurun_out/rq_q18_ao.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_ao.json 2> gpurun_out/bench_ao.err
