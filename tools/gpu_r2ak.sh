# Round 2 call ak: K10l with a cp.async double buffer; shared-atomic throughput µbench.
mkdir -p gpurun_out
./tools/ubench/atoms > gpurun_out/atoms_ak.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_tpch.py -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_ak.log 2>&1; echo exit=$? >> gpurun_out/pytest_ak.log
timeout 300 python tools/run_query.py --query q18 --sf 100 --reps 5 > gpurun_out/rq_q18_ak.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_ak.json 2> gpurun_out/bench_ak.err
