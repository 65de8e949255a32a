# Round 2 call ay: radix-select top-k with an early exit once the candidates fit the final sort.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_tpch.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "sort or topk or q3 or committed or live" > gpurun_out/pytest_ay.log 2>&1; echo exit=$? >> gpurun_out/pytest_ay.log
timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3_ay.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_ay.json 2> gpurun_out/bench_ay.err
