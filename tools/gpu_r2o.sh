# Round 2 call o: onesweep staging, K10w U=3: tests subset, Q9, sort µbench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tpch.py tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 200 --timeout-method thread -k "q9 or sort or topk or committed or live" > gpurun_out/pytest_o.log 2>&1; echo exit=$? >> gpurun_out/pytest_o.log
timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9_o.txt 2>&1
timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort_o.json 2> gpurun_out/mb_sort_o.err
