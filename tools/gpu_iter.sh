# iteration: full GPU tests + per-query timings + sort µbench
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for q in q1 q6 q3 q9 q18; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 3 > gpurun_out/rq_$q.txt 2>&1; done
timeout 600 python bench.py --workload sort --steps 3 --warmup 1 > gpurun_out/mb_sort.json 2> gpurun_out/mb_sort.err
