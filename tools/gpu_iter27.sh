timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for q in q3 q9; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 3 > gpurun_out/rq_$q.txt 2>&1; done
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err
