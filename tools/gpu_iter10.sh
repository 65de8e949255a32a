timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for q in q1 q6; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 3 > gpurun_out/rq_$q.txt 2>&1; done
SX_BULK=0 timeout 300 python tools/run_query.py --query q1 --sf 100 --reps 3 > gpurun_out/rq_q1_nobulk.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_ncu.log 2>&1
