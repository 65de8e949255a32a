# Round 2 call q (session 3 start): full GPU tests, Q9/Q3 queries, bench, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_q.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_q.log 2>&1; echo exit=$? >> gpurun_out/pytest_q.log
timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9_q.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 1 --warmup 3 > gpurun_out/ncu_q.log 2>&1
