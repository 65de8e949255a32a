# Round 2 call k: Q9 partsupp word index; tests, Q9 A/B, bench + launch list.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 --timeout-method thread -x > gpurun_out/pytest_k.log 2>&1; echo exit=$? >> gpurun_out/pytest_k.log
timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9_k.txt 2>&1
SX_Q9_PSW=0 timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9t_k.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_gb_wscan|k_psw" -c 12 --csv --log-file gpurun_out/launches_q9_k.csv python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q9 > gpurun_out/ncu_q9_k.log 2>&1
