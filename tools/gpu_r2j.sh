# Round 2 call j: fused orders bitmap for Q3; tests, Q3 timings, bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 --timeout-method thread -x > gpurun_out/pytest_j.log 2>&1; echo exit=$? >> gpurun_out/pytest_j.log
timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3_j.txt 2>&1
SX_Q3_PLAN=ops timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3ops_j.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_sf100_j.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_bench_j.log 2>&1
