# Round 2 call l: tests, warp top-k, partition histogram; µbenchmarks, bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 --timeout-method thread > gpurun_out/pytest_l.log 2>&1; echo exit=$? >> gpurun_out/pytest_l.log
for q in q3 q9; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 5 > gpurun_out/rq_${q}_l.txt 2>&1; done
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_l.json 2> gpurun_out/mb_join_l.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz_l.json 2> gpurun_out/mb_joinz_l.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_sf100_l.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_bench_l.log 2>&1
