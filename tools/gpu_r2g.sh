# Round 2 call g: tests, Q3 fused (records) vs ops, Q18, sort match/ballot, join, bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 --timeout-method thread --durations 8 > gpurun_out/pytest_g.log 2>&1; echo exit=$? >> gpurun_out/pytest_g.log
SX_Q3_PLAN=fused timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3fused_g.txt 2>&1
for q in q3 q18; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 5 > gpurun_out/rq_${q}_g.txt 2>&1; done
timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort_g.json 2> gpurun_out/mb_sort_g.err
SX_SORT_RANK=ballot timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort_gb.json 2> gpurun_out/mb_sort_gb.err
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_g.json 2> gpurun_out/mb_join_g.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz_g.json 2> gpurun_out/mb_joinz_g.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_join_g.csv python bench.py --workload join --steps 1 --warmup 0 > gpurun_out/ncu_join_g.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_sort_g.csv python bench.py --workload sort --steps 1 --warmup 0 > gpurun_out/ncu_sort_g.log 2>&1
