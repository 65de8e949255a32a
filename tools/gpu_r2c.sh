# Round 2: K10l (Q18 lean runs), K10q (Q3 fused), sort/join fixes (no match_any): tests, A/B timings, launch lists.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 240 > gpurun_out/pytest_c.log 2>&1; echo exit=$? >> gpurun_out/pytest_c.log
for q in q3 q18; do
  timeout 300 python tools/run_query.py --query $q --sf 100 --reps 5 > gpurun_out/rq_${q}_new.txt 2>&1
done
SX_Q3_PLAN=ops timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3_ops.txt 2>&1
SX_RUNS_LEAN=0 timeout 300 python tools/run_query.py --query q18 --sf 100 --reps 5 > gpurun_out/rq_q18_k10r.txt 2>&1
timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort.json 2> gpurun_out/mb_sort.err
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join.json 2> gpurun_out/mb_join.err
SX_PJ_INLINE=0 timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_noinl.json 2> gpurun_out/mb_join_noinl.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_join.csv python bench.py --workload join --steps 1 --warmup 0 > gpurun_out/ncu_join.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_sort.csv python bench.py --workload sort --steps 1 --warmup 0 > gpurun_out/ncu_sort.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
