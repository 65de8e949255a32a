# Round 2 call f: tests, Q3/Q18/Q6 A/B, µbench sweep, SF100 bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -v -p no:cacheprovider --timeout 200 --timeout-method thread --durations 10 > gpurun_out/pytest_f.log 2>&1; echo exit=$? >> gpurun_out/pytest_f.log
for q in q3 q18 q6; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 5 > gpurun_out/rq_${q}_f.txt 2>&1; done
SX_Q3_PLAN=ops timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3ops_f.txt 2>&1
SX_Q6_LAZY3=1 timeout 300 python tools/run_query.py --query q6 --sf 100 --reps 5 > gpurun_out/rq_q6l3_f.txt 2>&1
timeout 900 python bench.py --workload groupby --steps 3 --warmup 1 > gpurun_out/mb_gb_f.json 2> gpurun_out/mb_gb_f.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_gb_f.csv python bench.py --workload groupby --mb-groups 4,64,1024,65536,1048576 --steps 1 --warmup 0 > gpurun_out/ncu_gb_f.log 2>&1
