# Round 2 call m: K18p2, K14w tuning; tests, group-by sweep, Q3, bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 --timeout-method thread > gpurun_out/pytest_m.log 2>&1; echo exit=$? >> gpurun_out/pytest_m.log
timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3_m.txt 2>&1
SX_TOPK=select timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3sel_m.txt 2>&1
timeout 1200 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_m.json 2> gpurun_out/mb_gb_m.err
timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort_m.json 2> gpurun_out/mb_sort_m.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err
