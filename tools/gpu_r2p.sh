# Round 2 call p: K18p replicas, date fill; tests, group-by sweep, Q9, bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 --timeout-method thread > gpurun_out/pytest_p.log 2>&1; echo exit=$? >> gpurun_out/pytest_p.log
timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9_p.txt 2>&1
timeout 1200 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_p.json 2> gpurun_out/mb_gb_p.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_p.json 2> gpurun_out/bench_p.err
