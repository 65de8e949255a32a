# Round 2 call an: end-of-session validation (after Q9 year byte + K10l cp.async) — all GPU tests, smoke, bench (SF100 / SF10 / SF0.01 /
# reference arm), µbenchmarks (group-by sweep, join uniform + Zipf, sort), the bench launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_an.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_an.log 2>&1; echo exit=$? >> gpurun_out/pytest_an.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_an.log 2>&1; echo exit=$? >> gpurun_out/smoke_an.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_an.json 2> gpurun_out/bench_an.err
timeout 600 python bench.py --sf 10 --no-e2e --no-cpu --steps 10 --warmup 3 > gpurun_out/bench_sf10_an.json 2> gpurun_out/bench_sf10_an.err
timeout 600 python bench.py --sf 0.01 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_sf001_an.json 2> gpurun_out/bench_sf001_an.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_an.json 2> gpurun_out/bench_ref_an.err
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_an.json 2> gpurun_out/mb_gb_an.err
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_an.json 2> gpurun_out/mb_join_an.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz_an.json 2> gpurun_out/mb_joinz_an.err
timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort_an.json 2> gpurun_out/mb_sort_an.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_an.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_an.log 2>&1
