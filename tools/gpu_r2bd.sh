# Round 2 call bd: final validation (K19t 4-slot probe, <48> above 1024) — all GPU tests, smoke, bench (SF100 / SF10 / SF0.01 /
# reference arm), µbenchmarks (group-by sweep, join uniform + Zipf, sort), the bench launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_bd.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_bd.log 2>&1; echo exit=$? >> gpurun_out/pytest_bd.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_bd.log 2>&1; echo exit=$? >> gpurun_out/smoke_bd.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_bd.json 2> gpurun_out/bench_bd.err
timeout 600 python bench.py --sf 10 --no-e2e --no-cpu --steps 10 --warmup 3 > gpurun_out/bench_sf10_bd.json 2> gpurun_out/bench_sf10_bd.err
timeout 600 python bench.py --sf 0.01 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_sf001_bd.json 2> gpurun_out/bench_sf001_bd.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_bd.json 2> gpurun_out/bench_ref_bd.err
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_bd.json 2> gpurun_out/mb_gb_bd.err
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_bd.json 2> gpurun_out/mb_join_bd.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz_bd.json 2> gpurun_out/mb_joinz_bd.err
timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort_bd.json 2> gpurun_out/mb_sort_bd.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bd.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_bd.log 2>&1
