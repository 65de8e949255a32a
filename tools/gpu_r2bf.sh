# Round 2 call bf: final validation (dynamic work claims in the group-by) — all GPU tests, smoke, bench (SF100 / SF10 / SF0.01 /
# reference arm), µbenchmarks (group-by sweep, join uniform + Zipf, sort), the bench launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_bf.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_bf.log 2>&1; echo exit=$? >> gpurun_out/pytest_bf.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_bf.log 2>&1; echo exit=$? >> gpurun_out/smoke_bf.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_bf.json 2> gpurun_out/bench_bf.err
timeout 600 python bench.py --sf 10 --no-e2e --no-cpu --steps 10 --warmup 3 > gpurun_out/bench_sf10_bf.json 2> gpurun_out/bench_sf10_bf.err
timeout 600 python bench.py --sf 0.01 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_sf001_bf.json 2> gpurun_out/bench_sf001_bf.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_bf.json 2> gpurun_out/bench_ref_bf.err
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_bf.json 2> gpurun_out/mb_gb_bf.err
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_bf.json 2> gpurun_out/mb_join_bf.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz_bf.json 2> gpurun_out/mb_joinz_bf.err
timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort_bf.json 2> gpurun_out/mb_sort_bf.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bf.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_bf.log 2>&1
