# Round 2 call au: K8i probe with 32-bit slot indices at 4 CTAs/SM — radix/join tests, join µbench, launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_radix.py tests/test_gpu_sharded.py -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_au.log 2>&1; echo exit=$? >> gpurun_out/pytest_au.log
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_au.json 2> gpurun_out/mb_join_au.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz_au.json 2> gpurun_out/mb_joinz_au.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_join_au.csv python tools/join_one.py 2 > gpurun_out/ncu_join_au.log 2>&1
