# Round 2 call ax: persisting-L2 access window over the join's wave tables — radix tests, join µbench A/B, launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_radix.py -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_ax.log 2>&1; echo exit=$? >> gpurun_out/pytest_ax.log
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_ax.json 2> gpurun_out/mb_join_ax.err
SX_PJ_PERSIST=0 timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_ax0.json 2> gpurun_out/mb_join_ax0.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz_ax.json 2> gpurun_out/mb_joinz_ax.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_join_ax.csv python tools/join_one.py 2 > gpurun_out/ncu_join_ax.log 2>&1
