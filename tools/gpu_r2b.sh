# Round 2: onesweep sort + partitioned join v2 (staged scatter, inline-value probe): tests, µbench A/B, launch lists.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_radix.py tests/test_gpu_ops.py -x -q -p no:cacheprovider --timeout 300 -k "sort or join or radix or partition" > gpurun_out/pytest_b.log 2>&1; echo exit=$? >> gpurun_out/pytest_b.log
timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort.json 2> gpurun_out/mb_sort.err
SX_SORT=lsd timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort_lsd.json 2> gpurun_out/mb_sort_lsd.err
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join.json 2> gpurun_out/mb_join.err
SX_PJ_INLINE=0 SX_PART_SCATTER=rowid timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_old.json 2> gpurun_out/mb_join_old.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz.json 2> gpurun_out/mb_joinz.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_join.csv python bench.py --workload join --steps 1 --warmup 0 > gpurun_out/ncu_join.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_sort.csv python bench.py --workload sort --steps 1 --warmup 0 > gpurun_out/ncu_sort.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 240 -v > gpurun_out/pytest_all.log 2>&1; echo exit=$? >> gpurun_out/pytest_all.log
