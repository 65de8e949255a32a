timeout 900 python -m pytest tests/test_gpu_radix.py tests/test_gpu_ops.py -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload join --steps 2 --warmup 1 > gpurun_out/mb_join.json 2> gpurun_out/mb_join.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_join.csv python bench.py --workload join --mb-build-log2 25 --mb-probe-log2 28 --steps 1 --warmup 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_sort.csv python bench.py --workload sort --mb-sort-log2 26 --steps 1 --warmup 0 > /dev/null 2>&1
