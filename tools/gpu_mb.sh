# H5 tests + operator µbenchmarks (outputs in gpurun_out/)
timeout 900 python -m pytest tests/test_gpu_radix.py -x -q -p no:cacheprovider > gpurun_out/pytest_radix.log 2>&1; echo exit=$? >> gpurun_out/pytest_radix.log
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join.json 2> gpurun_out/mb_join.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_join_zipf.json 2> gpurun_out/mb_join_zipf.err
timeout 600 python bench.py --workload sort --steps 3 --warmup 1 > gpurun_out/mb_sort.json 2> gpurun_out/mb_sort.err
timeout 900 python bench.py --workload groupby --mb-groups 4,256,65536,1048576,16777216,67108864 --steps 3 --warmup 1 > gpurun_out/mb_gb.json 2> gpurun_out/mb_gb.err
