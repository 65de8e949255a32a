timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload groupby --mb-groups 4,256,4096,65536,1048576,16777216 --steps 2 --warmup 1 > gpurun_out/mb_gb.json 2> gpurun_out/mb_gb.err
timeout 900 python bench.py --workload join --steps 2 --warmup 1 > gpurun_out/mb_join.json 2> gpurun_out/mb_join.err
