timeout 600 python -m pytest tests/test_gpu_radix.py tests/test_gpu_ops.py -x -q -p no:cacheprovider > gpurun_out/pytest_part.log 2>&1; echo exit=$? >> gpurun_out/pytest_part.log
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join16.json 2> gpurun_out/mb_join16.err
