timeout 1200 python -m pytest tests/test_gpu_ops.py -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb.json 2> gpurun_out/mb_gb.err
