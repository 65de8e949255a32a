timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload sort --steps 3 --warmup 1 > gpurun_out/mb_sort.json 2> gpurun_out/mb_sort.err
