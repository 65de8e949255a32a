# Round 2 call as: K19t <48> up to 32768 hinted groups (~32 per partition at 1024 partitions).
mkdir -p gpurun_out
timeout 900 python bench.py --workload groupby --mb-groups 16384,32768 --steps 3 --warmup 1 > gpurun_out/mb_gb_as.json 2> gpurun_out/mb_gb_as.err
timeout 900 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "fixed_signature or k19" > gpurun_out/pytest_as.log 2>&1; echo exit=$? >> gpurun_out/pytest_as.log
