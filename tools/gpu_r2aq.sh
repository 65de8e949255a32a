# Round 2 call aq: K19t with 48 ids per warp (lane-private count/sum, per-warp min/max) up to 16384 hinted groups.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "groupby" > gpurun_out/pytest_aq.log 2>&1; echo exit=$? >> gpurun_out/pytest_aq.log
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_aq.json 2> gpurun_out/mb_gb_aq.err
