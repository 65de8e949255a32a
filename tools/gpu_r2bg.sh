# Round 2 call bg: group-by tests after the A/B-switch fix; SX_GB_K19V=16/48 smoke on two sweep points.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "groupby" > gpurun_out/pytest_bg.log 2>&1; echo exit=$? >> gpurun_out/pytest_bg.log
SX_GB_K19V=16 timeout 600 python bench.py --workload groupby --mb-groups 32,2048 --steps 2 --warmup 1 > gpurun_out/mb_gb_bg16.json 2> gpurun_out/mb_gb_bg16.err
SX_GB_K19V=48 timeout 600 python bench.py --workload groupby --mb-groups 32,2048 --steps 2 --warmup 1 > gpurun_out/mb_gb_bg48.json 2> gpurun_out/mb_gb_bg48.err
