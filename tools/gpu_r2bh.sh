# Round 2 call bh: K18p2's level-1 partitions claimed dynamically — group-by tests, the large-G sweep points.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "groupby" > gpurun_out/pytest_bh.log 2>&1; echo exit=$? >> gpurun_out/pytest_bh.log
timeout 900 python bench.py --workload groupby --mb-groups 2097152,4194304,8388608,16777216,33554432,67108864 --steps 2 --warmup 1 > gpurun_out/mb_gb_bh.json 2> gpurun_out/mb_gb_bh.err
