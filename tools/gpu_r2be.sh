# Round 2 call be: dynamic work claims in K18p (partitions) and K19t (chunks).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "groupby" > gpurun_out/pytest_be.log 2>&1; echo exit=$? >> gpurun_out/pytest_be.log
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_be.json 2> gpurun_out/mb_gb_be.err
