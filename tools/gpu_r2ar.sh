# Round 2 call ar: K19t variants <16, LP> / <48, !LP> dispatched per hint range.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "groupby" > gpurun_out/pytest_ar.log 2>&1; echo exit=$? >> gpurun_out/pytest_ar.log
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_ar.json 2> gpurun_out/mb_gb_ar.err
