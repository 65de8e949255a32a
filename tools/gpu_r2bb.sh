# Round 2 call bb: K19t <48> with a 4-slot fast probe.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "groupby" > gpurun_out/pytest_bb.log 2>&1; echo exit=$? >> gpurun_out/pytest_bb.log
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_bb.json 2> gpurun_out/mb_gb_bb.err
