# Round 2 call aa: K19t with 12 warps per CTA — fixed-signature tests, sweep points.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "fixed_signature or plain_shape" > gpurun_out/pytest_aa.log 2>&1; echo exit=$? >> gpurun_out/pytest_aa.log
timeout 900 python bench.py --workload groupby --mb-groups 4,16,64,1024,4096 --steps 3 --warmup 1 > gpurun_out/mb_gb_aa.json 2> gpurun_out/mb_gb_aa.err
