# Round 2 call ab: K18p fan-out A/B (SX_GB_PBITS = 8 / 9 / 10) at G = 8192 .. 2^19.
mkdir -p gpurun_out
for b in 10 9 8; do
  SX_GB_PBITS=$b timeout 900 python bench.py --workload groupby --mb-groups 8192,32768,131072,524288 --steps 2 --warmup 1 > gpurun_out/mb_gb_ab$b.json 2> gpurun_out/mb_gb_ab$b.err
done
SX_GB_PBITS=9 timeout 600 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "fixed_signature or plain_shape" > gpurun_out/pytest_ab.log 2>&1; echo exit=$? >> gpurun_out/pytest_ab.log
