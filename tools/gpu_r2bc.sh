# Round 2 call bc: A/B of the K19t variants over 64..16384 groups (SX_GB_K19V=48 forces <48, ~16 per partition).
mkdir -p gpurun_out
timeout 900 python bench.py --workload groupby --mb-groups 64,128,256,512,1024,2048 --steps 3 --warmup 1 > gpurun_out/mb_gb_bc16.json 2> gpurun_out/mb_gb_bc16.err
SX_GB_K19V=48 timeout 900 python bench.py --workload groupby --mb-groups 64,128,256,512,1024,2048 --steps 3 --warmup 1 > gpurun_out/mb_gb_bc48.json 2> gpurun_out/mb_gb_bc48.err
