timeout 900 python bench.py --workload groupby --steps 3 --warmup 1 > gpurun_out/mb_gb_v2.json 2> gpurun_out/mb_gb_v2.err
timeout 600 python bench.py --workload sort --steps 3 --warmup 1 > gpurun_out/mb_sort_v2.json 2> gpurun_out/mb_sort_v2.err
timeout 600 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz_v2.json 2> gpurun_out/mb_joinz_v2.err
