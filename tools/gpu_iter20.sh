timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 300 python tools/run_query.py --query q18 --sf 100 --reps 3 > gpurun_out/rq_q18.txt 2>&1
timeout 900 python bench.py --workload groupby --mb-groups 4,256,4096,65536,1048576,16777216 --steps 2 --warmup 1 > gpurun_out/mb_gb.json 2> gpurun_out/mb_gb.err
