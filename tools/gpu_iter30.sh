timeout 300 python tools/run_query.py --query q6 --sf 100 --reps 5 > gpurun_out/rq_q6.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_tpch.py -x -q -p no:cacheprovider -k "q6 or dense or bulk" > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
