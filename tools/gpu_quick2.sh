timeout 600 python -m pytest tests/test_gpu_tpch.py -x -q -p no:cacheprovider -k "q18 or committed or live or empty or wide" > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 300 python tools/run_query.py --query q18 --sf 100 --reps 3 > gpurun_out/rq_q18.txt 2>&1
