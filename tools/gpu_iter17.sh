for q in q1; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 5 > gpurun_out/rq_$q.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_tpch.py -x -q -p no:cacheprovider -k "q1 or dense" > gpurun_out/pytest_q1.log 2>&1; echo exit=$? >> gpurun_out/pytest_q1.log
