timeout 900 python -m pytest tests/test_gpu_tpch.py -x -q -p no:cacheprovider -k "ring or q18 or committed or hand" > gpurun_out/pytest_q18r.log 2>&1; echo exit=$? >> gpurun_out/pytest_q18r.log
timeout 300 python tools/run_query.py --query q18 --sf 100 --reps 5 > gpurun_out/rq_q18_ring.txt 2>&1
SX_RING=0 timeout 300 python tools/run_query.py --query q18 --sf 100 --reps 5 > gpurun_out/rq_q18_old.txt 2>&1
CAPS="r2_q18ring:k_runs_ring:0:1:q18" bash tools/gpu_cap.sh
