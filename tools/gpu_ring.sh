# Q1 ring (K9r): targeted tests, then per-query timings at SF100, ring on vs off
timeout 900 python -m pytest tests/test_gpu_tpch.py -x -q -p no:cacheprovider -k "ring or q1 or committed or hand" > gpurun_out/pytest_ring.log 2>&1; echo exit=$? >> gpurun_out/pytest_ring.log
timeout 300 python tools/run_query.py --query q1 --sf 100 --reps 5 > gpurun_out/rq_q1_ring.txt 2>&1
SX_RING=0 timeout 300 python tools/run_query.py --query q1 --sf 100 --reps 5 > gpurun_out/rq_q1_k9d.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gb_ring -c 3 python tools/run_query.py --query q1 --sf 100 --reps 3 > gpurun_out/ncu_ring.txt 2>&1
