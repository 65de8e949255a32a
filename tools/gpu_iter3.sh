timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_tpch.py -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for q in q3 q9 q18; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 3 > gpurun_out/rq_$q.txt 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gb_shared -c 1 -o gpurun_out/q9_pg -f python tools/run_query.py --query q9 --sf 100 --reps 1 > gpurun_out/q9_pg.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_q9.csv python tools/run_query.py --query q9 --sf 100 --reps 1 > /dev/null 2>&1
