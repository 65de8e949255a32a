# Round 2 call ai (experiment): is the K8i probe bound by its single output cursor? (SX_PJ_NOCLAIM: positions = probe index, all-hit input only)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_join_ai.csv python tools/join_one.py 2 > gpurun_out/ncu_join_ai.log 2>&1
SX_PJ_NOCLAIM=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_join_ai_nc.csv python tools/join_one.py 2 > gpurun_out/ncu_join_ai_nc.log 2>&1
