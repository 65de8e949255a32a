# join µbench: launch list (time + DRAM per kernel) of one run
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/mb_join_launches.csv python bench.py --workload join --steps 1 --warmup 0 > gpurun_out/mb_join_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/mb_join_launches.csv > gpurun_out/mb_join_launches.txt 2>&1
gzip -f gpurun_out/mb_join_launches.csv
