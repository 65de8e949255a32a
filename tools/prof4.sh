# Q9 fused check + per-query timings + ncu launch lists of the µbenchmarks (small) + full captures
timeout 900 python -m pytest tests/test_gpu_tpch.py -x -q -p no:cacheprovider > gpurun_out/pytest_tpch.log 2>&1; echo exit=$? >> gpurun_out/pytest_tpch.log
for q in q9 q3 q18; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 3 > gpurun_out/rq_$q.txt 2>&1; done
# launch lists (cold, serialised): join (flat + partitioned) 2^24 x 2^27, group-by G=65536 and 4, sort 2^26
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_join.csv python bench.py --workload join --mb-build-log2 24 --mb-probe-log2 27 --steps 1 --warmup 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_gb.csv python bench.py --workload groupby --mb-gb-log2 27 --mb-groups 4,65536 --steps 1 --warmup 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_sort.csv python bench.py --workload sort --mb-sort-log2 26 --steps 1 --warmup 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_q3.csv python tools/run_query.py --query q3 --sf 100 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_compact_local -s 1 -c 2 -o gpurun_out/q3_probe -f python tools/run_query.py --query q3 --sf 100 --reps 1 > gpurun_out/q3_probe.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gb_shared -c 1 -o gpurun_out/q9_fused -f python tools/run_query.py --query q9 --sf 100 --reps 1 > gpurun_out/q9_fused.log 2>&1
