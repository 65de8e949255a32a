# Round 2: K18 plain group-by, Q9 sorted date fill, L2 fetch granularity experiments.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -v -p no:cacheprovider --timeout 200 --timeout-method thread --durations 15 > gpurun_out/pytest_d.log 2>&1; echo exit=$? >> gpurun_out/pytest_d.log
timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9_new.txt 2>&1
for g in 32 64 128; do
  SX_L2_FETCH=$g timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9_l2f$g.txt 2>&1
  SX_L2_FETCH=$g timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3_l2f$g.txt 2>&1
done
G=4,64,1024,4096,65536,1048576,2097152,16777216
timeout 900 python bench.py --workload groupby --mb-groups $G --steps 3 --warmup 1 > gpurun_out/mb_gb.json 2> gpurun_out/mb_gb.err
SX_GB_SIMPLE=0 timeout 900 python bench.py --workload groupby --mb-groups $G --steps 2 --warmup 1 > gpurun_out/mb_gb_generic.json 2> gpurun_out/mb_gb_generic.err
SX_L2_FETCH=32 timeout 900 python bench.py --workload join --steps 2 --warmup 1 > gpurun_out/mb_join_l2f32.json 2> gpurun_out/mb_join_l2f32.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_gb.csv python bench.py --workload groupby --mb-groups 4,1024,65536,1048576 --steps 1 --warmup 0 > gpurun_out/ncu_gb.log 2>&1
timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3_new.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_onesweep|k_part_scatter_v|k_pji_probe" -s 3 -c 3 -o /tmp/r2_scat -f python bench.py --workload join --steps 1 --warmup 0 --mb-probe-log2 28 > gpurun_out/r2_scat.log 2>&1
python tools/rep_summary.py /tmp/r2_scat.ncu-rep r2_scat > gpurun_out/r2_scat_summary.txt 2>&1
ncu -i /tmp/r2_scat.ncu-rep --page raw --csv > gpurun_out/r2_scat_raw.csv 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_onesweep" -s 2 -c 1 -o /tmp/r2_os -f python bench.py --workload sort --steps 1 --warmup 0 --mb-sort-log2 26 > gpurun_out/r2_os.log 2>&1
python tools/rep_summary.py /tmp/r2_os.ncu-rep r2_os > gpurun_out/r2_os_summary.txt 2>&1
ncu -i /tmp/r2_os.ncu-rep --page source --csv --print-source sass > /tmp/r2_os_sass.csv 2>/dev/null
python tools/ncu_sass_hot.py /tmp/r2_os_sass.csv 30 > gpurun_out/r2_os_hot.txt 2>&1
python tools/ncu_stalls.py gpurun_out/r2_scat_raw.csv > gpurun_out/r2_scat_stalls.txt 2>&1
ncu -i /tmp/r2_os.ncu-rep --page raw --csv > gpurun_out/r2_os_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/r2_os_raw.csv > gpurun_out/r2_os_stalls.txt 2>&1
