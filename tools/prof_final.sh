timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for q in q6 q9; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 3 > gpurun_out/rq_$q.txt 2>&1; done
# round-1 ncu evidence for the current kernels (summaries go to profiles/)
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 25 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
RQ="python tools/run_query.py --sf 100 --reps 1"
cap f_q1_dense k_gb_dense 0 1 $RQ --query q1
cap f_q6_dense k_gb_dense 0 1 $RQ --query q6
cap f_q9_pg k_gb_shared 0 1 $RQ --query q9
cap f_q9_semi k_compact_dense 0 1 $RQ --query q9
cap f_q3_probe k_compact 2 4 $RQ --query q3
cap f_q18_runs k_runs_own_dense 0 1 $RQ --query q18
cap f_pj_probe k_pj_probe 4 1 python bench.py --workload join --mb-build-log2 25 --mb-probe-log2 28 --steps 1 --warmup 0
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_ncu.log 2>&1
du -sh gpurun_out
