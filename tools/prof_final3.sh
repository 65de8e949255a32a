# end-of-round evidence v11: tests, bench lines (SF100 default with e2e + cpu baseline, SF10, SF0.01),
# launch list, ncu --set full summaries of the dominant kernels
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 20 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --sf 10 --no-e2e --no-cpu > gpurun_out/bench_sf10.json 2> gpurun_out/bench_sf10.err
timeout 600 python bench.py --sf 0.01 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_sf001.json 2> gpurun_out/bench_sf001.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_ncu.log 2>&1
RQ="python tools/run_query.py --sf 100 --reps 1"
cap j_q1 k_gb_dense 0 1 $RQ --query q1
cap j_q6 k_gb_dense 0 1 $RQ --query q6
cap j_q9_wscan k_gb_wscan 0 1 $RQ --query q9
cap j_q9_contains k_compact_dense 0 1 $RQ --query q9
cap j_q3 k_compact 2 4 $RQ --query q3
cap j_q18 k_runs_own_dense 0 1 $RQ --query q18
du -sh gpurun_out
