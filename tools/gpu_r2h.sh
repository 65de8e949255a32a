# Round 2 call h: tests, Q3 fused v3 vs ops, Q6 (K9d dead-row skip), K18 ncu, bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 --timeout-method thread --durations 5 > gpurun_out/pytest_h.log 2>&1; echo exit=$? >> gpurun_out/pytest_h.log
SX_Q3_PLAN=fused timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3fused_h.txt 2>&1
for q in q3 q6 q1; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 5 > gpurun_out/rq_${q}_h.txt 2>&1; done
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  python tools/ncu_stalls.py gpurun_out/${name}_raw.csv > gpurun_out/${name}_stalls.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 25 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
SX_Q3_PLAN=fused cap r2h_q3 "k_q3_fused|k_q3_carry" 2 2 python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q3
cap r2h_gb4 "k_gbs_local" 1 1 python bench.py --workload groupby --mb-groups 4 --steps 1 --warmup 0 --mb-gb-log2 28
cap r2h_gb64k "k_gbs_part" 1 1 python bench.py --workload groupby --mb-groups 65536 --steps 1 --warmup 0 --mb-gb-log2 28
cap r2h_q6 "k_gb_dense" 1 1 python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q6
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
