# Round 2 call i: K10wr (Q9 ring), Q3 fused prefetch, Q18 sorted lookups; tests, A/B, ncu, bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 --timeout-method thread -x > gpurun_out/pytest_i.log 2>&1; echo exit=$? >> gpurun_out/pytest_i.log
for q in q9 q18; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 5 > gpurun_out/rq_${q}_i.txt 2>&1; done
SX_Q9_RING=0 timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9w_i.txt 2>&1
SX_Q3_PLAN=fused timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3fused_i.txt 2>&1
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
cap r2i_q9 "k_gb_wring" 1 1 python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q9
SX_Q3_PLAN=fused cap r2i_q3 "k_q3_fused" 1 1 python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q3
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err
