# Round 2 call aj: ncu --set full of Q18's k_runs_lean and Q3's k_q3_orders (what bounds them).
mkdir -p gpurun_out
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 40 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
cap r2aj_q18 "k_runs_lean" 1 1 python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q18
cap r2aj_q3 "k_q3_orders|k_q3_fused" 2 2 python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q3
