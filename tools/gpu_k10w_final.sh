cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 20 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
cap m_q9_wscan k_gb_wscan 0 1 python tools/run_query.py --sf 100 --reps 1 --query q9
