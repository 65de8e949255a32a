# one-off profiling batch (scratch; outputs summarised under profiles/)
cap() {  # cap <name> <kernel regex> <query> [launch-skip]
  ncu --set full --import-source on --clock-control none -k regex:$2 -s ${4:-0} -c 1 -o /tmp/$1 -f python tools/run_query.py --query $3 --sf 100 --reps 1 > /dev/null 2>&1
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_sass.csv 2>&1
}
cap gbsh_q9 k_gb_shared q9
cap probe_q3 "k_compact_local<sx::ProbeFnT" q3 1
cap small_q6 k_gb_small q6
