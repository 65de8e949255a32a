# Q9 scan variants: parity tests, SF100 bench per variant, ncu --set full of the K10w kernel
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 20 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
timeout 900 python -m pytest tests/test_gpu_tpch.py -x -q -p no:cacheprovider -k "q9" > gpurun_out/pytest_q9.log 2>&1; echo exit=$? >> gpurun_out/pytest_q9.log
SX_Q9_SCAN=wscan timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_wscan.json 2> gpurun_out/bench_wscan.err
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_gather.json 2> gpurun_out/bench_gather.err
SX_Q9_SCAN=wscan cap w_q9 k_gb_wscan 0 1 python tools/run_query.py --sf 100 --reps 1 --query q9
