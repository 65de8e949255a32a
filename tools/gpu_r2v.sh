# Round 2 call v: K19t branch-free fast path, G/4 fan-out (hint <= 4096) — parity tests, sweep, ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "groupby" > gpurun_out/pytest_v.log 2>&1; echo exit=$? >> gpurun_out/pytest_v.log
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_v.json 2> gpurun_out/mb_gb_v.err
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 40 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
cap r2v_gb4 "k_gbt" 0 1 python bench.py --workload groupby --mb-groups 4 --steps 1 --warmup 0
cap r2v_gb64 "k_gbt|k_part_scatter" 0 2 python bench.py --workload groupby --mb-groups 64 --steps 1 --warmup 0
cap r2v_gb1k "k_gbt|k_part_scatter" 0 2 python bench.py --workload groupby --mb-groups 1024 --steps 1 --warmup 0
