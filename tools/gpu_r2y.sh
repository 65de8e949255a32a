# Round 2 call y: K20 global-table reductions (4096 < G <= 2^21) — group-by tests, sweep, ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "groupby" > gpurun_out/pytest_y.log 2>&1; echo exit=$? >> gpurun_out/pytest_y.log
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_y.json 2> gpurun_out/mb_gb_y.err
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 40 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
cap r2y_gb64k "k_gr" 0 1 python bench.py --workload groupby --mb-groups 65536 --steps 1 --warmup 0
cap r2y_gb2m "k_gr" 0 1 python bench.py --workload groupby --mb-groups 2097152 --steps 1 --warmup 0
