# Round 2 call n: Q3 two-chunk pass, K18s up to 200 KB; tests subset, Q3, group-by points, onesweep ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tpch.py tests/test_gpu_ops.py -q -p no:cacheprovider --timeout 200 --timeout-method thread -k "q3 or groupby or topk or sort" > gpurun_out/pytest_n.log 2>&1; echo exit=$? >> gpurun_out/pytest_n.log
timeout 300 python tools/run_query.py --query q3 --sf 100 --reps 5 > gpurun_out/rq_q3_n.txt 2>&1
timeout 900 python bench.py --workload groupby --mb-groups 1024,2048,4096 --steps 3 --warmup 1 > gpurun_out/mb_gb_n.json 2> gpurun_out/mb_gb_n.err
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  python tools/ncu_stalls.py gpurun_out/${name}_raw.csv > gpurun_out/${name}_stalls.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 30 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
cap r2n_os "k_onesweep" 3 1 python bench.py --workload sort --steps 1 --warmup 0 --mb-sort-log2 26
cap r2n_q3 "k_q3_fused|k_q3_orders" 2 2 python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q3
