# Round 2 call e: q18-big hang diagnosis, tests, A/B timings, ncu captures.
mkdir -p gpurun_out
for v in "SX_GB_SORTED=2" "SX_GB_SORTED=2 SX_RUNS_LEAN=0" "SX_GB_SORTED=0" "SX_GB_SORTED=2 SX_GB_SIMPLE=0"; do
  echo "== $v" >> gpurun_out/diag_q18big.log
  env $v timeout 90 python tools/diag_q18big.py >> gpurun_out/diag_q18big.log 2>&1; echo "exit=$?" >> gpurun_out/diag_q18big.log
done
timeout 1200 python -m pytest tests -m gpu -v -p no:cacheprovider --timeout 200 --timeout-method thread --durations 15 --deselect "tests/test_gpu_tpch.py::test_q18_owned_runs[big]" > gpurun_out/pytest_e.log 2>&1; echo exit=$? >> gpurun_out/pytest_e.log
for q in q3 q9 q18; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 5 > gpurun_out/rq_${q}_e.txt 2>&1; done
timeout 600 python bench.py --workload sort --steps 5 --warmup 2 > gpurun_out/mb_sort_e.json 2> gpurun_out/mb_sort_e.err
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_e.json 2> gpurun_out/mb_join_e.err
timeout 900 python bench.py --workload groupby --mb-groups 4,64,1024,4096,65536,1048576,2097152 --steps 3 --warmup 1 > gpurun_out/mb_gb_e.json 2> gpurun_out/mb_gb_e.err
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
cap r2e_q3 "k_q3_fused" 1 1 python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q3
cap r2e_q18 "k_runs_lean" 1 1 python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q18
cap r2e_q9 "k_gb_wscan|k_date_fill" 2 2 python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q9
cap r2e_os "k_onesweep" 3 1 python bench.py --workload sort --steps 1 --warmup 0 --mb-sort-log2 26
cap r2e_part "k_part_scatter_r|k_pji_probe" 1 3 python bench.py --workload join --steps 1 --warmup 0 --mb-probe-log2 28
cap r2e_gb "k_gbs_local|k_gbs_part" 0 2 python bench.py --workload groupby --mb-groups 64,65536 --steps 1 --warmup 0 --mb-gb-log2 28
