# Round 2 call x: K7p pair partition kernel — radix/join/groupby tests, sweep, join µbench (uniform, Zipf), ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_radix.py -q -p no:cacheprovider --timeout 300 --timeout-method thread -k "groupby or radix or join or partition" > gpurun_out/pytest_x.log 2>&1; echo exit=$? >> gpurun_out/pytest_x.log
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_x.json 2> gpurun_out/mb_gb_x.err
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_x.json 2> gpurun_out/mb_join_x.err
SX_PART_SCATTER=reg SX_PART_RANK=atomic timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_xa.json 2> gpurun_out/mb_join_xa.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz_x.json 2> gpurun_out/mb_joinz_x.err
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 40 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
cap r2x_gb1k "k_part_pair|k_gbt" 0 2 python bench.py --workload groupby --mb-groups 1024 --steps 1 --warmup 0
cap r2x_gb64k "k_part_pair|k_gbs_part" 0 2 python bench.py --workload groupby --mb-groups 65536 --steps 1 --warmup 0
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_join_x.csv python bench.py --workload join --steps 1 --warmup 0 > /dev/null 2>&1
