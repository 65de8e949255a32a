# Round 2 call ba: ncu --set full of the final K19t variants (G = 4 direct <16, LP>; G = 32 direct <48>; G = 8192 partitioned <48>).
mkdir -p gpurun_out
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  python tools/ncu_stalls.py gpurun_out/${name}_raw.csv > gpurun_out/${name}_stalls.txt 2>&1
  rm -f /tmp/$name.ncu-rep
}
cap r2ba_gb4 "k_gbt" 0 1 python bench.py --workload groupby --mb-groups 4 --steps 1 --warmup 0
cap r2ba_gb32 "k_gbt" 0 1 python bench.py --workload groupby --mb-groups 32 --steps 1 --warmup 0
cap r2ba_gb8k "k_gbt|k_part_scatter_r|k_part_hist" 0 3 python bench.py --workload groupby --mb-groups 8192 --steps 1 --warmup 0
