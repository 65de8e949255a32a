# Round 2 call r: group-by sweep at HEAD + ncu captures of the K18 kernels at G = 4, 64, 65536, 2^22.
mkdir -p gpurun_out
timeout 1500 python bench.py --workload groupby --steps 2 --warmup 1 > gpurun_out/mb_gb_r.json 2> gpurun_out/mb_gb_r.err
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
for G in 4 64 65536 4194304; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_gb${G}_r.csv python bench.py --workload groupby --mb-groups $G --steps 1 --warmup 0 > /dev/null 2>&1
done
cap r2r_gb4 "k_gbs" 0 2 python bench.py --workload groupby --mb-groups 4 --steps 1 --warmup 0
cap r2r_gb64k "k_gbs|k_part" 0 4 python bench.py --workload groupby --mb-groups 65536 --steps 1 --warmup 0
