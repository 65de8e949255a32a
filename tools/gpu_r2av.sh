# Round 2 call av: ncu --set full of one K8i probe wave and the K7r scatter of the join µbench.
mkdir -p gpurun_out
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 30 > gpurun_out/${name}_hot.txt 2>&1
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
cap r2av_probe "k_pji_probe" 10 1 python tools/join_one.py 2
cap r2av_scatter "k_part_scatter_r" 1 1 python tools/join_one.py 2
