# usage: CAPS="name:regex:skip:count:query ..." bash tools/gpu_cap.sh  — ncu --set full summaries
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_hot.py /tmp/${name}_sass.csv 30 > gpurun_out/${name}_hot.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  rm -f /tmp/$name.ncu-rep /tmp/${name}_sass.csv
}
for c in $CAPS; do
  IFS=: read name rx sk ct q <<< "$c"
  cap $name $rx $sk $ct python tools/run_query.py --sf ${SF:-100} --reps 1 --query $q
done
