# Round 2 call z: K8f flat inline join — radix/join tests, join µbench (uniform, Zipf) with the three strategies.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_radix.py -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_z.log 2>&1; echo exit=$? >> gpurun_out/pytest_z.log
timeout 900 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mb_join_z.json 2> gpurun_out/mb_join_z.err
timeout 900 python bench.py --workload join-zipf --steps 3 --warmup 1 > gpurun_out/mb_joinz_z.json 2> gpurun_out/mb_joinz_z.err
cap() {  # cap <name> <regex> <skip> <count> <cmd...>
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $sk -c $ct -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/rep_summary.py /tmp/$name.ncu-rep "$name" > gpurun_out/${name}_summary.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  rm -f /tmp/$name.ncu-rep
}
cap r2z_kf "k_pji_build|k_pji_probe" 0 2 python tools/join_one.py 3
