for cfg in "16 3" "32 3" "32 2" "64 2" "8 3"; do
  set -- $cfg
  SX_PJ_PART_MB=$1 SX_PJ_L2DIV=$2 timeout 600 python bench.py --workload join --steps 3 --warmup 1 > gpurun_out/mbj_$1_$2.json 2> gpurun_out/mbj_$1_$2.err
done
