# Round 2 call ae: join µbench sensitivity (partition table size, waves per L2) + per-kernel times without cache flushes.
mkdir -p gpurun_out
for mb in 16 32 64; do for dv in 2 3; do
  SX_PJ_PART_MB=$mb SX_PJ_L2DIV=$dv timeout 600 python tools/join_one.py 2 > /dev/null 2>&1
  echo "== part_mb=$mb l2div=$dv" >> gpurun_out/join_sens_ae.txt
  SX_PJ_PART_MB=$mb SX_PJ_L2DIV=$dv timeout 600 python bench.py --workload join --steps 3 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_partitioned'], d['parity'][-3:])" >> gpurun_out/join_sens_ae.txt
done; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_join_ae.csv python tools/join_one.py 2 > gpurun_out/ncu_join_ae.log 2>&1
