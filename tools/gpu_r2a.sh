# Round 2, first GPU call: full GPU tests + smoke, SF100 bench, ring (K9r/K10rr) on vs off, launch list.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
for q in q1 q18; do
  timeout 300 python tools/run_query.py --query $q --sf 100 --reps 5 > gpurun_out/rq_${q}_ring.txt 2>&1
  SX_RING=0 timeout 300 python tools/run_query.py --query $q --sf 100 --reps 5 > gpurun_out/rq_${q}_noring.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_sf100.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_bench.log 2>&1
