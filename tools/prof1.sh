# one-off profiling batch (scratch; outputs summarised under profiles/)
cap() {  # cap <name> <kernel regex> <query>
  ncu --set full --import-source on --clock-control none -k regex:$2 -c 1 -o /tmp/$1 -f python tools/run_query.py --query $3 --sf 100 --reps 1 > /dev/null 2>&1
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_sass.csv 2>&1
}
timeout 600 python -m pytest tests/test_gpu_ops.py -q -m gpu -p no:cacheprovider -x -k groupby > gpurun_out/pytest_gb.log 2>&1; echo exit=$? >> gpurun_out/pytest_gb.log
python tools/run_query.py --query q9 --sf 100 --reps 3 > gpurun_out/rq_q9_b.txt 2>&1
cap runs_agg k_runs_agg q18
cap gb_small_q1 k_gb_small q1
cap probe_inner_q9 k_probe_inner q9
cap gb_shared_q9 k_gb_shared q9
du -sh gpurun_out/*
