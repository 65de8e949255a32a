# ncu --set full captures of the top kernels (scratch; summaries go to profiles/)
cap() {  # cap <name> <kernel regex> <query> [launch-skip] [count]
  ncu --set full --import-source on --clock-control none -k regex:"$2" -s ${4:-0} -c ${5:-1} -o gpurun_out/$1 -f python tools/run_query.py --query $3 --sf 100 --reps 1 > gpurun_out/$1.log 2>&1
}
cap q1_gb_small k_gb_small q1
cap q6_gb_small k_gb_small q6
cap q9_probe "k_compact_local<sx::ProbeFnT" q9 0 3
cap q9_gather k_gather_multi q9 0 2
cap q3_probe "k_compact_local<sx::ProbeFnT" q3 0 2
cap q18_runs k_runs_agg q18
ls -la gpurun_out/
