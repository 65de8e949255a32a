timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for q in q9 q3; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 3 > gpurun_out/rq_$q.txt 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_compact_dense -s 1 -c 2 -o gpurun_out/q3_dense -f python tools/run_query.py --query q3 --sf 100 --reps 1 > gpurun_out/q3_dense.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
