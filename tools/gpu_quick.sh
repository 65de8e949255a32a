# quick GPU iteration: targeted tests + per-query timings at SF100
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${TESTS:-} > gpurun_out/pytest_quick.log 2>&1; echo exit=$? >> gpurun_out/pytest_quick.log
for q in ${QUERIES:-q1 q6}; do timeout 300 python tools/run_query.py --query $q --sf 100 --reps 3 > gpurun_out/rq_$q.txt 2>&1; done
