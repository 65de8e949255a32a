# Round 2 call ad: Q9 partsupp' table packed into 8-byte slots — TPC-H tests, Q9 A/B, ncu of K10w.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tpch.py -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/pytest_ad.log 2>&1; echo exit=$? >> gpurun_out/pytest_ad.log
timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9_ad.txt 2>&1
SX_PT_NOPACK=1 timeout 300 python tools/run_query.py --query q9 --sf 100 --reps 5 > gpurun_out/rq_q9_ad_nopack.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gb_wscan" -s 2 -c 1 -o /tmp/r2ad_q9 -f python tools/run_query.py --sf 100 --reps 1 --warm 1 --query q9 > gpurun_out/r2ad_q9.log 2>&1
python tools/rep_summary.py /tmp/r2ad_q9.ncu-rep r2ad_q9 > gpurun_out/r2ad_q9_summary.txt 2>&1
