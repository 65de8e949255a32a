# K10w occupancy variants (3 vs 4 CTAs/SM)
timeout 600 python -m pytest tests/test_gpu_tpch.py -x -q -p no:cacheprovider -k "q9" > gpurun_out/pytest_q9.log 2>&1; echo exit=$? >> gpurun_out/pytest_q9.log
SX_Q9_SCAN=wscan timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_wscan3.json 2> gpurun_out/bench_wscan3.err
sed -i 's/__launch_bounds__(kBlock, 3) k_gb_wscan(/__launch_bounds__(kBlock, 4) k_gb_wscan(/' paper_2508_04701_b200/csrc/groupby.cuh
make sx > gpurun_out/make4.log 2>&1
cuobjdump -res-usage paper_2508_04701_b200/libsx.so 2>/dev/null | grep -A1 "k_gb_wscan" | grep -o "REG:[0-9]* STACK:[0-9]* SHARED:[0-9]* LOCAL:[0-9]*" >> gpurun_out/make4.log
SX_Q9_SCAN=wscan timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_wscan4.json 2> gpurun_out/bench_wscan4.err
