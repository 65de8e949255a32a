# Q18 owned-run kernel occupancy variant (4 CTAs/SM) vs current
sed -i 's/__global__ void __launch_bounds__(kBlock) k_runs_own_dense(/__global__ void __launch_bounds__(kBlock, 4) k_runs_own_dense(/' paper_2508_04701_b200/csrc/gb_host.cuh
make sx > gpurun_out/make_q18.log 2>&1
cuobjdump -res-usage paper_2508_04701_b200/libsx.so 2>/dev/null | grep -A1 "k_runs_own_dense" | grep -o "REG:[0-9]* STACK:[0-9]* SHARED:[0-9]* LOCAL:[0-9]*" >> gpurun_out/make_q18.log
timeout 600 python -m pytest tests/test_gpu_tpch.py -x -q -p no:cacheprovider -k "q18 or vs_live" > gpurun_out/pytest_q18.log 2>&1; echo exit=$? >> gpurun_out/pytest_q18.log
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_q18b4.json 2> gpurun_out/bench_q18b4.err
