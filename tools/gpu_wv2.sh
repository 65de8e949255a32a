# K10w variants: (C=1, 4 CTAs/SM) and (C=3, 3 CTAs/SM)
G=paper_2508_04701_b200/csrc/groupby.cuh; T=paper_2508_04701_b200/csrc/tpch.cu
sed -i 's/__launch_bounds__(kBlock, 3) k_gb_wscan(/__launch_bounds__(kBlock, 4) k_gb_wscan(/' $G
sed -i 's/  static constexpr int kWChunks = 2;/  static constexpr int kWChunks = 1;/' $T
make sx > gpurun_out/make_wv2.log 2>&1
cuobjdump -res-usage paper_2508_04701_b200/libsx.so 2>/dev/null | grep -A1 "k_gb_wscan" | grep -o "REG:[0-9]* STACK:[0-9]* SHARED:[0-9]* LOCAL:[0-9]*" >> gpurun_out/make_wv2.log
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_wv3.json 2> gpurun_out/bench_wv3.err
sed -i 's/__launch_bounds__(kBlock, 4) k_gb_wscan(/__launch_bounds__(kBlock, 3) k_gb_wscan(/' $G
sed -i 's/  static constexpr int kWChunks = 1;/  static constexpr int kWChunks = 3;/' $T
make sx >> gpurun_out/make_wv2.log 2>&1
cuobjdump -res-usage paper_2508_04701_b200/libsx.so 2>/dev/null | grep -A1 "k_gb_wscan" | grep -o "REG:[0-9]* STACK:[0-9]* SHARED:[0-9]* LOCAL:[0-9]*" >> gpurun_out/make_wv2.log
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_wv4.json 2> gpurun_out/bench_wv4.err
