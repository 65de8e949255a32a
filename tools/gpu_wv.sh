# K10w variants: (U=1, 4 CTAs/SM, C=2) and (U=1, 3 CTAs/SM, C=4)
G=paper_2508_04701_b200/csrc/groupby.cuh; T=paper_2508_04701_b200/csrc/tpch.cu
sed -i 's/__launch_bounds__(kBlock, 3) k_gb_wscan(/__launch_bounds__(kBlock, 4) k_gb_wscan(/' $G
sed -i 's/  static constexpr int kWRows = 2;/  static constexpr int kWRows = 1;/' $T
make sx > gpurun_out/make_wv.log 2>&1
cuobjdump -res-usage paper_2508_04701_b200/libsx.so 2>/dev/null | grep -A1 "k_gb_wscan" | grep -o "REG:[0-9]* STACK:[0-9]* SHARED:[0-9]* LOCAL:[0-9]*" >> gpurun_out/make_wv.log
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_wv1.json 2> gpurun_out/bench_wv1.err
sed -i 's/__launch_bounds__(kBlock, 4) k_gb_wscan(/__launch_bounds__(kBlock, 3) k_gb_wscan(/' $G
sed -i 's/  static constexpr int kWChunks = 2;/  static constexpr int kWChunks = 4;/' $T
make sx >> gpurun_out/make_wv.log 2>&1
cuobjdump -res-usage paper_2508_04701_b200/libsx.so 2>/dev/null | grep -A1 "k_gb_wscan" | grep -o "REG:[0-9]* STACK:[0-9]* SHARED:[0-9]* LOCAL:[0-9]*" >> gpurun_out/make_wv.log
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_wv2.json 2> gpurun_out/bench_wv2.err
