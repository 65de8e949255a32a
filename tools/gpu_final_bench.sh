timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --sf 10 --no-e2e --no-cpu > gpurun_out/bench_sf10.json 2> gpurun_out/bench_sf10.err
timeout 600 python bench.py --sf 0.01 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_sf001.json 2> gpurun_out/bench_sf001.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
