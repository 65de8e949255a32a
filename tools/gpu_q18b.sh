timeout 900 python -m pytest tests/test_gpu_tpch.py tests/test_gpu_ops.py -x -q -p no:cacheprovider > gpurun_out/pytest_q18b.log 2>&1; echo exit=$? >> gpurun_out/pytest_q18b.log
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_q18c.json 2> gpurun_out/bench_q18c.err
