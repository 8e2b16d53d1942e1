timeout 600 python -m pytest tests/test_gpu_gmres.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
