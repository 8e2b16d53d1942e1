set -x
timeout 1500 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_configs.py tests/test_gpu_precond.py -x -q > gpurun_out/pytest_pad.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pad.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_pad.json 2> gpurun_out/bench_pad.err
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 900 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
