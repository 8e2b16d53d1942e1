set -x
timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_bs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bs.log
timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_bs.json 2> /dev/null
