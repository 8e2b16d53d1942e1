set -x
timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_cgs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cgs.log
timeout 600 python bench.py --no-cpu --steps 2 --warmup 2 --ortho cgs2 > gpurun_out/bench_cgs1b.json 2> /dev/null
