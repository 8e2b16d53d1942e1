set -x
timeout 900 python -m pytest tests/test_gpu_gmres.py -x -q > gpurun_out/pytest_pair.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pair.log
timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_pair.json 2> gpurun_out/bench_pair.err
MDD_ARN_PAIR=0 timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_nopair.json 2> /dev/null
