set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_sym3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sym3.log
timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_sym3.json 2> gpurun_out/bench_sym3.err
MDD_NO_SYM=1 timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_nosym3.json 2> /dev/null
