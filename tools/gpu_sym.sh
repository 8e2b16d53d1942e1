set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_sym.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sym.log
timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_sym.json 2> gpurun_out/bench_sym.err
MDD_NO_SYM=1 timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_nosym.json 2> /dev/null
timeout 900 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench2_sym.json 2> /dev/null
