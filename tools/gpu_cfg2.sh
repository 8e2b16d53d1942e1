# order-2 / non-nested parity tests, then the cfg2 bench line
set -x
timeout 900 python -m pytest tests/test_gpu_nedelec2.py -x -q > gpurun_out/pytest_n2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_n2.log
timeout 1200 python bench.py --config 2 --steps 2 --warmup 1 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
