#!/bin/bash
# round-2 session A: config goldens (cfg1), the full GPU suite, the cfg4 bench line with the real CPU leg
mkdir -p gpurun_out
nproc > gpurun_out/r2a_host.txt; free -g >> gpurun_out/r2a_host.txt
python -m pytest tests/test_gpu_config_goldens.py -m gpu -x -q -s > gpurun_out/r2a_goldens.log 2>&1
echo "goldens rc=$?" >> gpurun_out/r2a_goldens.log
python bench.py --steps 3 --warmup 3 > gpurun_out/r2a_bench_cfg4.json 2> gpurun_out/r2a_bench_cfg4.err
echo "bench rc=$?" >> gpurun_out/r2a_bench_cfg4.err
python -m pytest tests -m gpu -x -q > gpurun_out/r2a_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2a_tests.log
tail -3 gpurun_out/r2a_goldens.log gpurun_out/r2a_tests.log gpurun_out/r2a_bench_cfg4.err
