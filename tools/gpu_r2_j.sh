#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/r2j_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2j_tests.log
grep -E "^\{|passed|failed|rc=" gpurun_out/r2j_tests.log | cut -c1-400 | tail -n 15
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2j_bench_cfg4.json 2> gpurun_out/r2j_bench_cfg4.err
echo "bench rc=$?"; tail -n 5 gpurun_out/r2j_bench_cfg4.err
