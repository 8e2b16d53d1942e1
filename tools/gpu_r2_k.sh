#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_gmres.py -m gpu -q > gpurun_out/r2k_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2k_tests.log
grep -E "^FAILED|^ERROR|passed|failed|rc=" gpurun_out/r2k_tests.log | cut -c1-300 | tail -n 15
