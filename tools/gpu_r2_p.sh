#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2p_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2p_tests.log
grep -E "^FAILED|^ERROR|passed|failed|rc=" gpurun_out/r2p_tests.log | cut -c1-300 | tail -n 15
