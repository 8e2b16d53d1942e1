#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_reference_suite.py tests/test_gpu_precond.py -m gpu -q -s > gpurun_out/r2m_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2m_tests.log
grep -E "^FAILED|^ERROR|passed|failed|skipped|rc=|SKIPPED" gpurun_out/r2m_tests.log | cut -c1-300 | tail -n 60
