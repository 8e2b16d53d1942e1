#!/bin/bash
# usage: gpu_r2_san.sh memcheck|racecheck|synccheck|initcheck
tool=$1
mkdir -p gpurun_out
timeout 300 python tools/sanitize_case.py > gpurun_out/r2_san_plain.log 2>&1 || { echo "plain run failed"; tail -n 5 gpurun_out/r2_san_plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 3 python tools/sanitize_case.py > gpurun_out/r2_san_$tool.log 2>&1
echo "$tool rc=$?"; tail -n 12 gpurun_out/r2_san_$tool.log | cut -c1-200
