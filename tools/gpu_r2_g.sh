#!/bin/bash
mkdir -p gpurun_out
python tools/prof_arnoldi.py 3 120 > gpurun_out/r2g_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_arnoldi_wide -s 100 -c 1 \
    -o gpurun_out/r2g_prof_wide_cfg3 python tools/prof_arnoldi.py 3 120 > gpurun_out/r2g_ncu.log 2>&1
echo "rc=$?"; tail -n 3 gpurun_out/r2g_plain.log gpurun_out/r2g_ncu.log
