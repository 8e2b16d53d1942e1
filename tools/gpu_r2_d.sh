#!/bin/bash
mkdir -p gpurun_out
python tools/prof_arnoldi.py 4 120 > gpurun_out/r2d_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_arnoldi_stream -s 100 -c 2 \
    -o gpurun_out/r2d_prof_stream python tools/prof_arnoldi.py 4 120 > gpurun_out/r2d_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/r2d_plain.log gpurun_out/r2d_ncu.log
