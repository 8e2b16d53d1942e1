#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/r2l_bench_cfg4.json 2> gpurun_out/r2l_bench_cfg4.err
echo "bench rc=$?"; tail -n 4 gpurun_out/r2l_bench_cfg4.err
timeout 1200 python tools/rank_emulation.py --config 4 --ranks 1,2,4,8 --sample-ranks 2 --steps 1 > gpurun_out/r2l_rank_emulation_cfg4.log 2>&1
echo "emu rc=$?"; tail -n 12 gpurun_out/r2l_rank_emulation_cfg4.log | cut -c1-400
