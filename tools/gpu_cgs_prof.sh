# CGS2 Arnoldi on one GPU: bench breakdown + launch list of the projection kernels late in the solve
timeout 600 python bench.py --no-cpu --steps 2 --warmup 2 --ortho cgs2 > gpurun_out/cgs_bench.json 2> gpurun_out/cgs_bench.err
MDD_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_mdot|k_maxpy|k_colsum|k_cgs_tail|k_vscale" --launch-skip 1400 -c 40 --csv --log-file gpurun_out/cgs_launches.csv \
  python bench.py --no-cpu --steps 1 --warmup 0 --ortho cgs2 > gpurun_out/cgs_ncu.log 2>&1
python tools/ncu_table.py gpurun_out/cgs_launches.csv > gpurun_out/cgs_launches_table.txt
