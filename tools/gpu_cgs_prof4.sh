timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_distributed.py -x -q > gpurun_out/c4_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/c4_pytest.log
for S in 2 3; do
MDD_CGS_STAGES=$S timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 --ortho cgs2 > gpurun_out/c4_bench_cgs_s$S.json 2> gpurun_out/c4_bench_cgs_s$S.err
done
timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/c4_bench_mgs.json 2> gpurun_out/c4_bench_mgs.err
MDD_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_cgs|k_colsum|k_vscale|k_mdot|k_maxpy" --launch-skip 1400 -c 16 --csv --log-file gpurun_out/c4_launches.csv \
  python bench.py --no-cpu --steps 1 --warmup 0 --ortho cgs2 > gpurun_out/c4_ncu.log 2>&1
python tools/ncu_table.py gpurun_out/c4_launches.csv > gpurun_out/c4_launches_table.txt
