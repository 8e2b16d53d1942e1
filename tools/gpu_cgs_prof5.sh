timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_distributed.py -x -q > gpurun_out/c11_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/c11_pytest.log
timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 --ortho cgs2 > gpurun_out/c11_bench_cgs.json 2> /dev/null
python -c "import json; d=json.load(open('gpurun_out/c11_bench_cgs.json')); print('cgs2 ms/step', d['ms_per_step'], d['ms_steps'])"
timeout 300 python tools/rank_emulation.py --ranks 8 --only-rank 5 --steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N8 rank5', round(d['ranks']['8']['max_ms'],2))"
MDD_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_cgs|k_colsum|k_vscale" --launch-skip 1400 -c 16 --csv --log-file gpurun_out/c11_launches.csv \
  python bench.py --no-cpu --steps 1 --warmup 0 --ortho cgs2 > gpurun_out/c11_ncu.log 2>&1
python tools/ncu_table.py gpurun_out/c11_launches.csv > gpurun_out/c11_launches_table.txt; head -9 gpurun_out/c11_launches_table.txt
