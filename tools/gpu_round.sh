# full check: gpu tests, smoke, default bench, reference arm, launch list with DRAM bytes
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
MDD_NO_GRAPH=1 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9200 --csv python bench.py --steps 1 --warmup 0 --no-cpu > gpurun_out/launches.csv 2> gpurun_out/launches.err
python tools/traffic_from_ncu.py gpurun_out/launches.csv cfg1 200 > gpurun_out/traffic_cfg1.json 2>&1
