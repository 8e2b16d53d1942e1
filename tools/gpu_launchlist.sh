# launch list (time + DRAM bytes) of one bench step with a host-driven GMRES loop, then per-family traffic
set -x
timeout 900 python bench.py --no-cpu > gpurun_out/bench_ll.json 2> gpurun_out/bench_ll.err
MDD_NO_GRAPH=1 timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 11000 --csv python bench.py --steps 1 --warmup 0 --no-cpu > gpurun_out/launches_final.csv 2> gpurun_out/launches_final.err
python tools/traffic_from_ncu.py gpurun_out/launches_final.csv cfg1 200 gpurun_out/traffic_new.json > gpurun_out/traffic_final.log 2>&1
