# launch list with DRAM bytes for one cfg1 bench step (host-driven GMRES loop), then per-family traffic
MDD_NO_GRAPH=1 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9200 --csv python bench.py --steps 1 --warmup 0 --no-cpu > gpurun_out/r01_launches_v2.csv 2> gpurun_out/r01_launches_v2.err
python tools/traffic_from_ncu.py gpurun_out/r01_launches_v2.csv cfg1 200 > gpurun_out/traffic_cfg1.json 2>&1
