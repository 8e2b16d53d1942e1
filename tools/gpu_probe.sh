# FP64 peaks + full-size runs of the larger BASELINE configs (one GPU)
set -x
mkdir -p /tmp/pb && nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o /tmp/pb/fp64_peak && /tmp/pb/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
python tools/fp64_cublas.py > gpurun_out/fp64_cublas.txt 2>&1
timeout 900 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
