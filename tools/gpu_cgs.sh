timeout 600 python bench.py --no-cpu --steps 2 --warmup 2 --ortho cgs2 > gpurun_out/bench_cgs1.json 2> /dev/null
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu --ortho cgs2 > gpurun_out/bench_cgs4.json 2> /dev/null
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_mgs4.json 2> /dev/null
