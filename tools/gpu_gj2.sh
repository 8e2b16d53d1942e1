set -x
./tools/allgather_bench 20000 > gpurun_out/allgather.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_precond.py tests/test_gpu_configs.py tests/test_gpu_nedelec2.py -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu4.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_gj2.json 2> gpurun_out/bench_gj2.err
CFG=1 REFACTORS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_factor.py > gpurun_out/factor_launches2.csv 2> gpurun_out/factor2.err
