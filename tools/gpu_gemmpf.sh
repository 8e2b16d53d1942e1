set -x
timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_nedelec2.py -x -q > gpurun_out/pytest_pf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pf.log
timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_pf.json 2> /dev/null
CFG=1 REFACTORS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_factor.py > gpurun_out/factor_launches3.csv 2> /dev/null
