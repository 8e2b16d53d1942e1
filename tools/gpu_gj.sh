# factorisation A/B: fused small-front GJ + CTA pivot-block inversion vs the warp sweep
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu3.log
MDD_NO_GJ_SMALL=1 MDD_INV_WARP=1 timeout 600 python bench.py --no-cpu > gpurun_out/bench_gj_old.json 2> gpurun_out/bench_gj_old.err
timeout 600 python bench.py --no-cpu > gpurun_out/bench_gj_new.json 2> gpurun_out/bench_gj_new.err
CFG=1 REFACTORS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/profile_factor.py > gpurun_out/factor_launches.csv 2> gpurun_out/factor.err
