# gpu tests with PDL solve + native decomposition; A/B bench of PDL on cfg1
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu2.log
MDD_PDL=0 timeout 600 python bench.py --no-cpu > gpurun_out/bench_nopdl.json 2> gpurun_out/bench_nopdl.err
timeout 600 python bench.py --no-cpu > gpurun_out/bench_pdl.json 2> gpurun_out/bench_pdl.err
