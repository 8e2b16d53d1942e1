set -x
timeout 900 python -m pytest tests/test_gpu_gmres.py -x -q > gpurun_out/pytest_wg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_wg.log
for wg in 0 1; do
MDD_ARN_WG=$wg timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_wg$wg.json 2> /dev/null
MDD_ARN_WG=$wg timeout 900 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench3_wg$wg.json 2> /dev/null
done
