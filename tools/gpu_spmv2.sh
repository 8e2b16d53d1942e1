timeout 600 python -m pytest tests/test_gpu_core.py -x -q > gpurun_out/pytest_spmv.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spmv.log
for v in 0 1 2 3; do
MDD_SPMV_VAR=$v timeout 600 python bench.py --no-cpu --steps 2 --warmup 2 > gpurun_out/bench_spmv$v.json 2> /dev/null
MDD_SPMV_VAR=$v MDD_SPMV_VAR=$v timeout 300 python tools/time_spmv.py >> gpurun_out/spmv_var.txt 2>&1
done
