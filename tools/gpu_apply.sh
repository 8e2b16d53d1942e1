rm -f gpurun_out/ta_sweep.json
for cfg in "2048 0" "2048 500" "2048 1000" "2048 2000" "2048 4000" "1536 1500" "3072 1000"; do
  set -- $cfg
  MDD_SOLVE=tma MDD_TSOLVE_ELEMS=$1 MDD_TSOLVE_PF=$2 timeout 300 python tools/time_apply.py >> gpurun_out/ta_sweep.json 2>> gpurun_out/ta_sweep.err
done
timeout 600 python -m pytest tests/test_gpu_precond.py -x -q > gpurun_out/gpu_tests.log 2>&1
