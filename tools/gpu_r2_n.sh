#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_distributed.py -m gpu -q -x > gpurun_out/r2n_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2n_tests.log
tail -n 3 gpurun_out/r2n_tests.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu $ARGS > gpurun_out/r2n_${tag}.json 2> gpurun_out/r2n_${tag}.err; echo "$tag rc=$?"; }
ARGS="--config 4" run cfg4 X=1
ARGS="--config 4 --no-drift" run cfg4_nodrift X=1
ARGS="--config 3" run cfg3 X=1
ARGS="--config 3 --no-drift" run cfg3_nodrift X=1
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2n_cfg*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f,round(d["ms_per_step"],1),d["config"]["final_rel_residual"],round(d["phases_ms"]["gmres_arnoldi"],1),round(d["roofline_all"]["k_arnoldi"]["frac"],3))
    except Exception as e: print(f,"failed",e)
P
