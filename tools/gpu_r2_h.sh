#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gmres.py -m gpu -q -x > gpurun_out/r2h_gmres_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_gmres_tests.log
tail -n 3 gpurun_out/r2h_gmres_tests.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu $ARGS > gpurun_out/r2h_${tag}.json 2> gpurun_out/r2h_${tag}.err; echo "$tag rc=$?"; }
ARGS="--config 4 --no-drift" run cfg4_nodrift_pf24 X=1
ARGS="--config 4 --no-drift" run cfg4_nodrift_pf0 MDD_ARN_PF_MB=0
ARGS="--config 4 --no-drift" run cfg4_nodrift_pf56 MDD_ARN_PF_MB=60
ARGS="--config 4" run cfg4_pf24 X=1
ARGS="--config 3 --no-drift" run cfg3_nodrift_pf24 X=1
ARGS="--config 3 --no-drift" run cfg3_nodrift_pf0 MDD_ARN_PF_MB=0
ARGS="--config 3" run cfg3_pf24 X=1
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2h_cfg*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f,round(d["ms_per_step"],1),d["config"]["final_rel_residual"],round(d["phases_ms"]["gmres_arnoldi"],1),round(d["roofline_all"]["k_arnoldi"]["frac"],3))
    except Exception as e: print(f,"failed",e)
P
python tools/prof_arnoldi.py 4 120 > gpurun_out/r2h_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_arnoldi_wide -s 100 -c 1 \
    -o gpurun_out/r2h_prof_wide_cfg4 python tools/prof_arnoldi.py 4 120 > gpurun_out/r2h_ncu.log 2>&1
echo "ncu rc=$?"
