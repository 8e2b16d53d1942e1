#!/bin/bash
# round-2 session B: the TMA-ring STREAM Arnoldi kernel: parity tests, then cfg3/cfg4 A/B against the old kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gmres.py -m gpu -x -q > gpurun_out/r2b_gmres_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_gmres_tests.log
tail -5 gpurun_out/r2b_gmres_tests.log
for cfg in 3 4; do
  timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu > gpurun_out/r2b_bench_cfg${cfg}_new.json 2> gpurun_out/r2b_bench_cfg${cfg}_new.err
  echo "new cfg$cfg rc=$?"
  MDD_ARN_STREAM=old timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu > gpurun_out/r2b_bench_cfg${cfg}_old.json 2> gpurun_out/r2b_bench_cfg${cfg}_old.err
  echo "old cfg$cfg rc=$?"
done
python - <<'P'
import json
for cfg in (3,4):
    for v in ("new","old"):
        try:
            d=json.loads(open(f"gpurun_out/r2b_bench_cfg{cfg}_{v}.json").read().strip().splitlines()[-1])
            print(cfg,v,round(d["ms_per_step"],1),d["config"]["iterations"],d["config"]["final_rel_residual"],{k:round(x,1) for k,x in d["phases_ms"].items() if k.startswith("gmres_") and "host" not in k},round(d["roofline_all"]["k_arnoldi"]["frac"],3))
        except Exception as e: print(cfg,v,"failed",e)
P
