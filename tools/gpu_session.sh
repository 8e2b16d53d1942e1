#!/bin/bash
# The gpurun recipes of this repo in one place (B200_PROFILING.md rules: ncu only after the same
# command exited 0 without it; one ncu tool per call).  Usage, from the repo root:
#   gpurun --timeout 3000 -- 'bash tools/gpu_session.sh check'        GPU suite, smoke, default bench, reference arm
#   gpurun --timeout 3600 -- 'bash tools/gpu_session.sh launchlist 4' ncu launch list (time + DRAM bytes) of one cfgN bench step
#   gpurun --timeout 1800 -- 'bash tools/gpu_session.sh arnoldi 4'    ncu --set full of the Arnoldi kernel at cfgN, m ~ 101
#   gpurun --timeout 1800 -- 'bash tools/gpu_session.sh emulate 4'    per-rank timing against tools/nccl_stub
#   gpurun --timeout 2000 -- 'bash tools/gpu_session.sh sanitize memcheck'
mkdir -p gpurun_out
what=$1; cfg=${2:-4}
case "$what" in
check)
  timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/pytest_gpu.log
  tail -n 3 gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/smoke.log
  timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "reference arm rc=$?"
  timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  ;;
launchlist)
  export MDD_NO_GRAPH=1   # kernels inside the conditional graph node are invisible to ncu
  timeout 900 python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu > gpurun_out/ll_plain.json 2> gpurun_out/ll_plain.err &&
  timeout 3000 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -c ${3:-40000} --csv --log-file gpurun_out/launches_cfg$cfg.csv python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu \
      > gpurun_out/ll_ncu.json 2> gpurun_out/ll_ncu.err
  echo "ncu rc=$?"
  python tools/launch_shares.py gpurun_out/launches_cfg$cfg.csv > gpurun_out/launches_cfg${cfg}_summary.md 2>&1
  cat gpurun_out/launches_cfg${cfg}_summary.md
  ;;
arnoldi)
  python tools/prof_arnoldi.py $cfg 120 > gpurun_out/arn_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_arnoldi -s 100 -c 1 \
      -o gpurun_out/prof_arnoldi_cfg$cfg -f python tools/prof_arnoldi.py $cfg 120 > gpurun_out/arn_ncu.log 2>&1
  echo "ncu rc=$?"; tail -n 2 gpurun_out/arn_plain.log gpurun_out/arn_ncu.log
  ;;
applyncu)
  # ncu --set full of the preconditioner-apply kernels (k_solve_tma levels, k_level_gather, k_scatter_owner) of one apply at cfgN
  # (cfg1 by default: at cfg4 ncu cannot save/restore the 46 GB of factors per pass)
  CFG=$cfg APPLIES=2 timeout 600 python tools/profile_apply.py > gpurun_out/apply_plain.log 2>&1 || { echo "plain run failed"; tail -n 5 gpurun_out/apply_plain.log; exit 1; }
  CFG=$cfg APPLIES=2 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_solve_tma|k_level_gather|k_scatter_owner' -c ${3:-60} \
      -o gpurun_out/prof_apply_cfg$cfg -f python tools/profile_apply.py > gpurun_out/apply_ncu.log 2>&1
  echo "ncu rc=$?"; tail -n 2 gpurun_out/apply_plain.log gpurun_out/apply_ncu.log | cut -c1-300
  ncu -i gpurun_out/prof_apply_cfg$cfg.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__average_warp_latency_issue_stalled_long_scoreboard.pct,smsp__average_warp_latency_issue_stalled_barrier.pct > gpurun_out/prof_apply_cfg${cfg}_raw.csv 2>&1
  ;;
emulate)
  timeout 1500 python tools/rank_emulation.py --config $cfg --ranks 1,2,4,8 --sample-ranks 2 --steps 1 > gpurun_out/rank_emulation_cfg$cfg.log 2>&1
  echo "rc=$?"; tail -n 12 gpurun_out/rank_emulation_cfg$cfg.log | cut -c1-300
  ;;
sanitize)
  # compute-sanitizer, one tool per call (memcheck | racecheck | synccheck | initcheck); closed on this pool in round 2
  tool=${2:-memcheck}
  timeout 300 python tools/sanitize_case.py > gpurun_out/san_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 3 python tools/sanitize_case.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -n 12 gpurun_out/san_$tool.log | cut -c1-200
  ;;
tmem)
  # the w tail of the wide Arnoldi kernel in tensor memory vs in L2: forced-path tests, then A/B bench lines
  timeout 900 python -m pytest tests/test_gpu_gmres.py -m gpu -q -x > gpurun_out/pytest_tmem.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_tmem.log
  timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_tmem_on.json 2> gpurun_out/bench_tmem_on.err; echo "tmem on rc=$?"
  MDD_ARN_TMEM=0 timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_tmem_off.json 2> gpurun_out/bench_tmem_off.err; echo "tmem off rc=$?"
  python - <<'PY'
import json
for f in ("on", "off"):
    try:
        d = json.loads(open(f"gpurun_out/bench_tmem_{f}.json").read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], {k: round(v, 1) for k, v in d["phases_ms"].items() if k.startswith("gmres_")})
    except Exception as e:
        print(f, "failed", e)
PY
  ;;
quick)
  # parity tests of the solve path and the config goldens, then one short bench line (no CPU leg)
  timeout 1200 python -m pytest tests/test_gpu_precond.py tests/test_gpu_config_goldens.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_quick.log
  timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
  python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], {k: round(v, 1) for k, v in d["phases_ms"].items()})
print({k: (round(v["frac"], 3), round(v["ms_per_launch"], 3)) for k, v in d["roofline_all"].items()})
PY
  ;;
arnsweep)
  # experiment knobs of the wide Arnoldi kernel, one short bench line each ("VAR=val" strings in $3..)
  shift 2
  for v in "" "$@"; do
    tag=$(echo "${v:-base}" | tr ' =' '__')
    env $v timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_arn_$tag.json 2> gpurun_out/bench_arn_$tag.err
    python - "$tag" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/bench_arn_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["ms_per_step"], 1), "arnoldi", round(d["phases_ms"]["gmres_arnoldi"], 1), "precond", round(d["phases_ms"]["gmres_precond"], 1), "final", d.get("final_rel_residual"))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
  ;;
*) echo "unknown recipe $what"; exit 2;;
esac
