# 128-thread solve CTAs (MDD_SOLVE_THREADS=128) x task sizes, cfg1 bench and the N=8 rank
MDD_SOLVE_THREADS=128 MDD_TSOLVE_ELEMS=1024 timeout 600 python -m pytest tests/test_gpu_precond.py tests/test_gpu_gmres.py -x -q > gpurun_out/nt_pytest.log 2>&1; echo "pytest(128,1024) rc=$?"; tail -1 gpurun_out/nt_pytest.log
for cfg in "" "MDD_SOLVE_THREADS=128 MDD_TSOLVE_ELEMS=1024" "MDD_SOLVE_THREADS=128 MDD_TSOLVE_ELEMS=2048" "MDD_SOLVE_THREADS=128 MDD_TSOLVE_ELEMS=768"; do
  r=$(env $cfg timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), 'precond', round(d['phases_ms']['gmres_precond'],1))")
  echo "cfg1 [$cfg]: $r"
  r=$(env $cfg timeout 300 python tools/rank_emulation.py --ranks 8 --only-rank 5 --steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ranks']['8']['max_ms'],2))")
  echo "N8 rank5 [$cfg]: $r"
done
