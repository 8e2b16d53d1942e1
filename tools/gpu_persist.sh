# persistent level-synchronous solve (MDD_SOLVE_PERSIST=1/2) vs per-level launches
MDD_SOLVE_PERSIST=1 timeout 600 python -m pytest tests/test_gpu_precond.py tests/test_gpu_gmres.py tests/test_gpu_configs.py -x -q > gpurun_out/p_pytest.log 2>&1; echo "pytest(persist=1) rc=$?"; tail -2 gpurun_out/p_pytest.log
grep -E "^E" gpurun_out/p_pytest.log | head -4 | cut -c1-300
for P in 0 1 2; do
  r=$(MDD_SOLVE_PERSIST=$P timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), 'precond', round(d['phases_ms']['gmres_precond'],1))")
  echo "cfg1 persist=$P: $r"
  r=$(MDD_SOLVE_PERSIST=$P timeout 300 python tools/rank_emulation.py --ranks 8 --only-rank 5 --steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ranks']['8']['max_ms'],2))")
  echo "N8 rank5 persist=$P: $r"
done
