# solve-level L2 prefetch distance sweep (cfg1 bench, device ms per step)
for cfg in "" "MDD_TSOLVE_PF=250" "MDD_TSOLVE_PF=1000" "MDD_TSOLVE_PF=2000" "MDD_TSOLVE_PF=4000"; do
  r=$(env $cfg timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), round(d['phases_ms']['gmres_precond'],1))")
  echo "[$cfg] $r"
done
