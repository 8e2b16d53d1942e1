# per-rank N=8 step time (rank 0, emulated collectives) under solve-task sizes and PDL
for cfg in "" "MDD_PDL=0" "MDD_TSOLVE_ELEMS=4096" "MDD_TSOLVE_ELEMS=2048" "MDD_TSOLVE_ELEMS=4096 MDD_SOLVE_MINB=8"; do
  r=$(env $cfg timeout 300 python tools/rank_emulation.py --ranks 8 --only-rank 5 --steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ranks']['8']['max_ms'],2))")
  echo "N8 rank5 [$cfg] $r ms"
done
for cfg in "" "MDD_TSOLVE_ELEMS=4096"; do
  r=$(env $cfg timeout 300 python tools/rank_emulation.py --ranks 1 --steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ranks']['1']['max_ms'],2))")
  echo "N1 cgs2 [$cfg] $r ms"
done
