for mr in 1 2 4 8; do
  MDD_TSOLVE_MINROWS=$mr CFG=1 REPS=20 timeout 300 python tools/time_apply.py >> gpurun_out/minrows.txt 2>/dev/null
  MDD_TSOLVE_MINROWS=$mr CFG=2 REPS=10 timeout 600 python tools/time_apply.py >> gpurun_out/minrows.txt 2>/dev/null
done
