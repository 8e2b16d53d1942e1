for pf in 0 150 300 500 800 1500; do
  MDD_TSOLVE_PF=$pf CFG=1 REPS=20 timeout 300 python tools/time_apply.py >> gpurun_out/pf.txt 2>/dev/null
done
