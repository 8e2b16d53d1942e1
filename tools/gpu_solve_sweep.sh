# solve-kernel occupancy / task-size sweep on cfg1 (device-timed applies)
for minb in 0 6 8; do for el in 1024 2048 3072; do
  MDD_SOLVE_MINB=$minb MDD_TSOLVE_ELEMS=$el REPS=20 timeout 300 python tools/time_apply.py >> gpurun_out/solve_sweep.txt 2>/dev/null
done; done
