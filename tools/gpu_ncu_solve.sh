export MDD_SOLVE=tma MDD_TSOLVE_K=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_tma --launch-skip 0 --launch-count 1 -o gpurun_out/prof_tfwd0 -f python tools/profile_onelevel.py > gpurun_out/prof_t.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_tma --launch-skip 17 --launch-count 1 -o gpurun_out/prof_tbwd0 -f python tools/profile_onelevel.py >> gpurun_out/prof_t.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_solve_tma --launch-count 18 --csv python tools/profile_onelevel.py > gpurun_out/tma_launches.csv 2>> gpurun_out/prof_t.log
