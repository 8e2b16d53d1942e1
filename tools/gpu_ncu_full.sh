# full ncu captures of the dominant kernels (each command exits 0 without ncu first in the bench run)
set -x
export CFG=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_tma --launch-skip 1 --launch-count 1 -o gpurun_out/prof_fwd_l1 -f python tools/profile_onelevel.py > gpurun_out/prof_solve.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_tma --launch-skip 16 --launch-count 1 -o gpurun_out/prof_bwd_l1 -f python tools/profile_onelevel.py >> gpurun_out/prof_solve.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_tma --launch-skip 17 --launch-count 1 -o gpurun_out/prof_bwd_l0 -f python tools/profile_onelevel.py >> gpurun_out/prof_solve.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm --launch-skip 13 --launch-count 1 -o gpurun_out/prof_gemm -f python tools/profile_factor.py > gpurun_out/prof_gemm.log 2>&1
