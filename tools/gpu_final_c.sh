# session-c final evidence: GPU suite, default bench line, ncu full capture of the tiled CGS2 pass
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final_pytest.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cgs_tile" --launch-skip 400 -c 1 \
  -o gpurun_out/r01c_prof_cgs_tile python bench.py --no-cpu --steps 1 --warmup 0 --ortho cgs2 > gpurun_out/final_ncu.log 2>&1; echo "ncu rc=$?"
