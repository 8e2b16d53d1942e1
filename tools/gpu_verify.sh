set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_v.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err
