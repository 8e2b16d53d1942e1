set -x
timeout 1500 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_configs.py tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_la.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_la.log
MDD_ARN_LA=0 timeout 600 python bench.py --no-cpu > gpurun_out/bench_la0.json 2> gpurun_out/bench_la0.err
timeout 600 python bench.py --no-cpu > gpurun_out/bench_la1.json 2> gpurun_out/bench_la1.err
MDD_ND_LEAF=96 timeout 600 python bench.py --no-cpu > gpurun_out/bench_leaf96.json 2> gpurun_out/bench_leaf96.err
MDD_ND_LEAF=128 timeout 600 python bench.py --no-cpu > gpurun_out/bench_leaf128.json 2> gpurun_out/bench_leaf128.err
MDD_ND_LEAF=40 timeout 600 python bench.py --no-cpu > gpurun_out/bench_leaf40.json 2> gpurun_out/bench_leaf40.err
