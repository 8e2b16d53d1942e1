rm -f gpurun_out/spmv.json
for v in "0 0" "0 4" "0 2" "1 8" "1 4" "1 2"; do set -- $v; MDD_SPMV=$1 MDD_SPMV_TPR=$2 timeout 200 python tools/time_spmv.py >> gpurun_out/spmv.json 2>>gpurun_out/spmv.err; done
