for cfg in "3072 32 64" "8192 16 64" "8192 32 64" "16384 16 64" "8192 16 48" "8192 16 96" "8192 16 128"; do
  set -- $cfg
  MDD_SOLVE_ELEMS=$1 MDD_SOLVE_QUANT=$2 MDD_ND_LEAF=$3 timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/sw_$1_$2_$3.json 2> gpurun_out/sw_$1_$2_$3.err
done
