for v in lb256_4 lb256_6 lb256_8; do
  MDD_LIB_PATH=probe_bin/libmdd_$v.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/swl_$v.json 2> gpurun_out/swl_$v.err
done
