# cfg3 / cfg4 on one GPU: MGS2 (default) vs CGS2 (row-tiled)
for c in 3 4; do for o in mgs cgs2; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu --ortho $o > gpurun_out/big_cfg${c}_${o}.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/big_cfg${c}_${o}.json')); p=d['phases_ms']; print('cfg$c $o', round(d['ms_per_step'],1), 'factor', round(p['factor'],1), 'gmres', round(p['gmres'],1), 'arnoldi', round(p['gmres_arnoldi'],1), 'iters', d['e2e'].get('iterations'))"
done; done
