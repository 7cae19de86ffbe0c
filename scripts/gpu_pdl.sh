mkdir -p gpurun_out/pdl
for r in 1 2; do for p in 0 1; do
  for c in c1 c1n c2 c5; do
    LPQ_PDL=$p timeout 300 python bench.py --config $c --no-cpu > gpurun_out/pdl/$c.$p.json 2>&1
    python -c "import json; d=json.load(open('gpurun_out/pdl/$c.$p.json')); print('pdl=$p', '$c', d['value'], d['roofline']['frac'])" 2>&1 | tail -1
  done
done; done
LPQ_PDL=1 timeout 600 python -m pytest tests/test_gpu_quantize.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
