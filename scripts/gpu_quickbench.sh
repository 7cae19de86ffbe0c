# a few bench configs (device value, no CPU leg), twice
for r in 1 2; do for c in ${CONFIGS:-c1 c1n c1log c1logn c5 c2}; do
  timeout 300 python bench.py --config $c --no-cpu > gpurun_out/qb.$c.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/qb.$c.json')); print('$c', d['value'], d['roofline']['frac'])" 2>&1 | tail -1
done; done
