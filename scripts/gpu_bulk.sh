LPQ_BULK=1 timeout 900 python -m pytest tests/test_gpu_quantize.py -m gpu -q -p no:cacheprovider -x -k "c2 or fixed or golden or elementwise or dependent" 2>&1 | tail -2
for r in 1 2; do for b in 0 1; do
  LPQ_BULK=$b timeout 300 python bench.py --config c2 --no-cpu --no-e2e > gpurun_out/bulk.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/bulk.json')); print('bulk=$b c2', d['value'], d['roofline']['frac'])"
done; done
