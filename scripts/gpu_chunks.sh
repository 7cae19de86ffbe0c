for r in 1 2; do for mc in 4 8 16 32; do
  for c in c1 c3; do
    LPQ_MIN_CHUNKS=$mc timeout 300 python bench.py --config $c --no-cpu --e2e-steps 5 > gpurun_out/mc.json 2>&1
    python -c "import json; d=json.load(open('gpurun_out/mc.json')); print('mc=$mc', '$c', 'e2e', d['e2e']['value'], 'ceil', d['e2e'].get('pcie_copy_ceiling'))"
  done
done; done
