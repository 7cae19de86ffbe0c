for r in 1 2; do for nt in 0 1; do
  echo "== LPQ_DEC_NT=$nt"; LPQ_DEC_NT=$nt timeout 600 python scripts/pcie_e2e_probe.py 2>&1 | grep "e2e call"
  LPQ_DEC_NT=$nt timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench e2e', d['e2e']['value'], 'ceiling', d['e2e']['pcie_copy_ceiling'])"
done; done
timeout 900 python -m pytest tests/test_gpu_quantize.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -x -k "host or c2_full" 2>&1 | tail -2
