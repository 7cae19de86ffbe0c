mkdir -p gpurun_out/hash
timeout 1500 python -m pytest tests/test_gpu_quantize.py tests/test_gpu_fuzz.py tests/test_gpu_gemm.py tests/test_gpu_vs_reference_lib.py tests/test_gpu_sweep.py tests/test_gpu_composed.py tests/test_gpu_optim.py -m gpu -q -p no:cacheprovider -x > gpurun_out/hash/pytest.txt 2>&1; tail -3 gpurun_out/hash/pytest.txt
for c in c1 c1log c1n c2 c3 c5; do
  timeout 300 python bench.py --config $c --no-cpu > gpurun_out/hash/bench_$c.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/hash/bench_$c.json')); print('$c', d['value'], d['roofline']['frac'])"
done
timeout 600 python bench.py --config c4s --steps 3 --warmup 3 --no-cpu > gpurun_out/hash/bench_c4s.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/hash/bench_c4s.json')); print('c4s', d['value'], d['roofline']['frac'])"
