mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quantize.py -q -p no:cacheprovider -x > gpurun_out/pytest_quick.txt 2>&1; echo pytest=$? >> gpurun_out/pytest_quick.txt
for c in ${CONFIGS:-c3s c1big c5}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']
print('$c', d['value'], d['unit'], 'ms', d['ms_per_step'], 'frac', r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['config'].get('launches_per_step'))" 2>&1 | tail -1
done
tail -2 gpurun_out/pytest_quick.txt
