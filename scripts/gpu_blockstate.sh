mkdir -p gpurun_out/blk
timeout 300 python scripts/time_act_plans.py 2>&1 | tail -10
for c in c3s c5; do
  timeout 300 python bench.py --config $c --no-cpu > gpurun_out/blk/bench_$c.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/blk/bench_$c.json')); print('$c', d['value'], d['roofline']['frac'])"
done
