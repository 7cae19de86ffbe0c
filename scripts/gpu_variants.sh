# A/B library variants (paper_1910_04540_b200/lib/var/*.so, built locally):
# each copied over lib/liblpq.so, then the listed bench configs (device value)
VARS=${VARS:-"0 A B"}
CONFIGS=${CONFIGS:-"c1 c1log c2"}
REPS=${REPS:-2}
mkdir -p gpurun_out/var
for r in $(seq $REPS); do
for v in $VARS; do
  cp paper_1910_04540_b200/lib/var/$v.so paper_1910_04540_b200/lib/liblpq.so
  for c in $CONFIGS; do
    timeout 300 python bench.py --config $c --no-cpu --steps ${STEPS:-20} --warmup 5 > gpurun_out/var/$v.$c.$r.json 2>&1
    python -c "import json; d=json.load(open('gpurun_out/var/$v.$c.$r.json')); print('$v', '$c', d['value'], d['roofline']['frac'], d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1
  done
done
done
