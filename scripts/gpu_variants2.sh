# A/B of library builds (lib/var/*.so) with an environment per variant
mkdir -p gpurun_out/var
for r in $(seq ${REPS:-2}); do
for v in $VARS; do
  cp paper_1910_04540_b200/lib/var/$v.so paper_1910_04540_b200/lib/liblpq.so
  for c in $CONFIGS; do
    LPQ_PDL=${PDL:-1} timeout 300 python bench.py --config $c --no-cpu > gpurun_out/var/$v.$c.json 2>&1
    python -c "import json; d=json.load(open('gpurun_out/var/$v.$c.json')); print('$v', '$c', d['value'], d['roofline']['frac'])" 2>&1 | tail -1
  done
done; done
