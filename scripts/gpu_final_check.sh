mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest.txt 2>&1; tail -3 gpurun_out/final/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; cat gpurun_out/final/smoke.txt
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; cat gpurun_out/final/bench.json
for c in c1 c1n c1log c3 c5 c4 c4raw; do
  timeout 300 python bench.py --config $c --no-cpu > gpurun_out/final/bench_$c.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/final/bench_$c.json')); print('$c', d['value'], d['roofline']['frac'])"
done
timeout 600 python bench.py --config c4s --steps 3 --warmup 3 --no-cpu > gpurun_out/final/bench_c4s.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/final/bench_c4s.json')); print('c4s', d['value'], d['roofline']['frac'])"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_elementwise -s 3 -c 1 \
   -o gpurun_out/final/c1 python scripts/prof_kernel.py c1 24 5 > gpurun_out/final/ncu_c1.log 2>&1
ncu -i gpurun_out/final/c1.ncu-rep --page raw --csv > gpurun_out/final/c1.raw.csv 2>/dev/null
rm -f gpurun_out/final/c1.ncu-rep; tail -1 gpurun_out/final/ncu_c1.log
