#!/bin/bash
# Every bench.py config once (1 GPU), one JSON line each -> gpurun_out/bench_all.jsonl
out=gpurun_out/bench_all.jsonl
: > $out
python bench.py >> $out 2>gpurun_out/bench_all.err
for c in c1 c1n c1log c1logn c3 c3s c1big; do
  python bench.py --config $c --steps 20 --warmup 5 >> $out 2>>gpurun_out/bench_all.err
done
python bench.py --config c4 --steps 5 --warmup 3 >> $out 2>>gpurun_out/bench_all.err
python bench.py --config c4ref --steps 5 --warmup 3 >> $out 2>>gpurun_out/bench_all.err
python bench.py --config c5 --steps 10 --warmup 3 >> $out 2>>gpurun_out/bench_all.err
python bench.py --impl reference --steps 3 --warmup 3 >> $out 2>>gpurun_out/bench_all.err
echo done
