#!/bin/bash
# Every bench.py config once (1 GPU), one JSON line each -> gpurun_out/bench_all.jsonl
out=gpurun_out/bench_all.jsonl
: > $out
timeout 900 python bench.py >> $out 2>gpurun_out/bench_all.err
for c in c1 c1n c1log c1logn c3 c3s c1big; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 >> $out 2>>gpurun_out/bench_all.err
done
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 >> $out 2>>gpurun_out/bench_all.err
timeout 600 python bench.py --config c4raw --steps 5 --warmup 3 >> $out 2>>gpurun_out/bench_all.err
timeout 900 python bench.py --config c4s --steps 3 --warmup 3 >> $out 2>>gpurun_out/bench_all.err
timeout 600 python bench.py --config c4ref --steps 5 --warmup 3 >> $out 2>>gpurun_out/bench_all.err
timeout 600 python bench.py --config c5 --steps 10 --warmup 3 >> $out 2>>gpurun_out/bench_all.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 >> $out 2>>gpurun_out/bench_all.err
python - <<'PY'
import json
for l in open("gpurun_out/bench_all.jsonl"):
    try:
        d = json.loads(l)
    except Exception:
        continue
    r = d.get("roofline") or {}
    print(d.get("impl", "b200"), d["config"].get("workload", "")[:60], d["value"], d["unit"], r.get("frac"),
          (d.get("e2e") or {}).get("value"), (d.get("clocks") or {}).get("reasons"))
PY
echo done
