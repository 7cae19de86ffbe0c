# per-kernel time of one C5 sweep (ncu launch list; cold, serialised -- shares only)
mkdir -p gpurun_out/c5
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c5/launches.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu --graph off > gpurun_out/c5/ncu.log 2>&1
tail -2 gpurun_out/c5/ncu.log
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/c5/launches.csv")))
hdr = None
data = collections.defaultdict(lambda: [0, 0.0, 0.0])
per = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if not hdr or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"][:70])
    per.setdefault(key, {})[d["Metric Name"]] = (d["Metric Unit"], float(d["Metric Value"].replace(",", "")))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (i, name), m in per.items():
    t = m.get("gpu__time_duration.sum", ("ns", 0))
    tus = t[1] * {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(t[0], 1e-3)
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        u, v = m.get(k, ("byte", 0))
        b += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    a = agg[name]; a[0] += 1; a[1] += tus; a[2] += b
tot = sum(a[1] for a in agg.values())
for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"{a[0]:5d} {a[1]/1e3:8.3f} ms {100*a[1]/tot:5.1f}% {a[2]/a[1]/1e3 if a[1] else 0:7.0f} GB/s  {name}")
print("total ms", tot / 1e3)
PY
