"""Key metrics of ncu --set full captures exported with `--page raw --csv`.

    python scripts/ncu_summary.py profiles/r02_*.raw.csv
"""
import csv
import sys

KEYS = [("dur_us", "gpu__time_duration.sum", 1e-3),
        ("dram_rd_MB", "dram__bytes_read.sum", None),
        ("dram_wr_MB", "dram__bytes_write.sum", None),
        ("sm_active_cyc", "sm__cycles_active.avg", 1),
        ("sm_elapsed_cyc", "sm__cycles_elapsed.avg", 1),
        ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
        ("warp_inst", "smsp__inst_executed.sum", 1),
        ("regs", "launch__registers_per_thread", 1),
        ("occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
        ("l2_hit_pct", "lts__t_sector_hit_rate.pct", 1),
        ("fma_pipe_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
        ("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
        ("grid", "Grid Size", None), ("block", "Block Size", None)]

UNIT_TO_MB = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}
UNIT_TO_US = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def summarize(path):
    rows = list(csv.reader(open(path)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        rec = {"kernel": d.get("Kernel Name", "")[:60]}
        for name, key, _ in KEYS:
            v = d.get(key)
            if v is None:
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                rec[name] = v
                continue
            if name.startswith("dram"):
                x *= UNIT_TO_MB.get(u.get(key, "byte"), 1e-6)
            if name == "dur_us":
                x *= UNIT_TO_US.get(u.get(key, "nsecond"), 1e-3)
            rec[name] = round(x, 3)
        if "sm_active_cyc" in rec and "sm_elapsed_cyc" in rec and rec["sm_elapsed_cyc"]:
            rec["sm_active_frac"] = round(rec["sm_active_cyc"] / rec["sm_elapsed_cyc"], 3)
        out.append(rec)
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for rec in summarize(p):
            print(p.split("/")[-1], rec)
