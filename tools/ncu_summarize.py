"""Summarise ncu output for profiles/:

  python tools/ncu_summarize.py launches <launches.csv> <out.md>
      per-kernel share of one solve from the --metrics gpu__time_duration.sum pass
  python tools/ncu_summarize.py full <report.ncu-rep> <out.md> [--traffic-json profiles/ncu_traffic.json] [--workload NAME]
      key --set full metrics per captured launch; the DRAM bytes of the fused
      polynomial pass go to ncu_traffic.json (bench.py's roofline.traffic)
"""

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "cycles/issued inst"),
]


def _to_bytes(val, unit):
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1 << 20}
    return v * scale.get(unit, 1)


def _to_us(val, unit):
    v = float(val.replace(",", ""))
    return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
                "second": 1e6, "s": 1e6}.get(unit, 1)


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += _to_us(r[vi], r[ui])
        cnt[name] += 1
    T = sum(tot.values())
    lines = ["| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / T:.1f}% | {v / cnt[k]:.2f} |")
    lines.append(f"| **total** | {sum(cnt.values())} | {T:.1f} | 100% | |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, traffic_json=None, workload=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for key, label in KEYS:
            if key in h:
                i = h.index(key)
                rec[label] = f"{r[i]} {units[i]}".strip()
        if "dram__bytes_read.sum" in h:
            i, j = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
            rec["_dram_bytes"] = _to_bytes(r[i], units[i]) + _to_bytes(r[j], units[j])
        recs.append(rec)
    labels = ["kernel"] + [lab for _, lab in KEYS]
    lines = ["| " + " | ".join(labels) + " |", "|" + "---|" * len(labels)]
    for rec in recs:
        lines.append("| " + " | ".join(str(rec.get(lab, "")) for lab in labels) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json:
        poly = [r["_dram_bytes"] for r in recs
                if ("sell" in r["kernel"] or "plane_ring" in r["kernel"]) and "_dram_bytes" in r]
        data = {}
        try:
            data = json.load(open(traffic_json))
        except Exception:
            pass
        if poly:
            if workload:  # per-workload entry (bench.py reads its own config's)
                data.setdefault("per_workload", {})[workload] = {
                    "poly_pass_bytes_per_launch": sum(poly) / len(poly), "source": rep}
            else:
                data["poly_pass_bytes_per_launch"] = sum(poly) / len(poly)
                data["source"] = rep
        json.dump(data, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        wk = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else None
        full(sys.argv[2], sys.argv[3], tj, wk)
