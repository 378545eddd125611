"""Markdown summary of an `ncu --set full` report (+ optional traffic json update).

    python scripts/ncu_summary.py REPORT.ncu-rep OUT.md "title" [kernel_key traffic.json]
"""
import csv
import io
import json
import subprocess
import sys

rep, out, title = sys.argv[1:4]
key = sys.argv[4] if len(sys.argv) > 4 else None
tj = sys.argv[5] if len(sys.argv) > 5 else None


def page(p, *extra):
    return subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(page("raw"))))
h, units, v = rows[0], rows[1], rows[2]
d = {h[i]: (v[i], units[i]) for i in range(len(h))}


def num(k):
    try:
        return float(d[k][0].replace(",", ""))
    except Exception:
        return None


def scaled(k, to="B"):
    x, u = num(k), d.get(k, ("", ""))[1]
    if x is None:
        return None
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
            "msecond": 1e-3, "second": 1.0}.get(u, 1.0)
    return x * mult


dur = scaled("gpu__time_duration.sum")
rd, wr = scaled("dram__bytes_read.sum"), scaled("dram__bytes_write.sum")
lines = [f"# {title}", "", f"Source: `{rep.split('/')[-1]}` (ncu --set full --clock-control none --import-source on; "
         "kernel replayed, cold caches: absolute time is not a bench number).", "",
         "| metric | value |", "|---|---|"]
for name, k in [("kernel", "Kernel Name"), ("grid", "launch__grid_size"), ("block", "launch__block_size"),
                ("registers/thread", "launch__registers_per_thread"),
                ("dyn. smem / block", "launch__shared_mem_per_block_dynamic")]:
    if k in d:
        lines.append(f"| {name} | {d[k][0]} {d[k][1]} |".replace(" | |", " |"))
lines.append(f"| duration | {d['gpu__time_duration.sum'][0]} {d['gpu__time_duration.sum'][1]} |")
if rd is not None:
    lines.append(f"| DRAM read + write | {rd / 1e6:.2f} + {wr / 1e6:.2f} MB |")
for name, k in [("DRAM throughput % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                ("L2 hit rate %", "lts__t_sector_hit_rate.pct"),
                ("SM issue slots busy %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
                ("achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
                ("warp-level instructions", "smsp__inst_executed.sum")]:
    if k in d:
        lines.append(f"| {name} | {d[k][0]} |")
st = [(k, num(k)) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
st = [(k, x) for k, x in st if x]
tot = sum(x for _, x in st) or 1
lines += ["", "Stall reasons (share of warp samples): " +
          ", ".join(f"{k[33:]} {x / tot * 100:.1f}%" for k, x in sorted(st, key=lambda y: -y[1])[:8]), ""]
src = list(csv.reader(io.StringIO(page("source", "--print-source", "cuda,sass"))))
cur, hdr, outl = None, None, []
for r in src:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")])
        ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except Exception:
        continue
    outl.append((ie, ss, cur, r[0], r[1].strip()[:90]))
ti = sum(o[0] for o in outl) or 1
ts = sum(o[1] for o in outl) or 1
lines += ["Hottest source lines (stall samples / executed instructions):", "", "| stall % | inst % | line | source |",
          "|---|---|---|---|"]
for o in sorted(outl, key=lambda x: -x[1])[:15]:
    lines.append(f"| {o[1] / ts * 100:.1f} | {o[0] / ti * 100:.1f} | {o[2]}:{o[3]} | `{o[4].replace('|', '/')}` |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:16]))
if key and tj and rd is not None:
    try:
        data = json.load(open(tj))
    except Exception:
        data = {}
    data[key] = rd + wr
    json.dump(data, open(tj, "w"), indent=1)
