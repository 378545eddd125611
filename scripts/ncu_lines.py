"""Summarise an ncu report: stall mix and the hottest source lines (by stall samples and instructions)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
d = {h[i]: v[i] for i in range(len(h))}
print("duration", d.get("gpu__time_duration.sum"), "inst", d.get("smsp__inst_executed.sum"),
      "dram rd/wr", d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum"))
st = [(k, float(d[k].replace(",", ""))) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
tot = sum(x for _, x in st)
print("stalls:", ", ".join(f"{k[33:]} {x / tot * 100:.1f}%" for k, x in sorted(st, key=lambda x: -x[1])[:7]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
cur = None; out = []; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8 or r[0] == "": continue
    try:
        ie = int(r[hdr.index("Instructions Executed")]); ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except Exception:
        continue
    out.append((ie, ss, cur, int(r[0]), r[1][:95]))
ti = sum(o[0] for o in out) or 1; ts = sum(o[1] for o in out) or 1
print("-- by stall samples")
for o in sorted(out, key=lambda x: -x[1])[:n]:
    print(f"{o[1] / ts * 100:5.1f}% st {o[0] / ti * 100:5.1f}% in {o[2]}:{o[3]} {o[4]}")
