"""Per-source-line stall summary of an ncu report (needs -lineinfo builds and
--import-source on).  python tools/ncu_lines.py <report.ncu-rep> [kernel-substring] [top]"""
import csv
import io
import subprocess
import sys


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, fn, path, hdr = [], None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or ksub not in (fn or ""):
        continue
    n = len(hdr) - 2  # metric columns sit at the end (source text may contain unescaped quotes)
    d = dict(zip(hdr[2:], r[len(r) - n:]))
    res.append((path.split("/")[-1], r[0], ",".join(r[1:len(r) - n]), d))
tot = sum(num(d.get("Warp Stall Sampling (All Samples)")) for *_, d in res) or 1
toti = sum(num(d.get("Instructions Executed")) for *_, d in res) or 1
reasons = [h for h in (hdr or []) if h.startswith("stall_") and "Not Issued" not in h]
print(f"samples {tot:.0f}  warp-instructions {toti:.0f}")
for f, ln, src, d in sorted(res, key=lambda x: -num(x[3].get("Warp Stall Sampling (All Samples)")))[:top]:
    s = num(d.get("Warp Stall Sampling (All Samples)"))
    i = num(d.get("Instructions Executed"))
    rs = sorted(((num(d.get(k)), k[6:]) for k in reasons), reverse=True)[:3]
    rs = " ".join(f"{k}:{v / max(s, 1) * 100:.0f}%" for v, k in rs if v > 0)
    print(f"{f}:{ln:>5} {s / tot * 100:5.1f}% inst {i / toti * 100:5.1f}%  [{rs}]  {src.strip()[:70]}")
