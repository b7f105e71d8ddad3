"""Instructions and stall samples aggregated per source line (first kernel of the report).
python tools/ncu_srclines.py <report.ncu-rep> [top]"""
import csv, io, subprocess, collections, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
def num(x):
    try: return float(x)
    except (TypeError, ValueError): return 0.0
fn = path = hdr = None
nfn = 0
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
for r in rows:
    if not r: continue
    if r[0] == "File Path": path = r[1]; continue
    if r[0] == "Function Name": fn = r[1]; nfn += 1; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    n = len(hdr) - 2
    d = dict(zip(hdr[2:], r[len(r) - n:]))
    key = ((path or "?").split("/")[-1], r[0])
    a = agg[key]
    a[0] += num(d.get("Instructions Executed")); a[1] += num(d.get("Warp Stall Sampling (All Samples)"))
    src = ",".join(r[1:len(r) - n]).strip()
    if src and not a[2]: a[2] = src[:90]
ti = sum(a[0] for a in agg.values()) or 1; ts = sum(a[1] for a in agg.values()) or 1
print(fn); print("warp-instructions", ti, "samples", ts)
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:>5} inst {100*a[0]/ti:5.1f}% stall {100*a[1]/ts:5.1f}%  {a[2]}")
