"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed).

  python tools/profile_summary.py launches <launches.csv> <out.md>
  python tools/profile_summary.py kernel <report.ncu-rep> <out.md>
"""
import collections
import csv
import io
import subprocess
import sys


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg, tot = collections.OrderedDict(), 0.0
    for r in data:
        if len(r) <= iV:
            continue
        name = r[iK].split("(")[0].replace("void ", "").replace("ab2::<unnamed>::", "")
        v = float(r[iV].replace(",", ""))
        u = r[iU]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)  # -> us
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    out = [f"# ncu launch list summary ({src})", "",
           "`ncu --metrics gpu__time_duration.sum --clock-control none` over the bench command;",
           "per-launch times are cold-cache and serialised: compare SHARES, not absolutes.", "",
           f"launches: {len(data)}, total {tot / 1e3:.3f} ms", "",
           "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {n} | {us / 1e3:.3f} | {100 * us / tot:.1f}% |")
    open(dst, "w").write("\n".join(out) + "\n")


def kernel(rep, dst):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    want = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
            "smsp__inst_executed.avg.per_cycle_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active"]
    cols = [h for h in want if h in hdr]
    out = [f"# ncu --set full summary ({rep})", "", "| " + " | ".join(cols) + " |",
           "|" + "---|" * len(cols), "| " + " | ".join(units[hdr.index(c)] for c in cols) + " |"]
    for r in data:
        out.append("| " + " | ".join(r[hdr.index(c)][:60] for c in cols) + " |")
    open(dst, "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    {"launches": launches, "kernel": kernel}[sys.argv[1]](sys.argv[2], sys.argv[3])
