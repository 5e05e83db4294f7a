"""Summarise ncu outputs for profiles/: a launch list CSV (--metrics ...) and
optional full captures (.ncu-rep).  Usage:

    python tools/ncu_summary.py <launches.csv> [<capture.ncu-rep> ...] > profiles/x.md
"""
import collections
import csv
import io
import subprocess
import sys


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per, names = collections.defaultdict(dict), {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per[r[idi]][r[mi]] = float(r[vi].replace(",", "") or 0)
        names[r[idi]] = r[ki]
    agg = collections.defaultdict(lambda: collections.Counter())
    for i, d in per.items():
        short = names[i].split("(")[0].replace("void mcfg::<unnamed>::", "")[:80]
        a = agg[short]
        a["launches"] += 1
        for k, v in d.items():
            a[k] += v
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    out = ["| kernel | launches | total us | share | avg us/launch | DRAM MB/launch | warp-instr/launch (M) |",
           "|---|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"])[:20]:
        n = a["launches"]
        t = a["gpu__time_duration.sum"]
        dram = (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / n / 1e6
        out.append(f"| `{k}` | {n} | {t/1e3:.1f} | {100*t/tot:.1f}% | {t/n/1e3:.1f} | {dram:.1f} | "
                   f"{a['smsp__inst_executed.sum']/n/1e6:.2f} |")
    return "\n".join(out)


WANT = ["Duration", "SM Frequency", "DRAM Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Issue Slots Busy", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "L2 Hit Rate", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "gpu__time_duration.sum"]


def capture_table(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    out = [f"### `{path.split('/')[-1]}`", ""]
    r = list(csv.reader(io.StringIO(det)))
    if not r:
        return "(empty capture)"
    h = r[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    seen = set()
    for row in r[1:]:
        key = (row[ii], row[mi])
        if row[mi] in WANT and key not in seen:
            seen.add(key)
            if len([s for s in seen if s[0] == row[ii]]) == 1:
                out.append(f"**{row[ki].split('(')[0].replace('void mcfg::<unnamed>::', '')}** (launch id {row[ii]})")
            out.append(f"- {row[mi]}: {row[vi]} {row[ui]}")
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hh = rr[0]
        for line in rr[2:]:
            out.append("- raw: " + ", ".join(f"{n}={line[hh.index(n)]}" for n in RAW if n in hh))
    stalls = []
    if len(rr) > 2:
        hh = rr[0]
        idx = [i for i, n in enumerate(hh) if "smsp__pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued")]
        vals = sorted(((float(rr[2][i].replace(",", "") or 0), hh[i].split("stalled_")[-1]) for i in idx), reverse=True)[:6]
        stalls = [f"{n} {int(v)}" for v, n in vals]
    out.append("- top stall samples: " + "; ".join(stalls))
    return "\n".join(out)


def main():
    print(launch_table(sys.argv[1]))
    for p in sys.argv[2:]:
        print()
        print(capture_table(p))


if __name__ == "__main__":
    main()
