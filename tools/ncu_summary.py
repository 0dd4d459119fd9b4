"""Condense ncu outputs into profiles/: launch-list shares (CSV from --metrics gpu__time_duration.sum ...) and
the key metrics of --set full captures (.ncu-rep).  Usage:
    python tools/ncu_summary.py launches <launches.csv> > profiles/xxx.md
    python tools/ncu_summary.py full <report.ncu-rep> > profiles/yyy.md
    python tools/ncu_summary.py seq <launches.csv> [first_id] [count]   (per-launch sequence, K3 level analysis)
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, recs = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"].split("(")[0].replace("void ", ""))
        v = d["Metric Value"].replace(",", "")
        recs.setdefault(key, {})[d["Metric Name"]] = float(v) if v not in ("", "n/a") else 0.0
    tot = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for (i, n), m in recs.items():
        t = m.get("gpu__time_duration.sum", 0.0) / 1e3
        by = (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / 1e6
        tot[n][0] += t
        tot[n][1] += 1
        tot[n][2] += by
    T = sum(v[0] for v in tot.values())
    print(f"# ncu launch list: {path}\n\n{len(recs)} launches, {T / 1e3:.2f} ms total (cold cache, serialised: compare shares)\n")
    print("| kernel | total ms | share | launches | avg us | DRAM MB/launch | DRAM GB/s |")
    print("|---|---|---|---|---|---|---|")
    for n, v in sorted(tot.items(), key=lambda x: -x[1][0]):
        avg = v[0] / v[1]
        mb = v[2] / v[1]
        print(f"| {n} | {v[0] / 1e3:.3f} | {100 * v[0] / T:.1f}% | {v[1]} | {avg:.1f} | {mb:.2f} | {mb / avg * 1e3 if avg else 0:.0f} |")


def seq(path, first=0, count=200):
    rows = list(csv.reader(open(path)))
    hdr, recs = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = int(d["ID"])
        m = recs.setdefault(key, {"name": d["Kernel Name"].split("(")[0].replace("void ", ""), "grid": d.get("Grid Size", "")})
        v = d["Metric Value"].replace(",", "")
        m[d["Metric Name"]] = float(v) if v not in ("", "n/a") else 0.0
    print("| id | kernel | grid | us | DRAM MB | GB/s |")
    print("|---|---|---|---|---|---|")
    for i, (k, m) in enumerate(recs.items()):
        if i < first or i >= first + count:
            continue
        t = m.get("gpu__time_duration.sum", 0.0) / 1e3
        by = (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / 1e6
        print(f"| {k} | {m['name'][:40]} | {m['grid']} | {t:.1f} | {by:.2f} | {by / t * 1e3 if t else 0:.0f} |")


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = r[0]
    per = collections.OrderedDict()
    for row in r[1:]:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") in WANT:
            per.setdefault((d["ID"], d["Kernel Name"].split("(")[0]), {})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    print(f"# ncu --set full: {path}\n")
    for i, ((kid, name), m) in enumerate(per.items()):
        print(f"## launch {kid}: `{name}`\n")
        for k in WANT:
            if k in m:
                print(f"- {k}: {m[k][0]} {m[k][1]}")
        if len(rr) > 2 + i:
            h, vals = rr[0], rr[2 + i]
            dv = {a: b for a, b in zip(h, vals)}
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                      "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"):
                if k in dv:
                    print(f"- {k}: {dv[k]}")
            st = [(a.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(b))
                  for a, b in dv.items() if "smsp__average_warps_issue_stalled" in a and a.endswith("per_issue_active.ratio")
                  and b not in ("", "n/a")]
            st.sort(key=lambda x: -x[1])
            print("- top stalls (cycles per issue): " + ", ".join(f"{a} {b:.2f}" for a, b in st[:6]))
        print()


if __name__ == "__main__":
    if sys.argv[1] == "seq":
        seq(sys.argv[2], *[int(a) for a in sys.argv[3:5]])
    else:
        {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
