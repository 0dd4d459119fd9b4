#!/usr/bin/env python
"""Per-launch DRAM traffic of the roofline kernels from ncu launch lists (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum), merged into profiles/ncu_traffic.json for bench.py's `traffic`:

    python tools/ncu_traffic.py <config> <launches.csv> [out.json]

solve_K3_dram_bytes = the bytes of the first complete A^{-1} application in the list (k_to_solve ... k_from_solve:
every level and reduce launch of both sweeps); local_K1_dram_bytes / AN_K4_dram_bytes = mean over the list's
k_elem_residual / k_elem_AN_cached launches.  ncu replays each kernel with cold caches, so these are upper bounds
of the live traffic (L2-resident right-hand sides and partial rows are counted as DRAM here).
"""
import collections
import csv
import json
import os
import sys


def launches(path):
    hdr, recs = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        m = recs.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})
        v = d["Metric Value"].replace(",", "")
        m[d["Metric Name"]] = float(v) if v not in ("", "n/a") else 0.0
    return list(recs.values())


def main():
    cfg, path = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                              "profiles", "ncu_traffic.json")
    L = launches(path)
    by = lambda m: m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    res = {}
    start = next((i for i, m in enumerate(L) if "k_to_solve" in m["name"]), None)
    if start is not None:
        end = next((i for i in range(start, len(L)) if "k_from_solve" in L[i]["name"]), None)
        if end is not None:
            res["solve_K3_dram_bytes"] = sum(by(m) for m in L[start:end + 1])
            res["solve_K3_launches"] = end - start + 1
    for fam, kn in (("local_K1", "k_elem_residual"), ("AN_K4", "k_elem_AN_cached")):
        v = [by(m) for m in L if kn + "(" in m["name"] or kn + "<" in m["name"] or m["name"].endswith(kn)]
        if v:
            res[fam + "_dram_bytes"] = sum(v) / len(v)
    res["source"] = os.path.basename(path)
    allj = {}
    if os.path.exists(out):
        allj = json.load(open(out))
    allj[cfg] = res
    json.dump(allj, open(out, "w"), indent=1)
    print(cfg, res)


if __name__ == "__main__":
    main()
