"""Per-launch table of one K3 solve from an ncu --csv launch list (tools/gpu_k3_launches.sh)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        e = data.setdefault(int(d["ID"]), {"name": d["Kernel Name"], "grid": d["Grid Size"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(data.values())


def main(path, skip=0):
    ls = load(path)
    # one solve = the launches between two consecutive first-level sweep kernels; take the (skip+1)-th solve
    starts = [i for i, e in enumerate(ls) if "sweep" in e["name"] and (i == 0 or "sweep" not in ls[i - 1]["name"]
                                                                         and "contact_fix" not in ls[i - 1]["name"])]
    starts = [i for i in range(len(ls)) if i == 0 or ls[i]["name"] != ls[i - 1]["name"] and False] or starts
    blk = ls[starts[skip]:starts[skip + 1]] if len(starts) > skip + 1 else ls
    tot = 0.0
    for e in blk:
        t = e.get("gpu__time_duration.sum", 0) / 1e3
        b = (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)) / 1e6
        tot += t
        print(f'{e["name"][:48]:48s} grid {e["grid"]:14s} {t:7.1f} us {b:8.2f} MB {b / max(t, 1e-9) * 1e-3:6.2f} TB/s')
    print(f"solve total {tot:.1f} us over {len(blk)} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
