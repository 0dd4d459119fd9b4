"""Summarise gpurun_out/devrun.log (one JSON line per tools/devrun.py run): per-family us per launch."""
import json
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/devrun.log"
for l in open(path):
    if not l.startswith("{"):
        print(l.strip()[:300])
        continue
    d = json.loads(l)
    p = d["prof_all"]
    per = {k: round(1e3 * v[0] / max(v[1], 1), 1) for k, v in p.items() if v[1]}
    print(d["config"], "T", d["T"], "fwd", d["fwd_s"], "bwd", d["bwd_s"], "dofsteps/s %.3g" % d["dof_steps_per_s"],
          "its", round(d["iters_fwd"]["mean"], 1), round(d["iters_adj"]["mean"], 1), "us/launch", per)
