# quick GPU loop: parity subset, timing probes, c5 launch list (ns units)
timeout 400 python -m pytest tests -m gpu -q -x -k "global_solve or c3s or c5s or c2s or c1" 2>&1 | tail -4
rm -f gpurun_out/devrun.log
for a in "c3 --horizon 3 --set accel_fwd=1" "c4 --horizon 20 --set accel_fwd=1 --set outer_warm=1" "c5 --horizon 2 --set accel_fwd=1 --set outer_warm=1" "c2 --horizon 10 --set accel_fwd=1"; do
  timeout 150 python tools/devrun.py $a >> gpurun_out/devrun.log 2>&1
done
python - <<'PY'
import json
for l in open("gpurun_out/devrun.log"):
    if not l.startswith("{"): print(l.strip()[:300]); continue
    d = json.loads(l); p = d["prof_all"]
    per = {k: round(1e3 * v[0] / max(v[1], 1), 1) for k, v in p.items() if v[1]}
    print(d["config"], "fwd", d["fwd_s"], "bwd", d["bwd_s"], "dofsteps/s %.3g" % d["dof_steps_per_s"], "its", d["iters_fwd"]["mean"], d["iters_adj"]["mean"], "us/launch", per)
PY
if [ "$1" = "ncu" ]; then
CMD="python tools/devrun.py c5 --horizon 1 --set accel_fwd=1 --set max_iter_fwd=4 --set max_iter_adj=3"
timeout 200 $CMD > gpurun_out/plain_c5.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sweep|k_to_solve|k_from_solve|k_elem|k_gather|k_contact" -c 120 --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_c5.log 2>&1
echo "ncu rc=$?"
fi
