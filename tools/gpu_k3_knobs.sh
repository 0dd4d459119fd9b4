# K3 switch sweep on c5 (developer probe): A^-1 time per setting, solution compared with the default run
mkdir -p gpurun_out
run() { env "$@" timeout 300 python tools/k3_time_probe.py c5 /tmp/k3ref_c5.pt 2>&1 | tail -1; }
rm -f /tmp/k3ref_c5.pt
run PD_K3_X=0
run PD_K3_RB=8
run PD_K3_RR=1
for sp in 4 8 12 16; do run PD_K3_SPLIT=$sp PD_K3_RR=1; done
run PD_K3_SPLIT=8 PD_K3_RR=1 PD_K3_RB=8
run PD_K3_X=0
