mkdir -p gpurun_out
T=${1:-t}
run() { echo "$* : $(env "$@" timeout 300 python tools/k3_trace.py ${CFG:-c5} 2>&1 | grep -v -i warn | head -4 | tr '\n' ' ')"; }
{
run PD_K3_PERSIST=0
run PD_K3_PERSIST=1
run PD_K3_PERSIST=1 PD_K3_LATEPF=1
run PD_K3_PERSIST=1 PD_ND_LEAF=128
run PD_K3_PERSIST=0 PD_ND_LEAF=128
} > gpurun_out/${T}_variants.txt 2>&1
cat gpurun_out/${T}_variants.txt
timeout 300 python tools/k3_ptrace.py c5 > gpurun_out/${T}_ptrace.txt 2>&1
cat gpurun_out/${T}_ptrace.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "solve or k3 or shard or c5s_contact_muscle_parity or determinism" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${T}_pytest.log
