mkdir -p gpurun_out
T=${1:-t}
run() { echo "$* : $(env "$@" timeout 300 python tools/k3_trace.py ${CFG:-c5} 2>&1 | grep -v -i warn | head -1)"; }
{
run PD_K3_MERGE_ROOT=0
run PD_K3_MERGE_ROOT=1
CFG=c3 run PD_K3_MERGE_ROOT=0
CFG=c3 run PD_K3_MERGE_ROOT=1
} > gpurun_out/${T}_variants.txt 2>&1
cat gpurun_out/${T}_variants.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "solve or k3 or shard or contact or plane or determinism or c5f or c4s or c5s" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${T}_pytest.log
