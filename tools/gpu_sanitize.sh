# one compute-sanitizer tool per call, on a small program that runs clean without it
CMD="python tools/devrun.py c4s --horizon 4"
timeout 200 $CMD > gpurun_out/plain_san.log 2>&1 && \
timeout 900 compute-sanitizer --tool ${1:-memcheck} --print-limit 20 $CMD > gpurun_out/sanitize_${1:-memcheck}.log 2>&1
echo "sanitizer rc=$?"; tail -5 gpurun_out/sanitize_${1:-memcheck}.log
