mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "c2s or c3s or c5s or c4s or determin or edge" 2>&1 | tail -2
timeout 200 python tools/timeline.py c5 --horizon 1 > gpurun_out/tl_c5.txt 2>&1; head -4 gpurun_out/tl_c5.txt | grep -E "span"
timeout 200 python tools/timeline.py c3 --horizon 2 > gpurun_out/tl_c3.txt 2>&1; head -4 gpurun_out/tl_c3.txt | grep -E "span"
