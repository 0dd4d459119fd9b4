mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "global_solve or c3s or c5s or c2s or c1 or determin or edge" 2>&1 | tail -3
timeout 300 python tools/timeline.py c5 --horizon 1 --seq 80 > gpurun_out/tl_c5.txt 2>&1; head -12 gpurun_out/tl_c5.txt; grep -A70 "gap before" gpurun_out/tl_c5.txt
timeout 300 python tools/timeline.py c3 --horizon 2 > gpurun_out/tl_c3.txt 2>&1; head -8 gpurun_out/tl_c3.txt
