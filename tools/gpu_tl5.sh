timeout 600 python -m pytest tests -m gpu -q -x -k "global_solve" 2>&1 | tail -1
timeout 200 python tools/timeline.py c5 --horizon 1 > gpurun_out/tl_c5x.txt 2>&1; grep -E "span|sweep_level" gpurun_out/tl_c5x.txt | cut -c1-120
timeout 200 python tools/timeline.py c3 --horizon 2 > gpurun_out/tl_c3x.txt 2>&1; grep -E "span|sweep_level" gpurun_out/tl_c3x.txt | cut -c1-120
