timeout 600 python -m pytest tests -m gpu -q -x -k "objective or c5s_contact or c2s_conv or determin" 2>&1 | tail -1
timeout 200 python tools/timeline.py c5 --horizon 1 > gpurun_out/tl_c5g.txt 2>&1; grep -E "span|k_gather" gpurun_out/tl_c5g.txt | cut -c1-120
timeout 200 python tools/timeline.py c3 --horizon 2 > gpurun_out/tl_c3g.txt 2>&1; grep -E "span|k_gather" gpurun_out/tl_c3g.txt | cut -c1-120
