mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "objective or c5s_muscle or c3s" 2>&1 | tail -2
timeout 200 python tools/timeline.py c5 --horizon 1 > gpurun_out/tl_c5b.txt 2>&1; head -10 gpurun_out/tl_c5b.txt | grep -E "span|elem_res"
timeout 200 python tools/timeline.py c3 --horizon 2 > gpurun_out/tl_c3b.txt 2>&1; head -10 gpurun_out/tl_c3b.txt | grep -E "span|elem_res"
