mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "global_solve or switches or c3s or c5s or c2s or c4s or determin or edge" 2>&1 | tail -2
for v in 0 1; do
  PD_K3_INLINE_REDUCE=$v timeout 200 python tools/timeline.py c5 --horizon 1 > gpurun_out/tl_c5_i$v.txt 2>&1
  echo "inline=$v rc=$?"; grep -E "span|sweep_level|sweep_reduce" gpurun_out/tl_c5_i$v.txt | cut -c1-150
done
timeout 200 python tools/timeline.py c3 --horizon 2 > gpurun_out/tl_c3.txt 2>&1; grep -E "span|sweep_level|sweep_reduce" gpurun_out/tl_c3.txt | cut -c1-150
