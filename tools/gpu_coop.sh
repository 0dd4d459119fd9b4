mkdir -p gpurun_out
PD_K3_COOP=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "global_solve or c3s_batched or c2s_conv or determin" 2>&1 | tail -2
for v in 0 1; do
  PD_K3_COOP=$v timeout 200 python tools/timeline.py c3 --horizon 2 > gpurun_out/tl_c3_co$v.txt 2>&1
  echo "c3 coop=$v rc=$?"; grep -E "span|sweep_level|sweep_coop|sweep_reduce" gpurun_out/tl_c3_co$v.txt | cut -c1-140
done
PD_K3_COOP=1 timeout 200 python tools/timeline.py c5 --horizon 1 > gpurun_out/tl_c5_co1.txt 2>&1
echo "c5 coop=1 rc=$?"; grep -E "span|sweep_level|sweep_coop|sweep_reduce" gpurun_out/tl_c5_co1.txt | cut -c1-140
