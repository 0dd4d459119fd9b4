mkdir -p gpurun_out
for nb in 2 3 4; do
  PD_K3_NBUF=$nb timeout 300 python tools/timeline.py c5 --horizon 1 > gpurun_out/tl_c5_nb$nb.txt 2>&1
  echo "nbuf=$nb"; head -5 gpurun_out/tl_c5_nb$nb.txt | grep -E "span|sweep"
done
PD_K3_NBUF=3 timeout 300 python tools/timeline.py c3 --horizon 2 > gpurun_out/tl_c3_nb3.txt 2>&1; head -4 gpurun_out/tl_c3_nb3.txt | grep -E "span|sweep"
