timeout 60 python tools/devrun.py c5 --horizon 1 --set max_iter_fwd=3 --set max_iter_adj=2 > gpurun_out/d5.log 2>&1; echo "c5 rc=$?"; tail -3 gpurun_out/d5.log | cut -c1-300
timeout 60 python tools/devrun.py c3 --horizon 1 --set max_iter_fwd=3 --set max_iter_adj=2 > gpurun_out/d3.log 2>&1; echo "c3 rc=$?"; tail -3 gpurun_out/d3.log | cut -c1-300
