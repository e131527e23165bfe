mkdir -p gpurun_out
timeout 300 python tools/dbg_cluster.py c1 c2b c3 c4 > gpurun_out/dbg_cluster.log 2>&1; echo dbg rc=$?
cat gpurun_out/dbg_cluster.log | tail -12
