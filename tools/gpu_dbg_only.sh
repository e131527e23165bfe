mkdir -p gpurun_out
timeout 300 python tools/dbg_cluster.py c2b > gpurun_out/dbg_cluster.log 2>&1; echo dbg rc=$?
cat gpurun_out/dbg_cluster.log | tail -12
