mkdir -p gpurun_out
timeout 300 python tools/dbg_cluster.py c1 c2b c4 c3 > gpurun_out/dbg_cluster.log 2>&1; echo dbg rc=$?
grep -v "^     node" gpurun_out/dbg_cluster.log | tail -20
timeout 900 python -m pytest tests/test_gpu_cluster.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_cl.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_cl.log
timeout 300 python tools/dbg_cluster.py c5 > gpurun_out/dbg_c5.log 2>&1; echo dbg5 rc=$?
grep -v "^     node" gpurun_out/dbg_c5.log | tail -5
