mkdir -p gpurun_out
timeout 300 python tools/dbg_cluster.py c1 c2b > gpurun_out/dbg_cluster.log 2>&1; echo dbg rc=$?
tail -80 gpurun_out/dbg_cluster.log
timeout 900 python -m pytest tests/test_gpu_cluster.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_cl.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_cl.log
