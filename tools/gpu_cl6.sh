mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cluster.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_cl.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_cl.log
timeout 300 python tools/dbg_cluster.py c2b c3 c5 2>&1 | grep -E "^c[0-9]|oracle" > gpurun_out/dbg6.log
for ga in 1000000 2100000; do echo "gabove=$ga" >> gpurun_out/dbg6.log; HDF_BISECT_GRID_ABOVE=$ga timeout 300 python tools/dbg_cluster.py c5 2>&1 | grep -E "^c[0-9]|oracle" >> gpurun_out/dbg6.log; done
for ga in 65536 131072; do echo "gabove=$ga" >> gpurun_out/dbg6.log; HDF_BISECT_GRID_ABOVE=$ga timeout 300 python tools/dbg_cluster.py c3 2>&1 | grep -E "^c[0-9]|oracle" >> gpurun_out/dbg6.log; done
cat gpurun_out/dbg6.log
