mkdir -p gpurun_out
for i in 1 2; do timeout 300 python tools/dbg_cluster.py c2b c4 c2a 2>&1 | grep -E "^c[0-9]|critical|oracle"; done > gpurun_out/dbg5.log; echo dbg rc=$?
timeout 900 python -m pytest tests/test_gpu_cluster.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_cl.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_cl.log
cat gpurun_out/dbg5.log
