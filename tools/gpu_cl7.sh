mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cluster.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_cl.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_cl.log
timeout 400 python tools/dbg_cluster.py c2b c4 c3 c5 2>&1 | grep -E "^c[0-9]|oracle|critical|rror" > gpurun_out/dbg7.log
cat gpurun_out/dbg7.log
