mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck python tools/dbg_cluster.py c1 32 > gpurun_out/san_cluster.log 2>&1; echo san rc=$?
head -60 gpurun_out/san_cluster.log
timeout 120 python tools/dbg_cluster.py c1 > gpurun_out/dbg_c1.log 2>&1; tail -5 gpurun_out/dbg_c1.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|Error|assert" gpurun_out/pytest_parity.log | head -40
