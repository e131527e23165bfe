mkdir -p gpurun_out
timeout 300 python tools/dbg_cluster.py c1 c2b c3 c4 > gpurun_out/dbg_cluster.log 2>&1; echo dbg rc=$?
cat gpurun_out/dbg_cluster.log | tail -12
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
