mkdir -p gpurun_out
: > gpurun_out/sweep7.log
echo "default N/6" >> gpurun_out/sweep7.log
timeout 400 python tools/dbg_cluster.py c5 c3 c4 c2b c2a c1 2>&1 | grep -E "^c[0-9]|oracle" | cut -c1-150 >> gpurun_out/sweep7.log
echo "N/5" >> gpurun_out/sweep7.log
HDF_BISECT_GRID_ABOVE=3355443 timeout 300 python tools/dbg_cluster.py c5 2>&1 | grep -E "^c[0-9]|oracle" | cut -c1-150 >> gpurun_out/sweep7.log
HDF_BISECT_GRID_ABOVE=52428 timeout 300 python tools/dbg_cluster.py c3 2>&1 | grep -E "^c[0-9]|oracle" | cut -c1-150 >> gpurun_out/sweep7.log
timeout 600 python -m pytest tests/test_gpu_cluster.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/sweep7.log
cat gpurun_out/sweep7.log
