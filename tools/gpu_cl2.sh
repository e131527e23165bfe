mkdir -p gpurun_out
timeout 300 python tools/dbg_cluster.py c1 c2b c4 c3 > gpurun_out/dbg_cluster.log 2>&1; echo dbg rc=$?
grep -v "^     node" gpurun_out/dbg_cluster.log | tail -20
HDF_BISECT_GRID_ABOVE=100000 timeout 300 python tools/dbg_cluster.py c2b > gpurun_out/dbg_cluster_g.log 2>&1; echo dbg rc=$?
grep -v "^     node" gpurun_out/dbg_cluster_g.log | tail -3
timeout 900 python -m pytest tests/test_gpu_cluster.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_cl.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_cl.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bisect -c 1 -o gpurun_out/prof_cl python tools/dbg_cluster.py c2b > gpurun_out/ncu_cl.log 2>&1; echo ncu rc=$?
grep -i "error" gpurun_out/ncu_cl.log | tail -3
