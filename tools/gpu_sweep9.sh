mkdir -p gpurun_out
: > gpurun_out/sweep9.log
for ga in 0 100000 140000 200000; do
  if [ $ga = 0 ]; then unset HDF_BISECT_GRID_ABOVE; else export HDF_BISECT_GRID_ABOVE=$ga; fi
  echo "gabove=$ga" >> gpurun_out/sweep9.log
  timeout 300 python tools/dbg_cluster.py c2b c2a c4 2>&1 | grep -E "^c[0-9]|oracle" | cut -c1-150 >> gpurun_out/sweep9.log
done
cat gpurun_out/sweep9.log
