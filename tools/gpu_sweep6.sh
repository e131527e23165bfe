mkdir -p gpurun_out
: > gpurun_out/sweep6.log
for ga in 4200000 8400000; do
  export HDF_BISECT_GRID_ABOVE=$ga; echo "gabove=$ga" >> gpurun_out/sweep6.log
  timeout 300 python tools/dbg_cluster.py c5 2>&1 | grep -E "^c[0-9]|oracle" | cut -c1-150 >> gpurun_out/sweep6.log
done
for ga in 0 32768 65536; do
  if [ $ga = 0 ]; then unset HDF_BISECT_GRID_ABOVE; else export HDF_BISECT_GRID_ABOVE=$ga; fi
  echo "gabove=$ga" >> gpurun_out/sweep6.log
  timeout 300 python tools/dbg_cluster.py c3 2>&1 | grep -E "^c[0-9]|oracle" | cut -c1-150 >> gpurun_out/sweep6.log
done
cat gpurun_out/sweep6.log
