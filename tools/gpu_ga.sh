mkdir -p gpurun_out
: > gpurun_out/ga.log
for ga in 0 1000000 2100000 4200000; do
  if [ $ga = 0 ]; then unset HDF_BISECT_GRID_ABOVE; else export HDF_BISECT_GRID_ABOVE=$ga; fi
  echo "gabove=$ga" >> gpurun_out/ga.log
  timeout 300 python tools/dbg_cluster.py c5 2>&1 | grep -E "^c[0-9]|timeline|oracle|rror" >> gpurun_out/ga.log
done
for ga in 0 65536 131072 262144; do
  if [ $ga = 0 ]; then unset HDF_BISECT_GRID_ABOVE; else export HDF_BISECT_GRID_ABOVE=$ga; fi
  echo "gabove=$ga" >> gpurun_out/ga.log
  timeout 300 python tools/dbg_cluster.py c3 2>&1 | grep -E "^c[0-9]|timeline|oracle|rror" >> gpurun_out/ga.log
done
cat gpurun_out/ga.log
