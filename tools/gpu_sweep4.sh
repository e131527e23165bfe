mkdir -p gpurun_out
: > gpurun_out/sweep4.log
for ga in 0 140000 200000 262144; do
  if [ $ga = 0 ]; then unset HDF_BISECT_GRID_ABOVE; else export HDF_BISECT_GRID_ABOVE=$ga; fi
  echo "gabove=$ga" >> gpurun_out/sweep4.log
  timeout 200 python tools/dbg_cluster.py c4 c3 2>&1 | grep -E "^c[0-9]|critical|oracle" | cut -c1-170 >> gpurun_out/sweep4.log
done
cat gpurun_out/sweep4.log
