# grid-mode threshold after the staged side words: c5 / c3 / c2b
mkdir -p gpurun_out
: > gpurun_out/sweep5.log
for ga in 0 300000 600000 1200000 2400000; do
  if [ $ga = 0 ]; then unset HDF_BISECT_GRID_ABOVE; else export HDF_BISECT_GRID_ABOVE=$ga; fi
  echo "gabove=$ga" >> gpurun_out/sweep5.log
  timeout 300 python tools/dbg_cluster.py c5 c2b 2>&1 | grep -E "^c[0-9]|oracle" | cut -c1-150 >> gpurun_out/sweep5.log
done
cat gpurun_out/sweep5.log
