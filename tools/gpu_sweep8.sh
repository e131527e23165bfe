mkdir -p gpurun_out
: > gpurun_out/sweep8.log
for cs in 8 12; do
  echo "cluster=$cs" >> gpurun_out/sweep8.log
  HDF_BISECT_CLUSTER=$cs timeout 400 python tools/dbg_cluster.py c5 c3 c2b 2>&1 | grep -E "^c[0-9]|oracle" | cut -c1-150 >> gpurun_out/sweep8.log
done
for cm in 1024 4096; do
  echo "ctamax=$cm" >> gpurun_out/sweep8.log
  HDF_BISECT_CTA_MAX=$cm timeout 400 python tools/dbg_cluster.py c3 c5 2>&1 | grep -E "^c[0-9]|oracle" | cut -c1-150 >> gpurun_out/sweep8.log
done
cat gpurun_out/sweep8.log
