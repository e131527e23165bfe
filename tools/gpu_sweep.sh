mkdir -p gpurun_out
: > gpurun_out/sweep.log
for cl in 16 8; do for cm in 2048 4096 8192 16384; do
  echo "cluster=$cl ctamax=$cm" >> gpurun_out/sweep.log
  HDF_BISECT_CLUSTER=$cl HDF_BISECT_CTA_MAX=$cm timeout 200 python tools/dbg_cluster.py c2b c4 c5 2>&1 | grep -E "^c[0-9]|timeline" >> gpurun_out/sweep.log
done; done
cat gpurun_out/sweep.log
