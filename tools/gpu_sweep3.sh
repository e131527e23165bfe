mkdir -p gpurun_out
: > gpurun_out/sweep3.log
for cl in 16 8; do for cm in 2048 4096; do
  echo "cluster=$cl ctamax=$cm" >> gpurun_out/sweep3.log
  HDF_BISECT_CLUSTER=$cl HDF_BISECT_CTA_MAX=$cm timeout 200 python tools/dbg_cluster.py c2b c4 c2a 2>&1 | grep -E "^c[0-9]|critical" | cut -c1-170 >> gpurun_out/sweep3.log
done; done
cat gpurun_out/sweep3.log
