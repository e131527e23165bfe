mkdir -p gpurun_out
: > gpurun_out/sweep2.log
for q in 1 4096 8192 16384; do for cm in 1024 2048 4096; do
  echo "quad_max=$q cta_max=$cm" >> gpurun_out/sweep2.log
  HDF_BISECT_QUAD_MAX=$q HDF_BISECT_CTA_MAX=$cm timeout 200 python tools/dbg_cluster.py c2b c4 2>&1 | grep -E "^c[0-9]|critical" | cut -c1-160 >> gpurun_out/sweep2.log
done; done
cat gpurun_out/sweep2.log
