mkdir -p gpurun_out
for v in "" "HDF_BISECT_CTA_MAX=4096" "HDF_BISECT_CTA_MAX=1024" "HDF_BISECT_CLUSTER=8" "HDF_BISECT_CLUSTER=8 HDF_BISECT_CTA_MAX=2048" "HDF_BISECT_CLUSTER=4 HDF_BISECT_CTA_MAX=2048"; do
  echo "== $v"; env $v timeout 300 python tools/dbg_cluster.py c2b c4 > gpurun_out/dbg_v.log 2>&1; grep -E "^c|timeline" gpurun_out/dbg_v.log
done
