mkdir -p gpurun_out
TAG=$1
python tools/dbg_cluster.py c2b > gpurun_out/ncu_cl_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bisect -s 1 -c 1 -o gpurun_out/prof_cl_$TAG python tools/dbg_cluster.py c2b > gpurun_out/ncu_cl_$TAG.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_cl_$TAG.log
