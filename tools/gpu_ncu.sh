# usage: bash tools/gpu_ncu.sh <tag> [bench args...]
mkdir -p gpurun_out
TAG=$1; shift
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline $@"
$CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_range_vpass|k_hpass_combine|k_bisect|k_coeffs" -s 4 -c 4 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo full rc=$?
tail -3 gpurun_out/ncu_full_$TAG.log
