# ncu launch list + full capture of the bench command (after it exits 0 without ncu)
mkdir -p gpurun_out
TAG=${TAG:-r01}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_range_vpass|k_hpass_combine|k_coeffs_mma|k_bisect" -s 4 -c 4 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo full rc=$?
