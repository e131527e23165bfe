# usage: bash tools/gpu_ncu_k.sh <kernel-regex> <tag> [config]
mkdir -p gpurun_out
CFG=${3:-c2b}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$1 -c 1 -o gpurun_out/prof_$2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config $CFG > gpurun_out/ncu_$2.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_$2.log
