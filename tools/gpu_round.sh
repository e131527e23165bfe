# one gpurun call: build check, smoke, GPU tests, bench (default + all configs), ncu launch list + full capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
bash tools/gpu_tests.sh
bash tools/gpu_bench.sh
bash tools/gpu_ncu.sh ${TAG:-r01}
