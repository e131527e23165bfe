# end-of-session refresh: smoke, all GPU tests, bench lines, reference arm, ncu launch list + full capture
bash tools/gpu_quick.sh
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
TAG=r01e bash tools/gpu_ncu_round.sh
