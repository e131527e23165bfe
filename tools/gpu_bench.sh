mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 900 python bench.py --all --steps 10 > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err; echo all rc=$?
cat gpurun_out/bench_all.json; tail -5 gpurun_out/bench_all.err
