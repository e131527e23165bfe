# smoke, all GPU tests, default bench line, all-config bench lines
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 900 python bench.py --all --steps 10 --no-cpu-baseline > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err; echo all rc=$?
