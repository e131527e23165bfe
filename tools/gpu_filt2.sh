mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_par.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
HDF_COEFFS_FMA=1 timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench_q2.json 2>> gpurun_out/bench_q.err; echo bench2 rc=$?
timeout 900 python bench.py --all --steps 10 --no-cpu-baseline > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err; echo all rc=$?
