mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1; echo parity rc=$?
tail -15 gpurun_out/pytest_parity.log
timeout 900 python bench.py --all --steps 10 --no-cpu-baseline > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err; echo all rc=$?
python - <<'PY'
import json
for l in open("gpurun_out/bench_all.json"):
    d = json.loads(l)
    print(d["config"]["workload"], d["value"], d["ms_per_step"], d["stages_ms_per_step"])
PY
tail -3 gpurun_out/bench_all.err
