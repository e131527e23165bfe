# Pipelined filter sweep (one gpurun call): c5 bench lines for HDF_PIPE_BANDS x HDF_PIPE_HSM, then the GPU
# tests that run the tensor-core row pass (device and host paths).  Output: gpurun_out/pipe_<tag>.jsonl
mkdir -p gpurun_out
TAG=${TAG:-p}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo build rc=$?
for cfgv in ${PIPE_CFGS:-"1:0" "4:69" "8:69"}; do
  B=${cfgv%%:*}; S=${cfgv##*:}
  HDF_PIPE_BANDS=$B HDF_PIPE_HSM=$S timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} 2>>gpurun_out/pipe_$TAG.err | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); d['pipe']='$cfgv'; print(json.dumps(d))" >> gpurun_out/pipe_$TAG.jsonl
  echo "pipe $cfgv rc=$?"
done
if [ -n "$PIPE_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "$PIPE_TESTS" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_$TAG.log
fi
