# c5 bench lines under different environment settings (one gpurun call):
#   ENVS="HDF_HTC_NB=8 HDF_HTC_NB=9" TAG=x bash tools/env_bench.sh   -> gpurun_out/env_<tag>.jsonl
# each entry of ENVS is one run (commas separate several variables of one run: A=1,B=2)
mkdir -p gpurun_out
TAG=${TAG:-e}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo build rc=$?
for e in $ENVS; do
  env $(echo $e | tr ',' ' ') timeout 300 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline ${BENCH_ARGS} 2>>gpurun_out/env_$TAG.err | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); d['env']='$e'; print(json.dumps(d))" >> gpurun_out/env_$TAG.jsonl
  echo "env $e rc=$?"
done
if [ -n "$SWEEP" ]; then timeout 900 python tools/sampled_sweep.py $SWEEP >> gpurun_out/sweep_$TAG.jsonl 2>> gpurun_out/sweep_$TAG.err; echo sweep rc=$?; fi
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "$TESTS" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_$TAG.log
fi
