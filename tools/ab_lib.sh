# A/B of two builds of libhdf.so inside one gpurun call (kernel variants that differ at compile time): put the
# two libraries in _variants/libhdf_A.so and _variants/libhdf_B.so (build, copy, change the source, build, copy; .so files
# travel with the snapshot), then `gpurun -- 'bash tools/ab_lib.sh'` -> gpurun_out/ab.jsonl (c5 bench lines, ABAB).
# Restore the library of the committed sources afterwards (python -m paper_1811_02363_b200.build).
mkdir -p gpurun_out
for v in A B A B; do
  cp _variants/libhdf_$v.so paper_1811_02363_b200/libhdf.so
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>>gpurun_out/ab.err | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); d['env']='$v'; print(json.dumps(d))" >> gpurun_out/ab.jsonl
  echo "variant $v rc=$?"
done
cp _variants/libhdf_B.so paper_1811_02363_b200/libhdf.so
timeout 600 python -m pytest tests -m gpu -q -x -k "tensor_core or c5_sampled or full_size" -p no:cacheprovider 2>&1 | tail -2
