# One gpurun call of a measurement round (run from the repo root on the GPU box):
#   TAG=r02a STEPS="smoke tests bench all launches full" CONFIGS="c5 c3 c4" bash tools/gpu_round.sh
# smoke: __graft_entry__ smoke(); tests: pytest -m gpu; bench: the default bench line (c5) with the
# cpu_baseline; all: one bench line per config; launches: ncu launch list of the default bench;
# full: one ncu --set full capture per config in CONFIGS (each only after the same command exited 0).
mkdir -p gpurun_out
TAG=${TAG:-r02}
STEPS=${STEPS:-"smoke tests bench all launches full"}
CONFIGS=${CONFIGS:-"c5"}
has() { case " $STEPS " in *" $1 "*) return 0;; esac; return 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt
(nproc; lscpu | grep "Model name") > gpurun_out/host_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo build rc=$?
if has smoke; then timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?; fi
if has tests; then
  timeout 1800 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest rc=$?
  tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
if has bench; then timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?; fi
if has all; then timeout 1200 python bench.py --all --steps 10 --no-cpu-baseline > gpurun_out/bench_all_$TAG.jsonl 2> gpurun_out/bench_all_$TAG.err; echo all rc=$?; fi
if has launches; then
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
  $CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c5.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo launches rc=$?
fi
if has full; then
  for c in $CONFIGS; do
    CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline"
    $CMD > gpurun_out/ncu_plain_${TAG}_$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_range_vpass|k_hpass_combine|k_coeffs|k_bisect|k_fallback}" -s ${NCU_S:-15} -c ${NCU_C:-5} -o gpurun_out/prof_${TAG}_$c $CMD > gpurun_out/ncu_full_${TAG}_$c.log 2>&1; echo full $c rc=$?
    # the reports are large: export the raw page and the per-line source page here, keep the report only if asked
    ncu -i gpurun_out/prof_${TAG}_$c.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_$c.csv 2>/dev/null
    python tools/ncu_summary.py --full-only gpurun_out/prof_${TAG}_$c.ncu-rep > gpurun_out/summary_${TAG}_$c.md 2>&1
    for k in ${NCU_SRC:-k_range_vpass k_hpass_combine k_coeffs_tc}; do
      python tools/ncu_lines.py gpurun_out/prof_${TAG}_$c.ncu-rep 40 $k > gpurun_out/lines_${TAG}_${c}_$k.txt 2>&1
    done
    [ -n "$KEEP_REP" ] || rm -f gpurun_out/prof_${TAG}_$c.ncu-rep
  done
fi
if has sweep; then
  for c in ${SWEEP_CONFIGS:-c5}; do timeout 900 python tools/sampled_sweep.py $c ${SWEEP_STRIDES:-1 4 16 64} >> gpurun_out/sweep_$TAG.jsonl 2>> gpurun_out/sweep_$TAG.err; echo sweep $c rc=$?; done
fi
