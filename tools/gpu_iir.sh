mkdir -p gpurun_out
timeout 300 python bench.py --variant iir --steps 10 --no-cpu-baseline > gpurun_out/bench_iir_c2b.json 2> gpurun_out/bench_iir.err; echo iir c2b rc=$?
timeout 300 python bench.py --variant iir --config c5 --steps 5 --no-cpu-baseline > gpurun_out/bench_iir_c5.json 2>> gpurun_out/bench_iir.err; echo iir c5 rc=$?
timeout 300 python bench.py --config c5 --steps 5 --no-cpu-baseline > gpurun_out/bench_fir_c5.json 2>> gpurun_out/bench_iir.err; echo fir c5 rc=$?
CMD="python bench.py --variant iir --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iir.csv $CMD > gpurun_out/ncu_launch_iir.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_iir" -s 2 -c 2 -o gpurun_out/prof_iir $CMD > gpurun_out/ncu_full_iir.log 2>&1; echo full rc=$?
tail -3 gpurun_out/bench_iir.err
