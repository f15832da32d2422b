# Default bench run (the driver's command) and the ncu launch list of the same command.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
SMI=$!
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py > gpurun_out/ncu_default.log 2>&1
echo "ncu rc=$?"
kill $SMI
tail -c 3000 gpurun_out/bench_default.log
