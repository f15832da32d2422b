# Round-2 profiling pass (one GPU): the default bench line, the ncu launch list of the same command, and
# ncu --set full captures of fused_kernel (2M sets, the bench's launch), pack_kernel + analyze_kernel
# (the split entry points, 200k sets) and simulate_kernel (100k config-5 sets, digests on).
TAG=${TAG:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_$TAG.csv &
SMI=$!
python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; echo "bench=$?"
kill $SMI
if [ -z "$NO_LAUNCHES" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu_launch=$?"
fi
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 3 -c 1 -o gpurun_out/prof_fused_$TAG \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --des-sets 0 > gpurun_out/ncu_fused_$TAG.log 2>&1; echo "ncu_fused=$?"
ncu --set full --clock-control none --import-source on -k regex:"pack_kernel|analyze_kernel" -c 2 -o gpurun_out/prof_split_$TAG \
    python tools/split_prof_run.py 200000 > gpurun_out/ncu_split_$TAG.log 2>&1; echo "ncu_split=$?"
DES_DIGEST=1 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/prof_des_$TAG \
    python tools/des_prof_run.py 100000 > gpurun_out/ncu_des_$TAG.log 2>&1; echo "ncu_des=$?"
