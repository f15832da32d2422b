set -x
CMD="python bench.py --sets-per-gpu 200000 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pack_kernel|analyze_kernel" -s 3 -c 2 -o gpurun_out/prof_v1 $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo ncu2=$?
