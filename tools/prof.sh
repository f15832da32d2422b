# usage: TAG=v2 bash tools/prof.sh  -> gpurun_out/prof_$TAG.ncu-rep, launches_$TAG.csv
set -x
TAG=${TAG:-x}
CMD="python bench.py --sets-per-gpu ${SETS:-200000} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KRE:-pack_kernel|analyze_kernel}" -s 3 -c ${NK:-2} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo ncu=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo ncu2=$?
