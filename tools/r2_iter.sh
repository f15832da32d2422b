# One build -> measure iteration on the GPU box: GPU tests, the bench (no e2e / cpu / des legs), and an
# ncu --set full capture of pack_kernel + analyze_kernel on 200k sets.   usage: TAG=x bash tools/r2_iter.sh
TAG=${TAG:-x}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -4
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --des-sets 0 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$TAG.json"))
r = d["roofline"]
print("value %.1fM sets/s  step %.3f ms  seq %.3f ms  %s %.3f ms" % (d["value"] / 1e6, d["ms_per_step"], r.get("sequential_step_ms", 0), r.get("kernel"), r.get("kernel_ms", 0)))
o = d.get("roofline_other_kernel", {})
print("other:", o.get("kernel"), o.get("kernel_ms"))
PY
if [ -z "$NO_NCU" ]; then
CMD="python bench.py --sets-per-gpu 200000 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --des-sets 0"
ncu --set full --clock-control none --import-source on -k regex:"${KRE:-pack_kernel|analyze_kernel}" -s 3 -c ${NK:-2} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo ncu=$?
fi
