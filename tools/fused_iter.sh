# One fused-kernel build -> measure iteration on the GPU box: the analysis GPU tests, the bench (analysis
# legs only) and an ncu --set full capture of fused_kernel at the bench's launch (2M sets).
TAG=${TAG:-x}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-parity or fullsize or admit}" 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --des-sets 0 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "
import json; d = json.load(open('gpurun_out/bench_$TAG.json')); r = d['roofline']
print('value %.1fM sets/s  step %.3f ms  kernel %.3f ms' % (d['value'] / 1e6, d['ms_per_step'], r['kernel_ms']))"
if [ -z "$NO_NCU" ]; then
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 3 -c 1 -o gpurun_out/prof_fused_$TAG \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --des-sets 0 > gpurun_out/ncu_fused_$TAG.log 2>&1; echo "ncu_fused=$?"
fi
