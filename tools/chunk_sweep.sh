for K in 1 2 4 8; do
  PAAM_PIPELINE_CHUNKS=$K python bench.py --steps 10 --no-e2e --no-cpu-baseline --des-sets 0 > gpurun_out/k$K.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/k$K.log').read().strip().splitlines()[-1]);print('K=$K', d['value'], d['ms_per_step'], d['roofline']['sequential_step_ms'])"
done
