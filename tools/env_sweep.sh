# A/B of runtime tuning knobs (environment variables) on the default bench:
# CASES="PAAM_PIPELINE_CHUNKS=2;PAAM_PIPELINE_CHUNKS=8 PAAM_PACK_BPSM=4" bash tools/env_sweep.sh
mkdir -p gpurun_out
IFS=';' read -ra CS <<< "${CASES:-}"
for c in "${CS[@]}"; do
  env $c timeout 900 python bench.py --steps ${STEPS:-10} --no-e2e --no-cpu-baseline --des-sets 0 > gpurun_out/es.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/es.log').read().strip().splitlines()[-1]);print('CASE [$c]', round(d['value']/1e6,1), 'Msets/s', round(d['ms_per_step'],3), 'ms/step')" || tail -3 gpurun_out/es.log
done
