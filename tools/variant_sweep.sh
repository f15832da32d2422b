# A/B of compile-time variants on the GPU: VARIANTS="-DX=1;-DX=0" bash tools/variant_sweep.sh
# Each variant: rebuild, quick parity (test_gpu_parity -k pipelined), bench (kernel times), one line each.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "${VS[@]}"; do
  (cd paper_2404_06452_b200 && make -s clean > /dev/null && make -s EXTRA="$v" > /dev/null 2>&1)
  timeout 600 python -m pytest -q -x ${PYTEST_FILES:-tests/test_gpu_parity.py} -k "${PYTEST_K:-pipelined or worked or random_small or validation}" > gpurun_out/vs_pytest.log 2>&1
  pt=$?
  timeout 900 python bench.py --steps ${STEPS:-10} --no-e2e --no-cpu-baseline ${BENCH_EXTRA:---des-sets 0} > gpurun_out/vs.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/vs.log').read().strip().splitlines()[-1]);print('VARIANT [$v] pytest=$pt', round(d['value']/1e6,1), 'Msets/s pack', round(d['roofline']['kernel_ms'] if d['roofline']['kernel']=='pack_kernel' else d['roofline_other_kernel']['kernel_ms'],3), 'analyze', round(d['roofline']['kernel_ms'] if d['roofline']['kernel']=='analyze_kernel' else d['roofline_other_kernel']['kernel_ms'],3), 'verdict_only', round(d['verdict_only']['value']/1e6,1), 'des', round(d['des']['value']) if 'des' in d else None)" || tail -5 gpurun_out/vs.log
done
(cd paper_2404_06452_b200 && make -s clean > /dev/null && make -s > /dev/null 2>&1)
