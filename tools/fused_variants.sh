# A/B of compile-time variants of fused_kernel on the GPU: VARIANTS="-DX=1;-DX=0" bash tools/fused_variants.sh
# Each variant: rebuild, the bench-size parity test, the bench's analysis legs (3 runs), one line each.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "${VS[@]}"; do
  touch paper_2404_06452_b200/csrc/fused.cu
  make -s -C paper_2404_06452_b200 EXTRA="$v" > /dev/null 2>&1
  timeout 600 python -m pytest -q -x tests/test_gpu_fullsize.py -k analysis_parity > gpurun_out/fv_pytest.log 2>&1
  pt=$?
  for r in 1 2 3; do
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --des-sets 0 > gpurun_out/fv.json 2>/dev/null
    python -c "import json; d = json.load(open('gpurun_out/fv.json')); print('VARIANT [$v] pytest=$pt %.1f Msets/s kernel %.3f ms verdict_only %.1f' % (d['value'] / 1e6, d['roofline']['kernel_ms'], d['verdict_only']['value'] / 1e6))"
  done
done
touch paper_2404_06452_b200/csrc/fused.cu; make -s -C paper_2404_06452_b200 > /dev/null 2>&1
