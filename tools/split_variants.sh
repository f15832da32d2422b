# A/B of compile-time variants of pack_kernel / analyze_kernel (the split entry points) on the GPU:
# VARIANTS="-DX=1;-DX=0" bash tools/split_variants.sh -- rebuild, split-path parity tests, bench split_path.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "${VS[@]}"; do
  touch paper_2404_06452_b200/csrc/pack.cu paper_2404_06452_b200/csrc/analyze.cu
  make -s -C paper_2404_06452_b200 EXTRA="$v" > /dev/null 2>&1
  timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "random_small or validation or wide" > gpurun_out/sv_pytest.log 2>&1
  pt=$?
  for r in 1 2; do
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --des-sets 0 > gpurun_out/sv.json 2>/dev/null
    python -c "import json; d = json.load(open('gpurun_out/sv.json'))['split_path']; print('VARIANT [$v] pytest=$pt pack %.3f ms analyze %.3f ms' % (d['pack_kernel_ms'], d['analyze_kernel_ms']))"
  done
done
touch paper_2404_06452_b200/csrc/pack.cu paper_2404_06452_b200/csrc/analyze.cu; make -s -C paper_2404_06452_b200 > /dev/null 2>&1
