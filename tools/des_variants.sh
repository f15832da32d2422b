# A/B of compile-time variants of simulate_kernel on the GPU: VARIANTS="-DX=1;-DX=0" bash tools/des_variants.sh
# Each variant: rebuild, the DES GPU tests, the 1M-set timing (digests on / off), one line each.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "${VS[@]}"; do
  touch paper_2404_06452_b200/csrc/simulate.cu
  make -s -C paper_2404_06452_b200 EXTRA="$v" > /dev/null 2>&1
  timeout 900 python -m pytest -q -x tests/test_gpu_des.py > gpurun_out/dv_pytest.log 2>&1
  echo "VARIANT [$v] pytest=$? $(python tools/des_time.py 1000000 2>&1 | tail -1)"
done
touch paper_2404_06452_b200/csrc/simulate.cu; make -s -C paper_2404_06452_b200 > /dev/null 2>&1
