# A/B of analyze_kernel's L2 prefetch of the next record (ANA_PF 0: none, 1: every line, 2: live lines):
# split-path parity tests, bench split_path timing, and the kernel's DRAM bytes (ncu, 200k sets).
mkdir -p gpurun_out
for v in ${PFS:-0 1 2}; do
  touch paper_2404_06452_b200/csrc/analyze.cu
  make -s -C paper_2404_06452_b200 EXTRA="-DANA_PF=$v" > /dev/null 2>&1
  timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullsize.py > gpurun_out/pf_pytest.log 2>&1
  pt=$?
  for r in 1 2; do
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --des-sets 0 > gpurun_out/pf.json 2>/dev/null
    python -c "import json; d = json.load(open('gpurun_out/pf.json'))['split_path']; print('ANA_PF=$v pytest=$pt pack %.3f ms analyze %.3f ms' % (d['pack_kernel_ms'], d['analyze_kernel_ms']))"
  done
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none \
      -k regex:analyze_kernel -s 2 -c 1 --csv python bench.py --sets-per-gpu 200000 --steps 1 --warmup 3 --no-e2e \
      --no-cpu-baseline --des-sets 0 > gpurun_out/pf_ncu_$v.csv 2>/dev/null; grep -E "dram__|inst_executed|duration" gpurun_out/pf_ncu_$v.csv | tail -4
done
touch paper_2404_06452_b200/csrc/analyze.cu; make -s -C paper_2404_06452_b200 > /dev/null 2>&1
