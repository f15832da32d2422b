cd paper_2404_06452_b200
for cfg in "8 4" "9 4" "10 4" "8 5" "9 5"; do
  set -- $cfg
  make -s clean > /dev/null; make -s EXTRA="-DPACK_MINB=$1 -DANA_MINB=$2" > /dev/null 2>&1
  cd ..
  python bench.py --steps 10 --no-e2e --no-cpu-baseline --des-sets 0 > gpurun_out/lb.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/lb.log').read().strip().splitlines()[-1]);print('PACK_MINB=$1 ANA_MINB=$2', round(d['value']/1e6,1), round(d['roofline']['kernel_ms'],3), round(d['roofline_other_kernel']['kernel_ms'],3))"
  cd paper_2404_06452_b200
done
make -s clean > /dev/null; make -s > /dev/null 2>&1
