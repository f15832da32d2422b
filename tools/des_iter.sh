# One DES build -> measure iteration on the GPU box: the DES GPU tests, the 1M-set timing (digests on /
# off), the DES parity sample, and (unless NO_NCU) an ncu --set full capture on 100k sets with digests.
TAG=${TAG:-x}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-des or sim or case or fifo}" 2>&1 | tail -4
python tools/des_time.py 1000000 > gpurun_out/des_time_$TAG.json 2>&1; cat gpurun_out/des_time_$TAG.json
python tools/parity_des.py --every 8192 > gpurun_out/parity_des_$TAG.json 2>&1; echo "parity_des=$?"; cat gpurun_out/parity_des_$TAG.json | head -c 600; echo
if [ -z "$NO_NCU" ]; then
DES_DIGEST=1 ncu --set full --clock-control none --import-source on -k regex:simulate_kernel -c 1 -o gpurun_out/prof_des_$TAG \
    python tools/des_prof_run.py ${NCU_SETS:-30000} > gpurun_out/ncu_des_$TAG.log 2>&1; echo "ncu_des=$?"
fi
