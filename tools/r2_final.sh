# Round-2 final pass: profiling (r2_profile.sh), then 16M-set analysis parity and the 1M-set DES parity
# sample on the final kernels.
TAG=${TAG:-r02b}
export TAG
bash tools/r2_profile.sh
python tools/parity_16m.py > gpurun_out/parity_16m_$TAG.json 2> gpurun_out/parity_16m_$TAG.err; echo "parity16m=$?"
python tools/parity_des.py > gpurun_out/parity_des_$TAG.json 2> gpurun_out/parity_des_$TAG.err; echo "parity_des=$?"
