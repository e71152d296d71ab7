# A/B of the region order (SIEVE_C_FIRST): count kernel on config 3, config 4,
# the G=8 top block; config 5 batch; plus the parity suite on the variant
set -x
SIEVE_LIBRARY=build/libsieve_cfirst.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
bash tools/ab.sh "default cfirst" 3 2,10000000001 1000000000000,1010000000000 8750000003,10000000001 | tee gpurun_out/ab_order.txt
for rep in 1 2; do python tools/time_batch.py; SIEVE_LIBRARY=build/libsieve_cfirst.so python tools/time_batch.py; done 2>&1 | tee -a gpurun_out/ab_order.txt
