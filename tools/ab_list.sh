# A/B of the list emission (SIEVE_LIST_WORDS variants): config 4 list, same box
set -x
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2 3; do
  for v in default lw1 lw3 lw4; do
    if [ "$v" = default ]; then python tools/list_time.py; else SIEVE_LIBRARY=build/libsieve_$v.so python tools/list_time.py; fi
  done
done 2>&1 | grep "list ms" | tee gpurun_out/ab_list.txt
