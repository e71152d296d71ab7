# A/B of list-emission variants (config 4 list, same box): tools/ab_list.sh "v1 v2 ..." (default = in-tree lib)
set -x
VARIANTS=${1:-"default st0"}
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2 3; do
  for v in $VARIANTS; do
    if [ "$v" = default ]; then python tools/list_time.py; else SIEVE_LIBRARY=build/libsieve_$v.so python tools/list_time.py; fi
  done
done 2>&1 | grep "list ms" | tee gpurun_out/ab_list.txt
