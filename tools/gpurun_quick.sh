# Quick GPU iteration: parity tests, then bench sweeps (args: sweep specs)
set -x
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
bash tools/sweep.sh "$@" 2>&1 | tee gpurun_out/sweep.txt
