set -x
cp gpurun_out/pytest_gpu.log gpurun_out/pytest_gpu_prev.log 2>/dev/null
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
python tools/bench_modes.py --report=gpurun_out/report.json > gpurun_out/modes.jsonl 2> gpurun_out/modes.err; tail -4 gpurun_out/modes.jsonl; tail -3 gpurun_out/modes.err
python tools/rank_blocks.py > gpurun_out/rank_blocks.txt 2>&1; cat gpurun_out/rank_blocks.txt
python tools/batch_ranks.py > gpurun_out/batch_ranks.txt 2>&1; tail -5 gpurun_out/batch_ranks.txt
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; tail -2 gpurun_out/launches.csv
