# Round profiling pass (run under gpurun): GPU tests, bench, modes, K0, the
# ncu launch list and one `--set full` capture of the sieve kernel.
# tools/make_profile_summary.py <tag> turns gpurun_out/ into profiles/.
set -x
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
python tools/bench_modes.py > gpurun_out/modes.jsonl 2> gpurun_out/modes.err; cat gpurun_out/modes.jsonl; tail -3 gpurun_out/modes.err
./build/k0_peaks > gpurun_out/k0.json; cat gpurun_out/k0.json
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sieve -c 1 -o gpurun_out/prof_sieve python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
