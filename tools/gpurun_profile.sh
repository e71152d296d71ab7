# Round profiling pass (run under gpurun): GPU tests, bench, modes + oracle
# report, K0, per-rank blocks, F3 A/B, phase counters, the ncu launch list and
# `--set full` captures of the sieve kernel (config 3 from bench.py, the
# config-5 batch kernel, the config-4 count kernel).
# tools/make_profile_summary.py <tag> turns gpurun_out/ into profiles/.
set -x
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
python tools/bench_modes.py --report=gpurun_out/report.json > gpurun_out/modes.jsonl 2> gpurun_out/modes.err; cat gpurun_out/modes.jsonl; tail -3 gpurun_out/modes.err
make build/k0_peaks > /dev/null 2>&1; ./build/k0_peaks > gpurun_out/k0.json; cat gpurun_out/k0.json
python tools/rank_blocks.py > gpurun_out/rank_blocks.txt 2>&1; cat gpurun_out/rank_blocks.txt
python tools/f3_ab.py > gpurun_out/f3_ab.jsonl 2>&1; cat gpurun_out/f3_ab.jsonl
python tools/phase_prof.py > gpurun_out/phase.json 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sieve -c 1 -o gpurun_out/prof_sieve python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
python tools/one_batch.py > gpurun_out/ob.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sieve -c 1 -o gpurun_out/prof_batch python tools/one_batch.py > gpurun_out/ncu_batch.log 2>&1
RANGE=1000000000000,1010000000000 python tools/one_launch.py > gpurun_out/ol.log 2>&1 && RANGE=1000000000000,1010000000000 ncu --set full --clock-control none --import-source on -k regex:k_sieve -c 1 -o gpurun_out/prof_config4 python tools/one_launch.py > gpurun_out/ncu_c4.log 2>&1
CFG=3 CALLS=1 python tools/bitmap_prof.py > gpurun_out/bp.log 2>&1 && CFG=3 CALLS=1 ncu --set full --clock-control none --import-source on -k regex:k_sieve -c 1 -o gpurun_out/prof_bitmap python tools/bitmap_prof.py > gpurun_out/ncu_bitmap.log 2>&1
SIEVE_LIBRARY=$PWD/paper_1205_4883_b200/libsieve_check.so python -m pytest tests -x -q -m gpu > gpurun_out/pytest_check.log 2>&1; tail -3 gpurun_out/pytest_check.log
# summaries on the box (the reports exceed gpurun's 64 MiB copy-back): profiles/ files under gpurun_out/prof_summary
mkdir -p gpurun_out/prof_summary
PROFILE_DST=gpurun_out/prof_summary python tools/make_profile_summary.py ${TAG:-r02} > gpurun_out/prof_summary/make_summary.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_bitmap.ncu-rep "ncu --set full: config 3 range in bitmap mode (625 MB), one sieve_bitmap_async launch" > gpurun_out/prof_summary/${TAG:-r02}_ncu_bitmap.txt 2>&1
python tools/line_stalls.py gpurun_out/prof_bitmap.ncu-rep k_sieveILi4ELi1ELb0E 25 >> gpurun_out/prof_summary/${TAG:-r02}_ncu_bitmap.txt 2>&1
rm -f gpurun_out/prof_batch.ncu-rep gpurun_out/prof_config4.ncu-rep gpurun_out/prof_bitmap.ncu-rep
ls -la gpurun_out gpurun_out/prof_summary
