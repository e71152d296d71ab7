# (C) scaled first hit A/B (SIEVE_C_SCALED 1 = default, 0 = cs0): parity
# subset, then configs 3 / 4 / the G=8 top block (count kernel), config 5, config 2 bitmap
python -m pytest tests -x -q -m gpu -k "config3 or skip_residues or random_intervals or multi_segment or thread_and_occ or config4 or batch or top_of_range or p_squared or tiny or small_ranges" 2>&1 | tail -2
bash tools/ab.sh "default cs0" 3 2,10000000001 1000000000000,1010000000000 8750000003,10000000001
for r in 1 2; do for v in default cs0; do if [ $v = default ]; then L=""; else L=build/libsieve_$v.so; fi; SIEVE_LIBRARY=$L python tools/time_batch.py; SIEVE_LIBRARY=$L python tools/bench_modes.py 2 2>/dev/null | cut -c1-160 | sed "s/^/$v /"; done; done
