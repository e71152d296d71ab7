# A/B of the bitmap/list write-back variants on one box:
#   tools/ab_bitmap.sh "default old ctacopy" ROUNDS
VARIANTS=$1; ROUNDS=${2:-2}
for r in $(seq $ROUNDS); do
  for v in $VARIANTS; do
    if [ "$v" = default ]; then lib=""; else lib="SIEVE_LIBRARY=build/libsieve_$v.so"; fi
    env $lib python tools/bench_modes.py 2 segment_kb=208 3b 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        print('$v', 'cfg', d['config'], 'ok', d['ok'], 'kernel_ms %.4f' % d['kernel_ms'], 'wb_only_ms %.4f' % d['writeback_only_ms'], 'wb_frac %.3f' % d['writeback_only_frac'], 'e2e_frac %.3f' % d['hbm_frac_end_to_end'], '| count-only kernel_ms %.4f wb_only_ms %.4f wb_frac %.3f' % (d['count_only_kernel_ms'], d['count_only_writeback_only_ms'], d['count_only_writeback_only_frac']))
    elif 'rror' in l: print('$v', l.strip())
"
  done
done
