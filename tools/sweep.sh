# quick parameter sweep of the headline bench (no cpu baseline)
for args in "$@"; do
  python bench.py --steps 10 --warmup 2 --no-cpu-baseline $args 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$args', 'ms=%.3f'%d['ms_per_step'], 'sieve_ms=%.3f'%r['kernel_ms'], 'frac=%.3f'%r['frac'], 'ok=',d['verified'], 'clk=',d['clocks']['sm_mhz'])
    elif 'Error' in l or 'error' in l: print(l.strip())
"
done
