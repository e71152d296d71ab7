# Wheel-init diagnostic A/B (profiles/r02_negative_ab.txt item 10): build the
# variant first (tools/build_variants.sh wdiag -DSIEVE_WHEEL_DIAG=1), then run
# this under gpurun.
for v in default wdiag default wdiag; do if [ $v = default ]; then L=""; else L=build/libsieve_$v.so; fi; SIEVE_LIBRARY=$L python tools/phase_prof.py | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['cta_cycles_per_seg']), round(d['init%'],2), round(d['cta_cycles_per_seg']*d['init%']/100), d['ms_with_prof'])"; done
bash tools/ab.sh "default wdiag" 2 2,10000000001
