for v in default wdiag default wdiag; do if [ $v = default ]; then L=""; else L=build/libsieve_$v.so; fi; SIEVE_LIBRARY=$L python tools/phase_prof.py | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['cta_cycles_per_seg']), round(d['init%'],2), round(d['cta_cycles_per_seg']*d['init%']/100), d['ms_with_prof'])"; done
bash tools/ab.sh "default wdiag" 2 2,10000000001
