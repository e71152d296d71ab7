for r in 1 2; do for v in default ph16 ph4 ilp4 ilp16; do if [ $v = default ]; then L=""; else L=build/libsieve_$v.so; fi
SIEVE_LIBRARY=$L python tools/time_batch.py | sed "s/^/$v /"
SIEVE_LIBRARY=$L python tools/time_config.py 1000000000000 1010000000000 | sed "s/^/$v c4 /"
SIEVE_LIBRARY=$L python tools/time_config.py 2 10000000001 | sed "s/^/$v c3 /"
done; done
