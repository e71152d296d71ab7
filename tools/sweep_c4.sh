for L in $1; do
  if [ "$L" = "default" ]; then unset SIEVE_LIBRARY; else export SIEVE_LIBRARY=build/libsieve_$L.so; fi
  for o in "${@:2}"; do echo "== $L $o $(REPS=3 python tools/run_config.py 1000000000000 1010000000000 $o >/dev/null; python - <<PY
import subprocess,time,os,sys
PY
)"; done
done
