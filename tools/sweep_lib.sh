# run tools/sweep.sh args against variant libraries: sweep_lib.sh "lib1 lib2" "args..."
for L in $1; do
  if [ "$L" = "default" ]; then unset SIEVE_LIBRARY; else export SIEVE_LIBRARY=build/libsieve_$L.so; fi
  echo "== $L"; shift_args="${@:2}"; bash tools/sweep.sh "${@:2}"
done
