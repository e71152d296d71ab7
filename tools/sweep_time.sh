# sweep_time.sh "lib1 lib2" lo hi "opt1" "opt2" ...
for L in $1; do
  if [ "$L" = "default" ]; then unset SIEVE_LIBRARY; else export SIEVE_LIBRARY=build/libsieve_$L.so; fi
  python tools/time_config.py $2 $3 "${@:4}"
done
