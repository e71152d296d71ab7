# A/B of library variants on the same box: tools/ab.sh "v1 v2 ..." REPS RANGE...
VARIANTS=$1; REPS=$2; shift 2
for rep in $(seq $REPS); do
  for v in $VARIANTS; do
    if [ "$v" = default ]; then python tools/ab_ranges.py "$@"; else SIEVE_LIBRARY=build/libsieve_$v.so python tools/ab_ranges.py "$@"; fi
  done
done 2>&1 | sort | awk '{k=$1" "$2; v[k]=v[k]" "$3} END {for (k in v) print k, v[k]}' | sort
