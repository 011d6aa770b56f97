#!/bin/bash
# A/B timing of environment settings on ONE box, interleaved:
#   scripts/ab_env.sh "51 101" "HJB_MAXT=576" "HJB_MAXT=320" ...
# each entry = best of 4 device-timed solve chunks in a fresh process
sizes="$1"; shift
for r in 1 2 3; do
  for n in $sizes; do
    for e in "$@"; do
      it=300; [ "$n" -ge 101 ] && it=100
      best=$(env HJB_AUTOTUNE=0 $e timeout 180 python scripts/prof_sweep.py $n $it 4 | sed -n 's/.*sweep=\([0-9.]*\) us.*/\1/p' | sort -g | head -1)
      echo "r$r n=$n [$e] best_us=$best"
    done
  done
done
