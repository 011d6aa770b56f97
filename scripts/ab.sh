#!/bin/bash
# A/B timing of library variants on ONE box, interleaved:
#   scripts/ab.sh "51 101" lib1.so lib2.so ...
# each entry = best of 4 device-timed solve chunks in a fresh process
sizes="$1"; shift
for r in 1 2 3; do
  for n in $sizes; do
    for lib in "$@"; do
      it=300; [ "$n" -ge 101 ] && it=100
      best=$(HJB_LIB=$lib timeout 180 python scripts/prof_sweep.py $n $it 4 | sed -n 's/.*sweep=\([0-9.]*\) us.*/\1/p' | sort -g | head -1)
      echo "r$r n=$n $(basename $lib .so) best_us=$best"
    done
  done
done
