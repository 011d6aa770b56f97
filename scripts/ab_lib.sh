#!/bin/bash
# A/B of library builds (HJB_LIB) on the ENO/TVD-RK 4D step, interleaved on one box:
#   scripts/ab_lib.sh "101" "3 3 gd" paper_2101_05916_b200/_variants/libhjb_base.so paper_2101_05916_b200/libhjb.so
sizes="$1"; scheme="$2"; shift 2
for r in 1 2; do
  for n in $sizes; do
    for lib in "$@"; do
      it=12; [ "$n" -ge 101 ] && it=6
      read -r o k h <<< "$scheme"
      out=$(HJB_LIB=$lib timeout 300 python scripts/prof_ho.py $n $it $o $k 2 ${h:-gd} | tail -1)
      echo "r$r n=$n [$(basename $lib)] $out"
    done
  done
done
