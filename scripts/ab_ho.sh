#!/bin/bash
# A/B of the ENO/TVD-RK 4D kernels by env setting, interleaved on one box:
#   scripts/ab_ho.sh "51 101" "3 3" "HJB_HO_ENO3G=0" "HJB_HO_ENO3G=1" ...
# (second argument: spatial order and RK order)
sizes="$1"; scheme="$2"; shift 2
for r in 1 2; do
  for n in $sizes; do
    for envs in "$@"; do
      it=12; [ "$n" -ge 101 ] && it=6
      out=$(env $envs timeout 300 python scripts/prof_ho.py $n $it $scheme 2 | tail -1)
      echo "r$r n=$n [$envs] $out"
    done
  done
done
