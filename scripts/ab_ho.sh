#!/bin/bash
# A/B of the ENO/TVD-RK 4D kernels by env setting, interleaved on one box:
#   scripts/ab_ho.sh "51 101" "3 3 [gd|lf|lfg]" "HJB_HO_ENO3G=0" "HJB_HO_ENO3G=1" ...
# (second argument: spatial order, RK order and the numerical Hamiltonian)
sizes="$1"; scheme="$2"; shift 2
set -- "$@"
for r in 1 2; do
  for n in $sizes; do
    for envs in "$@"; do
      it=12; [ "$n" -ge 101 ] && it=6
      read -r o k h <<< "$scheme"
      out=$(env $envs timeout 300 python scripts/prof_ho.py $n $it $o $k 2 ${h:-gd} | tail -1)
      echo "r$r n=$n [$envs] $out"
    done
  done
done
