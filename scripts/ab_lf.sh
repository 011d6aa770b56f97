#!/bin/bash
# A/B of two library builds on the Lax-Friedrichs paths (first order 101^4 / 51^4, ENO3/RK3 101^4):
#   edit the two library paths below; run from the repo root on the GPU box
for r in 1 2; do for lib in paper_2101_05916_b200/_variants/libhjb_prelf.so paper_2101_05916_b200/libhjb.so; do
  echo "r$r [$(basename $lib)] fo101: $(HJB_LIB=$lib python scripts/prof_ho.py 101 20 1 1 1 lf | tail -1)"
  echo "r$r [$(basename $lib)] fo51: $(HJB_LIB=$lib python scripts/prof_ho.py 51 200 1 1 1 lf | tail -1)"
  echo "r$r [$(basename $lib)] eno3: $(HJB_LIB=$lib python scripts/prof_ho.py 101 6 3 3 1 lf | tail -1)"
done; done
