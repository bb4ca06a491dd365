#!/bin/bash
# Times every A/B library variant (and the default) on the given (p, form) list.
# usage: tools/ab_run.sh "4:laplace 3:laplace" [nz]
cases=$1; nz=${2:-32}
for so in paper_1310_1191_b200/libprism_b200.so paper_1310_1191_b200/libprism_b200_ab_*.so; do
  lib=$(basename $so)
  for c in $cases; do
    p=${c%%:*}; f=${c##*:}
    PRISM_B200_LIB=$lib timeout 300 python tools/time_p.py --p $p --coeff $f --nz $nz 2>&1 | tail -1
  done
done
