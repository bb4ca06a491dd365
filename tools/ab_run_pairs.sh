#!/bin/bash
# Times each A/B library only on the degree its name says (ab_<x><p><tag>), plus the default.
# usage: tools/ab_run_pairs.sh coeff nz [name-prefix]
coeff=$1; nz=${2:-64}; pre=${3:-}
for so in paper_1310_1191_b200/libprism_b200_ab_${pre}*.so; do
  lib=$(basename $so); p=$(echo $lib | sed -E 's/libprism_b200_ab_[a-z]+([0-9]).*/\1/')
  PRISM_B200_LIB=$lib timeout 300 python tools/time_p.py --p $p --coeff $coeff --nz $nz 2>&1 | tail -1
done
for p in $(ls paper_1310_1191_b200/libprism_b200_ab_${pre}*.so | sed -E 's/.*_ab_[a-z]+([0-9]).*/\1/' | sort -u); do
  timeout 300 python tools/time_p.py --p $p --coeff $coeff --nz $nz 2>&1 | tail -1
done
