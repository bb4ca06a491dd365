#!/bin/bash
# Kernel-time sweep over p (ncu launch list, cold, serialised) + full profiles.
# usage: tools/sweep.sh <tag> [full_p ...]      (full captures: Laplace at those p)
tag=$1; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/sweep_$tag.csv bash -c "for p in 1 2 3 4 5 6 7; do for c in laplace cdr elasticity; do python tools/prof_run.py --p \$p --nz 16 --launches 2 --coeff \$c; done; done" > /dev/null 2>&1
for fp in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:"sumfact|p1_thread|p2_lane|elastic" -s 2 -c 1 -o gpurun_out/prof_${tag}_p$fp \
    python tools/prof_run.py --p $fp --nz 16 --launches 3 > /dev/null 2>&1
done
echo sweep done
