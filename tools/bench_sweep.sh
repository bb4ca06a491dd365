#!/bin/bash
# Event-timed per-p sweep through bench.py (warm, 1 GPU).  usage: tools/bench_sweep.sh <tag>
# p <= 5 at 1M prisms (nz 64); p = 6, 7 at 262K (nz 16) so K fits in HBM.
tag=$1
mkdir -p gpurun_out
out=gpurun_out/bsweep_$tag.jsonl
: > $out
for coeff in laplace cdr; do
  for p in 1 2 3 4 5 6 7; do
    nz=64; [ $p -ge 6 ] && nz=16
    timeout 300 python bench.py --p $p --coeff $coeff --nz $nz --steps 5 --warmup 3 --no-e2e --no-cpu >> $out 2>> gpurun_out/bsweep_$tag.err
  done
done
python tools/bench_sweep_summary.py $out
