#!/bin/bash
# Event-timed per-p sweep through bench.py (warm, 1 GPU).  usage: tools/bench_sweep.sh <tag> [forms...]
# 1M prisms per p (nz 64); steps whose matrices exceed the output budget stream through a chunk ring.
tag=$1; shift
forms=${*:-laplace cdr elasticity}
mkdir -p gpurun_out
out=gpurun_out/bsweep_$tag.jsonl
: > $out
for coeff in $forms; do
  for p in 1 2 3 4 5 6 7; do
    timeout 600 python bench.py --p $p --coeff $coeff --steps 3 --warmup 3 --no-e2e --no-cpu >> $out 2>> gpurun_out/bsweep_$tag.err
  done
done
python tools/bench_sweep_summary.py $out
