#!/bin/bash
# Quick GPU check of chosen p: golden parity + ncu launch times.  usage: tools/quick.sh <tag> <p>...
tag=$1; shift
python -m pytest tests/test_gpu_golden.py -x -q -m gpu 2>&1 | tail -1
ps="$*"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/quick_$tag.csv \
  bash -c "for p in $ps; do python tools/prof_run.py --p \$p --nz 16 --launches 2; python tools/prof_run.py --p \$p --nz 16 --launches 2 --coeff cdr; done" > /dev/null 2>&1
python tools/sweep_summary.py gpurun_out/quick_$tag.csv
