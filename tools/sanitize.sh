#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every kernel
# family of tools/sanitize_kernels.py; logs in gpurun_out/sanitize/.
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p $OUT
FAMS=${FAMS:-p1 p2 sumfact pairs dense elastic load fused tc32 initprobe host}
TOOLS=${TOOLS:-memcheck racecheck synccheck initcheck}
for tool in $TOOLS; do
  for fam in $FAMS; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
        timeout ${TMO:-900} compute-sanitizer --tool $tool $extra --print-limit 20 \
      python tools/sanitize_kernels.py --only $fam > $OUT/${tool}_${fam}.log 2>&1
    echo "rc=$?" >> $OUT/${tool}_${fam}.log
    echo "$tool $fam: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/${tool}_${fam}.log | tr '\n' ' ') $(tail -1 $OUT/${tool}_${fam}.log)"
  done
done | tee $OUT/summary.txt
