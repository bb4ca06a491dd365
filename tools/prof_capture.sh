#!/bin/bash
# ncu --set full captures (source-correlated) of one launch per (p, form):
#   CAPS="4:laplace 3:laplace 2:laplace" TAG=r02c tools/prof_capture.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-cap}
for c in ${CAPS:-4:laplace}; do
  p=${c%%:*}; form=${c#*:}
  timeout ${TMO:-600} ncu --set full --import-source on --clock-control none -c 1 -s ${SKIP:-1} \
    -k regex:"${KREGEX:-sumfact|p1_|p2_|elastic}" -o gpurun_out/${TAG}_p${p}_${form} -f \
    python tools/prof_run.py --p $p --coeff $form --nz ${NZ:-16} --launches 2 > gpurun_out/${TAG}_p${p}_${form}.log 2>&1
  echo "$c rc=$?"
done
