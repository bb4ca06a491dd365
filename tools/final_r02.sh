#!/bin/bash
# Round-2 measurement set: default bench line (headline + p=1..7 Laplace/CDR
# sweep + load vectors + e2e + CPU reference), the reference arm, an elasticity
# and an FP32 sweep, the ncu launch list of the bench command, full captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02z}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
timeout 900 python bench.py --coeff elasticity --p 1,2,3,4,5,6,7 --sweep "" --steps 3 --no-e2e --no-cpu --no-load \
  > gpurun_out/${T}_elastic.json 2> gpurun_out/${T}_elastic.err
timeout 900 python bench.py --precision f32 --p 1,2,3,4,5,6,7 --sweep "" --steps 3 --no-e2e --no-cpu \
  > gpurun_out/${T}_f32.json 2> gpurun_out/${T}_f32.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --sweep "" --no-e2e --no-cpu --no-parity --no-load \
  > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sumfact_kernel -s 2 -c 1 \
  -o gpurun_out/${T}_p4 -f python tools/prof_run.py --p 4 --nz 16 --launches 3 > /dev/null 2>&1
echo done
