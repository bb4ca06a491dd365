#!/bin/bash
# One gpurun call: GPU tests, the default bench line, and the strong-scaling
# partition check (N = 1 vs 2 ranks sharing the one leased GPU).
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-run}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
  echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
fi
if [ -n "$STRONG" ]; then
  timeout 600 python bench.py --scaling strong --steps 3 --warmup 3 --sweep "" --no-e2e --no-cpu \
    > gpurun_out/${TAG}_strong1.json 2> gpurun_out/${TAG}_strong1.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --scaling strong --steps 3 --warmup 3 --sweep "" --no-e2e --no-cpu \
    > gpurun_out/${TAG}_strong2.json 2> gpurun_out/${TAG}_strong2.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --sweep-p 1,2,3,4 --reps 2 --no-cpu \
    > gpurun_out/${TAG}_weak2.json 2> gpurun_out/${TAG}_weak2.err
fi
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
exit 0
