#!/usr/bin/env bash
# Sharded C4 step on one GPU (one shard, no collective) and under torchrun with one rank (NCCL
# process group up, split upload forced), B = 1 and 256.  Output: gpurun_out/c4_quick*.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python - > gpurun_out/c4_quick.log 2>&1 <<'PY'
import json, bench
for B, k in ((1, 300), (256, 30)):
    print(json.dumps(bench.run_sharded_c4(None, 1_000_000, B, k, 5)))
PY
echo rc=$?
BENCH_DIST=1 MC_C4_SPLIT_UPLOAD=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
  --master-addr 127.0.0.1 --master-port 29533 scripts/c4_dist.py > gpurun_out/c4_quick_dist.log 2>&1
echo rc=$?
