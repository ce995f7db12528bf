#!/bin/bash
# Sweeps the peer-memory collective kernel's launch shape (graph-timed, 2 GPUs).
for cfg in "512 32 2" "1024 32 1" "256 32 4" "512 64 2" "512 16 2" "1024 64 2"; do
  set -- $cfg
  echo "== threads=$1 chunk_kb=$2 per_sm=$3"
  C3D_SYMM_THREADS=$1 C3D_SYMM_CHUNK_KB=$2 C3D_SYMM_PER_SM=$3 timeout 120 python -m torch.distributed.run \
    --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 tools/coll_bench.py \
    --axis 0 --graph --sizes 0.03,2,8,16,32,64 2>&1 | grep busbw
done
