#!/bin/bash
# Runs the multi-GPU bench under several NCCL settings and summarises collective time.
# usage (on a GPU box): bash tools/nccl_sweep.sh NGPU
N=${1:-4}
mkdir -p gpurun_out
run() {
  local tag=$1; shift
  env "$@" C3D_PROF_DUMP=1 timeout 300 python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N \
    --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sw_$tag.log 2> gpurun_out/sw_$tag.err
  echo "== $tag ($*) rc=$? $(python -c "import json,sys; l=json.loads(open('gpurun_out/sw_$tag.log').read().strip().splitlines()[-1]); print(round(l['value']), 'seq/s', round(l['ms_per_step'],3), 'ms')" 2>/dev/null)"
  python tools/comm_summary.py gpurun_out/sw_$tag.err $N 2 | tail -4
}
run default X=1
run simple NCCL_PROTO=Simple
run ch32 NCCL_MIN_NCHANNELS=32
run ch32s NCCL_MIN_NCHANNELS=32 NCCL_PROTO=Simple
run ring NCCL_ALGO=Ring NCCL_MIN_NCHANNELS=24
run nvls NCCL_NVLS_ENABLE=1 NCCL_ALGO=NVLS,Ring
run cc NCCL_MIN_CTAS=32 NCCL_MAX_CTAS=32
