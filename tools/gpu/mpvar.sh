# N=4 (2x2x1) bench variants: default, NCCL collectives, no fused RS, both
TAG=${1:-mpvar}
run() {
  name=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29741 bench.py --gpus 4 --steps 20 --warmup 5 --no-fp32 --no-cfg4 --no-cpu-baseline --no-matmul > gpurun_out/${TAG}_$name.log 2>&1
  echo "$name rc=$?"
  tail -1 gpurun_out/${TAG}_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['collectives']['ms_per_step'], d['collectives']['nvlink_bus_gbs'], d['roofline']['achieved'])"
}
run default C3D_DUMMY=1
run nccl C3D_NCCL_COLL=1
run nofrs C3D_NO_FUSED_RS=1
run nccl_nofrs C3D_NCCL_COLL=1 C3D_NO_FUSED_RS=1
