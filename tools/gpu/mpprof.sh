TAG=${1:-mpprof}
C3D_PROF_DUMP=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29741 bench.py --gpus 4 --steps 5 --warmup 3 --no-fp32 --no-cfg4 --no-cpu-baseline --no-matmul > gpurun_out/${TAG}_n4.log 2>&1
echo "rc=$?"
grep "c3d prof" gpurun_out/${TAG}_n4.log | head -80
