TAG=${1:-mp4}
for g in 2x2x1 1x2x2 2x1x2; do
  n=4
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2971$n tools/mp_parity.py $g > gpurun_out/${TAG}_mp_$g.log 2>&1; echo "mp $g rc=$?"
  grep -c PASS gpurun_out/${TAG}_mp_$g.log; grep FAIL gpurun_out/${TAG}_mp_$g.log | head -5
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29740 bench.py --gpus 4 --steps 20 --warmup 5 --no-fp32 > gpurun_out/${TAG}_bench_n4.log 2>&1; echo "bench4 rc=$?"
tail -1 gpurun_out/${TAG}_bench_n4.log | cut -c1-400
