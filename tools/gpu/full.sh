# full GPU suite (multi-GPU cases need >= 4 GPUs), then the N=1 bench
TAG=${1:-full}
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/${TAG}_gputest.log
for g in 2x1x1 2x2x1 1x2x2; do
  n=$(python -c "import sys; d=[int(v) for v in '$g'.split('x')]; print(d[0]*d[1]*d[2])")
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2970$n tools/mp_parity.py $g > gpurun_out/${TAG}_mp_$g.log 2>&1; echo "mp $g rc=$?"
  grep -c PASS gpurun_out/${TAG}_mp_$g.log; grep FAIL gpurun_out/${TAG}_mp_$g.log | head -5
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_n1.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench_n1.log | cut -c1-600
