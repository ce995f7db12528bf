# multi-GPU suite on a 4-GPU box: pytest (2- and 4-rank parity), mp_parity logs per grid, N=2/N=4 bench
TAG=${1:-mpall}
timeout 1200 python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest multigpu rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29712 tools/mp_parity.py 2x1x1 > gpurun_out/${TAG}_mp_2x1x1.log 2>&1; echo "mp 2x1x1 rc=$?"
for g in 2x2x1 1x2x2 2x1x2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29714 tools/mp_parity.py $g > gpurun_out/${TAG}_mp_$g.log 2>&1; echo "mp $g rc=$?"
  grep -c PASS gpurun_out/${TAG}_mp_$g.log; grep FAIL gpurun_out/${TAG}_mp_$g.log | head -5
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29720 bench.py --gpus 2 --steps 20 --warmup 5 --no-fp32 --no-cfg4 > gpurun_out/${TAG}_bench_n2.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/${TAG}_bench_n2.log | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29740 bench.py --gpus 4 --steps 20 --warmup 5 --no-fp32 --no-cfg4 > gpurun_out/${TAG}_bench_n4.log 2>&1; echo "bench4 rc=$?"
tail -1 gpurun_out/${TAG}_bench_n4.log | cut -c1-300
