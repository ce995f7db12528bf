# cfg1/2/5 on 1, 2 and 4 GPUs (3-D and the 1-D baseline) -> gpurun_out/${TAG}_configs_n*.jsonl
TAG=${1:-cfg5}
python tools/configs_bench.py > gpurun_out/${TAG}_configs_n1.jsonl 2> gpurun_out/${TAG}_configs_n1.err; echo "n1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2980$n tools/configs_bench.py > gpurun_out/${TAG}_configs_n$n.jsonl 2> gpurun_out/${TAG}_configs_n$n.err; echo "n$n rc=$?"
done
timeout 600 python -m pytest tests/test_ops_gpu.py -q -k batched 2>&1 | tail -2
cat gpurun_out/${TAG}_configs_n*.jsonl
