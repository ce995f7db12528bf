set -x
nvidia-smi -L
python -m pytest tests -m gpu -q -k "not mp_parity" > gpurun_out/r02a_gputest.log 2>&1; echo "pytest rc=$?"
for n in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2960$n tools/mp_parity.py > gpurun_out/r02a_mp_parity_n$n.log 2>&1; echo "mp$n rc=$?"; done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench_n1.log 2>&1; echo "bench rc=$?"
