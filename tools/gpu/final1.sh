# single-GPU: full gpu test suite, default bench (all extras), smoke
TAG=${1:-final1}
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1200 python bench.py > gpurun_out/${TAG}_bench_n1.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench_n1.log > gpurun_out/${TAG}_bench_n1.json
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/${TAG}_bench_ref.log | cut -c1-300
