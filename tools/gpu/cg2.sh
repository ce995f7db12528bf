# CTA-pair GEMM check: GEMM parity tests, GEMM microbench with / without pairs, layer tests, bench
TAG=${1:-cg2}
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/${TAG}_gemmtest.log 2>&1; echo "gemm tests rc=$?"; tail -3 gpurun_out/${TAG}_gemmtest.log
timeout 200 python tools/gemm_bench.py > gpurun_out/${TAG}_gb_on.log 2>&1; echo "gb on rc=$?"; cat gpurun_out/${TAG}_gb_on.log
C3D_NO_CG2=1 timeout 200 python tools/gemm_bench.py > gpurun_out/${TAG}_gb_off.log 2>&1; echo "gb off rc=$?"; cat gpurun_out/${TAG}_gb_off.log
timeout 900 python -m pytest tests -m gpu -q -x -k "not mp_parity" > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_gputest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-fp32 --no-cpu-baseline --no-cfg4 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'])"
C3D_NO_CG2=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-fp32 --no-cpu-baseline --no-cfg4 > gpurun_out/${TAG}_bench_off.log 2>&1; echo "bench off rc=$?"
tail -1 gpurun_out/${TAG}_bench_off.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'])"
