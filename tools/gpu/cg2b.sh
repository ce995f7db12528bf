TAG=${1:-cg2b}
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/${TAG}_gemmtest.log 2>&1; echo "gemm tests rc=$?"; tail -2 gpurun_out/${TAG}_gemmtest.log
C3D_GEMM_VERBOSE=1 timeout 200 python tools/gemm_bench.py 2>&1 | tee gpurun_out/${TAG}_gb_on.log
