TAG=${1:-sk}
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/${TAG}_test.log 2>&1; echo "gemm tests rc=$?"; tail -3 gpurun_out/${TAG}_test.log
timeout 200 python tools/gemm_bench.py 2>&1 | tee gpurun_out/${TAG}_gb.log
C3D_NO_SK=1 timeout 200 python tools/gemm_bench.py 2>&1 | tee gpurun_out/${TAG}_gb_nosk.log
