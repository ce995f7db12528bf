# GEMM parity + microbench + layer tests
TAG=${1:-gb}
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py tests/test_ops_gpu.py -q -x > gpurun_out/${TAG}_test.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_test.log
timeout 200 python tools/gemm_bench.py 2>&1 | tee gpurun_out/${TAG}_gb.log
