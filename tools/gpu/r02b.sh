set -x
timeout 900 python -m pytest tests/test_blocks_gpu.py -x -q > gpurun_out/r02b_blocks.log 2>&1; echo "blocks rc=$?"
timeout 600 python -m pytest tests/test_layer_gpu.py -x -q > gpurun_out/r02b_layer.log 2>&1; echo "layer rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --no-fp32 > gpurun_out/r02b_bench.log 2>&1; echo "bench rc=$?"
