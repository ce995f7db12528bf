TAG=${1:-fwdcmp}
timeout 600 python -m pytest tests/test_blocks_gpu.py tests/test_layer_gpu.py tests/test_bench_shape_gpu.py -q -x > gpurun_out/${TAG}_test.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_test.log
for v in new old; do
  if [ $v = old ]; then export C3D_FWD_BK128=1; fi
  per=$(python tools/profile_step.py 1 | awk '/launches_per_step/{print $2}')
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:flash_fwd -s 2 -c 1 --csv --log-file gpurun_out/${TAG}_$v.csv python tools/profile_step.py 3 > /dev/null 2>&1
  grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/${TAG}_$v.csv | head -2
  timeout 300 python bench.py --steps 20 --warmup 5 --no-fp32 --no-cpu-baseline --no-cfg4 --no-matmul 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'])"
done
