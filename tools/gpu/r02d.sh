timeout 900 python -m pytest tests/test_blocks_gpu.py -x -q 2>&1 | tail -15
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:flash -s 2 -c 2 --csv python tools/profile_step.py 3 2>/dev/null | grep flash | awk -F'","' '{print $5, $NF}'
