ncu --set full --clock-control none --import-source on -k regex:flash_bwd -s 1 -c 1 -o gpurun_out/r02e_bwd python tools/profile_step.py 2 > /dev/null 2>&1
ls -la gpurun_out/
