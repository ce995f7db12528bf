TAG=${1:-fb}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flash_bwd -s 1 -c 1 -o gpurun_out/${TAG} python tools/profile_step.py 1 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
rm -f gpurun_out/${TAG}.ncu-rep
