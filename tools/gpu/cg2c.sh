TAG=${1:-cg2c}
for m in on off; do
  if [ $m = off ]; then export C3D_NO_CG2=1; fi
  timeout 300 ncu --set full --clock-control none -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/${TAG}_$m python tools/gemm_bench.py fc1_dx > gpurun_out/${TAG}_${m}_ncu.log 2>&1; echo "ncu $m rc=$?"
  ncu -i gpurun_out/${TAG}_$m.ncu-rep --page raw --csv > gpurun_out/${TAG}_${m}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$m.ncu-rep --page details --csv > gpurun_out/${TAG}_${m}_details.csv 2>/dev/null
  rm -f gpurun_out/${TAG}_$m.ncu-rep
done
