TAG=r02h
timeout 900 ncu --set full --clock-control none -k "regex:flash|ln_bwd_sums|ln_fwd|colsum|rowdot|convert|splitk" -s 14 -c 14 -o gpurun_out/${TAG}_other python tools/profile_step.py 1 > gpurun_out/${TAG}_other_ncu.log 2>&1; echo "other ncu rc=$?"
ncu -i gpurun_out/${TAG}_other.ncu-rep --page raw --csv > gpurun_out/${TAG}_other_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_other.ncu-rep
