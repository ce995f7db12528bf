# Round-2 evidence for profiles/: launch list of one cfg3 N=1 step, ncu --set full of every
# tc_gemm launch of one step (summary + traffic json) and of the other step kernels.
TAG=${1:-r02}
per=$(python tools/profile_step.py 1 | awk '/launches_per_step/{print $2}')
echo "launches_per_step=$per"
ncu --metrics gpu__time_duration.sum --clock-control none -s $((2*per)) -c $per --csv \
    --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt
cat gpurun_out/${TAG}_launches_summary.txt
ng=$(grep -c "tc_gemm" gpurun_out/${TAG}_launches.csv)
echo "tc_gemm launches in list: $ng"
timeout 900 ncu --set full --clock-control none -k regex:tc_gemm -s 12 -c 12 -o gpurun_out/${TAG}_gemm \
    python tools/profile_step.py 1 > gpurun_out/${TAG}_gemm_ncu.log 2>&1; echo "gemm ncu rc=$?"
ncu -i gpurun_out/${TAG}_gemm.ncu-rep --page raw --csv > gpurun_out/${TAG}_gemm_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_gemm.ncu-rep
timeout 900 ncu --set full --clock-control none -k "regex:flash|ln_bwd_sums|ln_fwd|colsum|rowdot|convert|splitk" \
    -s 14 -c 14 -o gpurun_out/${TAG}_other python tools/profile_step.py 1 > gpurun_out/${TAG}_other_ncu.log 2>&1; echo "other ncu rc=$?"
ncu -i gpurun_out/${TAG}_other.ncu-rep --page raw --csv > gpurun_out/${TAG}_other_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_other.ncu-rep
ls -la gpurun_out/ | grep $TAG
