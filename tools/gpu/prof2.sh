# usage: bash tools/gpu/prof2.sh TAG
# launch list of one cfg3 N=1 step + ncu --set full of: tc_gemm (FC1 fwd, the 3rd GEMM),
# flash_fwd, flash_bwd, colsum_chunk. Outputs under gpurun_out/.
TAG=$1
per=$(python tools/profile_step.py 1 | awk '/launches_per_step/{print $2}')
echo "launches_per_step=$per"
ncu --metrics gpu__time_duration.sum --clock-control none -s $((2*per)) -c $per --csv \
    --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt
head -24 gpurun_out/${TAG}_launches_summary.txt
for spec in "tc_gemm:2" "flash_fwd:0" "flash_bwd:0" "colsum_chunk:0" "gelu_save:0" "ln_bwd_vec:0"; do
  k=${spec%%:*}; s=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:$k -s $((s + 0)) -c 1 \
      -o gpurun_out/${TAG}_$k python tools/profile_step.py 1 > /dev/null 2>&1
  ncu -i gpurun_out/${TAG}_$k.ncu-rep --page raw --csv > gpurun_out/${TAG}_${k}_raw.csv 2>/dev/null
done
ls gpurun_out/ | grep $TAG
