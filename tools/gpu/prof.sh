# usage: bash tools/gpu/prof.sh TAG [kernel-regex ...]
# launch list of one cfg3 N=1 step (ncu gpu__time_duration, clocks not locked) and one
# `ncu --set full` capture per kernel regex. Outputs under gpurun_out/.
TAG=$1; shift
per=$(python tools/profile_step.py 1 | awk '/launches_per_step/{print $2}')
echo "launches_per_step=$per"
ncu --metrics gpu__time_duration.sum --clock-control none -s $((2*per)) -c $per --csv \
    --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt
cat gpurun_out/${TAG}_launches_summary.txt | head -30
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${TAG}_$k python tools/profile_step.py 2 > /dev/null 2>&1
  ncu -i gpurun_out/${TAG}_$k.ncu-rep --page details --csv > gpurun_out/${TAG}_${k}_details.csv 2>/dev/null
done
