# usage: bash tools/gpu/kprof.sh TAG KERNEL_REGEX COUNT  -- ncu --set full of COUNT launches of
# one layer step (tools/profile_step.py), raw CSV out
TAG=$1; K=$2; C=${3:-1}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -c $C \
    -o gpurun_out/${TAG} python tools/profile_step.py 1 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
rm -f gpurun_out/${TAG}.ncu-rep
