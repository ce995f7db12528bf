# single-GPU suite + N=1 bench + launch list
TAG=${1:-quick}
timeout 1200 python -m pytest tests -m gpu -q -x -k "not mp_parity" > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_gputest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-fp32 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'])"
per=$(python tools/profile_step.py 1 | awk '/launches_per_step/{print $2}')
ncu --metrics gpu__time_duration.sum --clock-control none -s $((2*per)) -c $per --csv --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt; head -20 gpurun_out/${TAG}_launches_summary.txt
