per=$(python tools/profile_step.py 1 | awk '/launches_per_step/{print $2}')
for d in 0 1 2; do
  C3D_FLASH_DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:flash -s 2 -c 2 --csv python tools/profile_step.py 3 2>/dev/null | grep flash | awk -F'","' -v d=$d '{print "dbg="d, $5, $NF}'
done
