for d in 0 1 2; do
  echo "dbg=$d"
  C3D_FLASH_DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:flash_bwd -s 1 -c 1 --csv python tools/profile_step.py 2 2>/dev/null | grep flash | awk -F'","' '{print $NF}'
  C3D_FLASH_DBG=$d C3D_FLASH_TRACE=1 python tools/profile_step.py 1 2>&1 | grep "it  [0-9]:" | head -4
done
