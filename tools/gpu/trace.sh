C3D_FLASH_TRACE=1 python tools/profile_step.py 1 2>&1 | tail -20
