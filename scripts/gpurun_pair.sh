export RTUCKER_LIB=$PWD/paper_2506_04840_b200/librtucker_prof.so
RTK_FUSED_DBG=4 timeout 60 python scripts/one_power_step.py 1000 1000000 60 2 2>&1 | tail -3
RTK_FUSED_DBG=6 timeout 60 python scripts/one_power_step.py 1000 1000000 60 2 2>&1 | tail -3
RTK_FUSED_DBG=68 timeout 60 python scripts/one_power_step.py 1000 1000000 60 2 2>&1 | tail -3
