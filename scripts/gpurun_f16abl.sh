# fp16 pair engine: role timers (PROF build) and ablations (ABL build), C5 mode-1 shape via the test hook
set -x
RTK_EXTRA_NVCC_FLAGS=-DRTK_PAIR_PROF=1 python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
RTK_POWER_F16=1 timeout 120 python scripts/one_power_step.py 1000 1000000 60 3 2>&1 | grep "pair prof" | tail -2
RTK_EXTRA_NVCC_FLAGS=-DRTK_PAIR_ABL=1 python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
for d in 0 1 2 8 16 32 3 40 11; do
  echo "== dbg $d"
  RTK_PAIR_DBG=$d RTK_POWER_F16=1 timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pair_power_kernel -s 1 -c 1 --csv \
    python scripts/one_power_step.py 1000 1000000 60 1 2>/dev/null | grep duration | awk -F'","' '{print $NF}'
done
