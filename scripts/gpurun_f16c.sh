set -x
for lag in 2 4 6 8 12; do echo "lag $lag"; RTK_PAIR_LAG=$lag timeout 300 python scripts/prof_solve.py c5 3 2>&1 | tail -1; done
echo sa3; RTK_PAIR_SA=3 timeout 300 python scripts/prof_solve.py c5 3 2>&1 | tail -1
echo sa3 lag8; RTK_PAIR_SA=3 RTK_PAIR_LAG=8 timeout 300 python scripts/prof_solve.py c5 3 2>&1 | tail -1
RTK_EXTRA_NVCC_FLAGS=-DRTK_PAIR_PROF=1 python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
RTK_POWER_F16=1 timeout 120 python scripts/one_power_step.py 1000 1000000 60 3 2>&1 | grep "pair prof" | tail -2
