export RTK_PAIR=1
for sa in 2 3 2 3; do for L in 8; do echo "SA $sa lag $L"; RTK_PAIR_SA=$sa RTK_PAIR_LAG=$L timeout 60 python scripts/one_power_step.py 1000 1000000 60 20 | tail -1; done; done
RTK_PAIR_SA=3 RTK_PAIR_LAG=4 timeout 60 python scripts/one_power_step.py 1000 1000000 60 20 | tail -1
RTK_PAIR_SA=3 RTK_PAIR_LAG=12 timeout 60 python scripts/one_power_step.py 1000 1000000 60 20 | tail -1
