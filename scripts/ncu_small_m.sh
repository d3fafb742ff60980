# pair vs one-CTA engine for the power steps of narrower unfoldings (C5 modes 2/3, C3 modes 1-3)
for shape in "1000 50000 60" "1000 2500 60" "400 160000 40" "400 12000 40" "400 900 40"; do
  for e in "RTK_PAIR=1" "RTK_PAIR=0"; do
    t=$(env $e ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pair_power|fused_power" -s 2 -c 3 --csv python scripts/one_power_step.py $shape 3 2>/dev/null | grep -E "pair_power|fused_power" | awk -F'","' '{print $(NF)}' | sed 's/"//g' | tr '\n' ' ')
    echo "$shape $e: $t"
  done
done
