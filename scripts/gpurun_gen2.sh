for v in "RTK_PAIR_GENDBG=0" "RTK_PAIR_GENDBG=2" "RTK_PAIR_GENDBG=4" "RTK_PAIR_GENDBG=6" "RTK_PAIR_SKETCH_GEN=0"; do
  echo -n "$v: "; env $v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pair_power_kernel -c 1 --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | grep -o '"[0-9.]*"$'
done
