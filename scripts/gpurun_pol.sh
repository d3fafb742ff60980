# L2 policy of the streamed op1 tiles vs the small solver's cold code
set -x
for pol in 0 1 2; do
  echo "== pair op1 policy $pol"
  RTK_PAIR_OP1POL=$pol timeout 300 python scripts/prof_solve.py c5 3 2>&1 | tail -1
  RTK_PAIR_OP1POL=$pol timeout 120 python scripts/step_clocks.py c5 2>&1 | grep "step [12]:" | head -4
  RTK_PAIR_OP1POL=$pol timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:pair_power_kernel -s 1 -c 2 --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | grep -o '"[0-9.]*"$' | tr '\n' ' '; echo
done
for v in 0 4; do
  echo "== one-CTA var $v"
  RTK_FUSED_VAR=$v timeout 300 python scripts/prof_solve.py c4 3 2>&1 | tail -1
  RTK_FUSED_VAR=$v timeout 120 python scripts/step_clocks.py c4 2>&1 | grep "step [12]:" | head -3
done
