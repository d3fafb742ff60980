# A/B of the fused kernel's experiment switches on C5 (device ms by kind/mode, prof_solve)
for v in "0 0" "1 0" "1 4" "3 4" "3 8" "3 16" "5 0" "7 8" "2 8"; do
  set -- $v
  echo "== RTK_FUSED_VAR=$1 RTK_FUSED_PF=$2"
  RTK_FUSED_VAR=$1 RTK_FUSED_PF=$2 timeout 120 python scripts/prof_solve.py c5 3
done
