for v in 2 4 1; do
  RTK_EXTRA_NVCC_FLAGS="-DRTK_OPR=$v" python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
  echo -n "OPR $v: "; ncu --metrics gpu__time_duration.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:omega_planes -c 1 --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | grep -o '"[0-9.]*"$' | tr '\n' ' '; echo
done
for c in 8; do for tb in 128 512; do :; done; done
python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
