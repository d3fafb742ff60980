for v in 1 0; do
  RTK_EXTRA_NVCC_FLAGS="-DRTK_NR2=$v" python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
  echo "== NR2 $v"
  timeout 120 python scripts/step_clocks.py c5 2>&1 | grep "step [15]:" | head -2
  for r in 1 2; do for c in c5 c4; do timeout 300 python scripts/prof_solve.py $c 5 2>&1 | tail -1 | cut -c1-60,170-250; done; done
  [ $v = 0 ] && timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
done
python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
