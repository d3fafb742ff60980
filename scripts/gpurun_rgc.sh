for v in 8 1 2 4; do
  RTK_EXTRA_NVCC_FLAGS="-DRTK_RGC=$v" python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
  echo "== RGC $v"
  bash scripts/gpurun_reduce.sh | sed -n 2,5p | cut -c1-20,120-200
  for c in c5 c4; do timeout 300 python scripts/prof_solve.py $c 5 2>&1 | tail -1 | cut -c1-220; done
done
python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
