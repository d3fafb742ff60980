# ring-depth variants of the fp16 pair engine: kernel time of the C5 mode-1 power steps (ncu)
t() { ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:pair_power_kernel -s 1 -c 2 --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | grep -o '"[0-9.]*"$' | tr '\n' ' '; echo; }
for v in "-DRTK_PRAH=4" "-DRTK_PRAH=2" "-DRTK_PRAH=4 -DRTK_PRQ=4" "-DRTK_PRAH=2 -DRTK_PRQ=2"; do
  RTK_EXTRA_NVCC_FLAGS="$v" python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
  echo "== $v"; t
done
