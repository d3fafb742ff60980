# fp16 pair engine with group-private half-stage slots: correctness + ring-depth variants (ncu kernel time)
t() { ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:pair_power_kernel -s 1 -c 2 --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | grep -o '"[0-9.]*"$' | tr '\n' ' '; echo; }
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "f16" 2>&1 | tail -2
timeout 300 python scripts/f16_probe2.py 2>&1 | tail -8
for v in "-DRTK_PRAH=5 -DRTK_PRQH=2" "-DRTK_PRAH=4 -DRTK_PRQH=4" "-DRTK_PRAH=3 -DRTK_PRQH=4" "-DRTK_PRAH=4 -DRTK_PRQH=2"; do
  RTK_EXTRA_NVCC_FLAGS="$v" python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
  echo "== $v"; t
done
