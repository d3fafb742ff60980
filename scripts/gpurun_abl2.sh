# op1 vs op2 A-load ablations of the fp16 pair engine, then the tc_op2 max|M| change: tests
RTK_EXTRA_NVCC_FLAGS=-DRTK_PAIR_ABL=1 python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
for d in 0 64 128 2; do
  echo -n "dbg $d: "
  RTK_PAIR_DBG=$d RTK_POWER_F16=1 timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:pair_power_kernel -s 1 -c 1 --csv \
    python scripts/one_power_step.py 1000 1000000 60 1 2>/dev/null | grep -v "^==" | grep -o '"[0-9.]*"$' | tr '\n' ' '; echo
done
python -m paper_2506_04840_b200.build --force > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c5 c3 c4; do timeout 300 python scripts/prof_solve.py $c 5 2>&1 | tail -1 | cut -c1-200; done
