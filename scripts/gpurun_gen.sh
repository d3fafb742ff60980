# in-kernel Omega generation in the pair sketch: tests, A/B timings, sketch kernel time
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for g in 1 0; do RTK_PAIR_SKETCH_GEN=$g timeout 300 python scripts/prof_solve.py c5 5 2>&1 | tail -1 | cut -c1-220; done
for g in 1 0; do RTK_PAIR_SKETCH_GEN=$g timeout 300 python scripts/prof_solve.py c3 5 2>&1 | tail -1 | cut -c1-220; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:pair_power_kernel -c 1 --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | grep -o '"[0-9.]*"$' | tr '\n' ' '; echo
