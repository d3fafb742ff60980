timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ldl.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_ldl.log
timeout 120 python scripts/step_clocks.py c5 | grep -E "mode 1 step [01]"
for c in c5 c4 c3; do timeout 120 python scripts/prof_solve.py $c 3; done
