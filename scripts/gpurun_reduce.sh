# reduce_gram / step_kernel durations in a C5 solve, L2 not flushed between kernels
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"reduce_gram|step_kernel" --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | head -40
