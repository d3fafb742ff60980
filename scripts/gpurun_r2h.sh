# probe: where C3/C4/C5 time goes -- shift on/off A/B, graph replay A/B, in-order launch lists of one solve
set -x
for c in c3 c4 c5; do timeout 300 python scripts/probe_shift_ab.py $c 20 3; done > gpurun_out/shift_ab_r2h.txt 2>&1
for c in c3 c4 c5; do timeout 300 python scripts/graph_ab.py $c 20 3; done > gpurun_out/graph_ab_r2h.txt 2>&1
for c in c3 c4; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/seq_$c.csv \
     python scripts/one_solve.py $c > /dev/null 2>&1; echo ncu $c rc $?
done
cat gpurun_out/shift_ab_r2h.txt gpurun_out/graph_ab_r2h.txt
