for v in "RTK_PAIR_F16=0" "RTK_PAIR_F16=1" "CUDA_LAUNCH_BLOCKING=1"; do echo "== $v"; env $v timeout 120 python scripts/scale_probe.py 1e15 2>&1 | tail -3; done
for s in 1e10 1e12 1e13; do echo "== scale $s"; timeout 120 python scripts/scale_probe.py $s 2>&1 | tail -2; done
