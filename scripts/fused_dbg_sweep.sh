# fused-kernel bottleneck sweep on the C5 mode-1 shape (needs a -DRTK_FUSED_PROF=1 build):
# kernel cycles (CTA 0) with parts disabled.  bits: 2 no MMA, 16 no LDS, 32 no TMEM st,
# 64 no A loads, 128 no Q loads, 512 aliased 4-deep TMEM ring (timing only); 4 = print
for d in ${@:-4 254 766 516 518}; do
  echo -n "dbg $d: "
  RTK_FUSED_DBG=$d timeout 120 python scripts/one_power_step.py 1000 1000000 60 3 2>&1 | grep "fused dbg" | tail -1 | awk '{print $5}'
done
