# pipe utilisation of the power-step kernel per (l, path): FFMA tile kernel vs fused tcgen05 engine
M=gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active
for l in 10 15 30 40 60 80; do for p in ffma tc; do
  [ $p = tc ] && [ $l -gt 64 ] && continue
  echo "== l=$l path=$p"
  RTK_PATH=$p ncu --metrics $M --clock-control none -k regex:"tile_kernel|fused_power|pair_power" -s 1 -c 1 \
    python -c "
import sys, torch; sys.path.insert(0, '.'); import paper_2506_04840_b200 as rt
g = torch.Generator(device='cuda'); g.manual_seed(0); n, m, l = 1000, 250000, $l
M = torch.randn((m, n), device='cuda', generator=g).t(); Q = torch.randn((n, l), device='cuda', generator=g)
rt.power_step(M, Q); rt.power_step(M, Q); torch.cuda.synchronize()" 2>&1 | grep -E "duration|dram|pipe"
done; done
