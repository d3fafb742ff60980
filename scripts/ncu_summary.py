"""Key metrics of one ncu --page raw --csv export (profiles/r1_ncu_fused_c5_mode1.txt format)."""
import csv
import sys

KEYS = [
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "derived__memory_l1_conflicts_shared_nway", "dram__bytes_read.sum", "dram__bytes_read.sum.per_second",
    "dram__bytes_write.sum", "gpu__time_duration.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "launch__block_size",
    "launch__grid_size", "launch__registers_per_thread", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "sm__cycles_elapsed.avg",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__inst_executed_op_shared_ld.sum",
]
rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
for k in KEYS:
    if k in h:
        i = h.index(k)
        print(f"{k:90s} {v[i]} {u[i]}")
