#!/usr/bin/env python
"""Key raw metrics of every kernel in an ncu report."""
import csv, subprocess, sys
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg.per_second', 'launch__shared_mem_per_block_dynamic',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers']
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
kn = hdr.index("Kernel Name")
for r in data:
    print("==", r[kn][:110])
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w:60s} {r[i]:>16s} {units[i]}")
stalls = [(h, r) for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled_')]
for r in data:
    tot = float(r[hdr.index('smsp__pcsamp_sample_count')])
    st = sorted(((float(r[hdr.index(h)] or 0), h[len('smsp__pcsamp_warps_issue_stalled_'):]) for h, _ in stalls), reverse=True)
    print("   stalls:", ", ".join(f"{n}={v/tot*100:.0f}%" for v, n in st[:8]))
