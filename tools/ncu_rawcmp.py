import csv, sys
want = sys.argv[1].split(',') if len(sys.argv) > 1 and not sys.argv[1].endswith('.csv') else None
files = [a for a in sys.argv[1:] if a.endswith('.csv')]
rows = []
for f in files:
    r = list(csv.reader(open(f)))
    hdr = r[0]
    for row in r[2:]:
        if 'escoin_jit' in ''.join(row):
            rows.append(dict(zip(hdr, row))); break
keys = ["gpu__time_duration.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
 "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
 "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
 "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
 "launch__grid_size", "launch__block_size", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
 "smsp__average_warp_latency_issue_stalled_barrier", ]
stall = [k for k in rows[0] if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
for k in keys + sorted(stall):
    if k in rows[0]:
        vals = [r.get(k, '') for r in rows]
        try:
            if all(float(v.replace(',', '')) < 0.05 for v in vals): continue
        except: pass
        print("%-90s %s" % (k.replace("smsp__average_warps_issue_stalled_", "stall:"), "  ".join("%14s" % v for v in vals)))
