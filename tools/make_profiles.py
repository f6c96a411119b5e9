"""Summarise ncu captures from gpurun_out/ into committed files under profiles/.

usage: python tools/make_profiles.py TAG WORKLOAD
  reads  gpurun_out/launches_<WL>_<TAG>.csv   (ncu --metrics gpu__time_duration.sum launch list)
         gpurun_out/prof_<WL>_<TAG>.ncu-rep   (ncu --set full of the sconv launches)
         gpurun_out/bench_<WL>_<TAG>.json     (the bench line of the same code)
  writes profiles/<TAG>_<WL>_launches.csv, profiles/<TAG>_<WL>_ncu.md, profiles/ncu_traffic.json
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % active"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue % active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thread-instr"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__occupancy_limit_registers", "CTAs/SM (regs)"),
]


def raw(rep):
    if rep.endswith("_raw.csv") or not os.path.exists(rep):
        # exported on the GPU box (`ncu -i REP --page raw --csv`): the .ncu-rep of
        # pattern-specialised kernels is too large to bring back
        out = open(rep[:-len(".ncu-rep")] + "_raw.csv" if rep.endswith(".ncu-rep") else rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(tag, wl):
    os.makedirs("profiles", exist_ok=True)
    # launch list
    lpath = "gpurun_out/launches_%s_%s.csv" % (wl, tag)
    lines = [l for l in open(lpath) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr, data = rows[0], rows[1:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    with open("profiles/%s_%s_launches.csv" % (tag, wl), "w") as f:
        f.write("kernel,duration_ns\n")
        tot = sconv = 0.0
        for r in data:
            f.write('"%s",%s\n' % (r[ik][:120], r[iv]))
            tot += float(r[iv])
            if "sconv" in r[ik]:
                sconv += float(r[iv])
    # full capture
    h, u, d = raw("gpurun_out/prof_%s_%s.ncu-rep" % (wl, tag))
    idx = {k: i for i, k in enumerate(h)}
    bench = json.load(open("gpurun_out/bench_%s_%s.json" % (wl, tag)))
    layers = [l["layer"] for l in bench["layers"]]
    md = ["# ncu summary %s — %s" % (tag, bench["config"]["workload"]), "",
          "Launch list (cold-cache, serialised; `ncu --metrics gpu__time_duration.sum`): sconv kernels = "
          "%.1f%% of all GPU time in the profiled run (the rest is the bench's L2-flush fills and input setup)."
          % (100.0 * sconv / max(tot, 1.0)), "",
          "Full capture (`ncu --set full --clock-control none`), one launch per layer:", ""]
    md.append("| metric | " + " | ".join(layers[:len(d)]) + " |")
    md.append("|---" * (len(d) + 1) + "|")
    for m, name in METRICS:
        if m in idx:
            md.append("| %s (%s) | " % (name, u[idx[m]]) + " | ".join(r[idx[m]] for r in d) + " |")
    stalls = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    md.append("")
    md.append("Top warp-stall samples per launch:")
    md.append("")
    for name, r in zip(layers, d):
        st = sorted(((float(r[idx[k]] or 0), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in stalls),
                    reverse=True)[:6]
        md.append("- %s: %s" % (name, ", ".join("%s %d" % (n, v) for v, n in st)))
    md.append("")
    md.append("Bench line of the same code: %.0f images/s, roofline frac %.4f (%s)." % (
        bench["value"], bench["roofline"]["frac"], bench["roofline"]["kernel"]))
    open("profiles/%s_%s_ncu.md" % (tag, wl), "w").write("\n".join(md) + "\n")
    # traffic per launch for bench.py's roofline.traffic
    tpath = "profiles/ncu_traffic.json"
    tr = json.load(open(tpath)) if os.path.exists(tpath) else {}
    rd, wr = idx["dram__bytes_read.sum"], idx["dram__bytes_write.sum"]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    tr[wl] = {name: (float(r[rd]) * scale[u[rd]] + float(r[wr]) * scale[u[wr]]) for name, r in zip(layers, d)}
    tr["_note"] = "dram__bytes_read.sum + dram__bytes_write.sum per launch from one ncu --set full capture (%s)" % tag
    json.dump(tr, open(tpath, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
