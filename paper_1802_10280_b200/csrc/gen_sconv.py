#!/usr/bin/env python3
"""Code generator for the register-tiled sconv kernel variants (sm_100a).

"Kernel customization" (paper §3.4): the paper instantiates C++
templates over filter size, ofmap size and stride.  Here the part that
templates cannot express is generated: the per-record dispatch of the hot
loop.  Each record of a bucket (one input channel c, one output-channel
group of Q channels) is a nonzero weight w with a code = q*K*K + kh*K + kw.
The thread holds Q x (PH x PW) fp32 accumulators and the input window
X~[c][oh0*S .. +XH][ow0*S .. +XW] in registers; the record's code selects,
at compile time, which accumulators and which window registers its PH*PW
FFMAs use:

    acc[q][ph][pw] += w * x[ph*S + kh][pw*S + kw]          (Alg.2 line 9)

The dispatch is a warp-uniform indirect branch (PTX ``brx.idx.uni``) over
the Q*K*K cases — NVVM lowers a C++ switch to a compare tree, so the loop is
emitted as inline PTX.  The next record is loaded while the current one's
FFMAs issue.  One loop runs a warp's whole chunk: a NEXT record (code
Q*K*K) reloads the input window of the next channel in place, DONE
(Q*K*K+1) leaves.

Usage: gen_sconv.py OUTDIR   (writes variant_<name>.cu + variants_table.inc)
"""
import os
import sys
import re
import zlib

# name, K, S, PH, PW, Q   (Q*PH*PW accumulators; ptxas wants acc <= ~112 regs
# so accumulators and window registers can sit in opposite register banks)
# Measured on B200 (tools/microbench4.cu): the warp-uniform indirect branch
# costs ~65-170 cycles per record per warp, and once the Q*K*K cases exceed
# ~12 KB of SASS the targets miss the instruction cache (NC=63: 13.5 TFLOP/s
# vs NC<=36: ~23 TFLOP/s).  So keep NC = Q*K*K <= ~36.
# mode "brx": per-record indirect dispatch; mode "mask": dense per-bucket
# weight block swept in fixed (tap, q) order with warp-uniform forward
# branches over the absent (zero) slots — no indirect branches at all.
REL_D = 8  # "_x" variants: successor window of the per-case jump tables (measured: 8 > 6, 12, 18)

VARIANTS_MASK = [
    ("m3s1_q4_4x4", 3, 1, 4, 4, 4),
    ("m5s1_q2_4x4", 5, 1, 4, 4, 2),
]
# "_s": one shared dispatch site (one small jump table; pays a direct branch
# and an exposed jump-table load per record) — better when Q*K*K is large.
VARIANTS = [
    ("t3s1_q4_4x4_nx", 3, 1, 4, 4, 4),
    ("t3s1_q4_1x13_rx", 3, 1, 1, 13, 4),
    ("t5s1_q2_4x4_nx", 5, 1, 4, 4, 2),
    ("t3s2_q4_2x4_nx", 3, 2, 2, 4, 4),

]


def min_blocks(K, S, PH, PW, Q):
    """CTAs per SM the variant is compiled for (launch bounds): 2 when the
    accumulators + window + ~40 bookkeeping registers fit in 128."""
    XH, XW = (PH - 1) * S + K, (PW - 1) * S + K
    return 2 if Q * PH * PW + XH * XW <= 112 else 1


def chunk_loop(K, S, PH, PW, Q, vec, single=True):
    """One warp's record stream for a whole channel chunk, as one dispatch loop.

    Codes 0..NC-1: FFMA block of (q, kh, kw).  NC (NEXT): payload = byte
    offset of the next channel's window; reload the XH x XW window registers
    from shared memory (vector loads if `vec`) and continue.  NC+1: DONE.
    """
    P = PH * PW
    XH, XW = (PH - 1) * S + K, (PW - 1) * S + K
    XWV = (XW + 3) // 4
    NC = Q * K * K
    nacc = Q * P
    nx = XH * XW
    x0 = nacc                # "+f"(x[i]) window registers (reloaded in place)
    pidx = nacc + nx         # "+r"(p)
    bidx = pidx + 1          # "r"(wbase): shared address of the warp's window in channel 0
    ridx = pidx + 2          # "r"(rowb): row stride in bytes
    # Records are prefetched two ahead: the load issued in case i (record
    # i+3) is first read by the register rotation at the end of case i+1, so
    # shared-memory latency under load is covered by a whole case.
    L = ["{",
         ".reg .b32 cd, wb, cn, wn, cnn, wnn, wa;",
         ".reg .f32 w, d0, d1, d2, d3;",
         "ld.shared.v2.b32 {cd, wb}, [%%%d];" % pidx,
         "ld.shared.v2.b32 {cn, wn}, [%%%d+8];" % pidx,
         "ld.shared.v2.b32 {cnn, wnn}, [%%%d+16];" % pidx,
         "add.u32 %%%d, %%%d, 24;" % (pidx, pidx),
         "mov.b32 w, wb;",
         "ts: .branchtargets " + ", ".join(["L%d" % i for i in range(NC)] + ["LNEXT", "LEND"]) + ";"]
    tail = ["mov.b32 w, wn;",
            "mov.b32 cd, cn;",
            "mov.b32 wn, wnn;",
            "mov.b32 cn, cnn;",
            "ld.shared.v2.b32 {cnn, wnn}, [%%%d];" % pidx,
            "add.u32 %%%d, %%%d, 8;" % (pidx, pidx),
            "brx.idx.uni cd, ts;"]
    # ONE dispatch site: ptxas emits a jump table per brx.idx, and 38 tables
    # of 38 entries overflow the constant cache (indexed LDC misses stalled
    # every record).  Cases end with a direct branch back to DISPATCH.
    # With single=False every case ends with its own brx.idx (the jump-table
    # LDC overlaps the case's FFMAs, but each site gets its own table).
    if single:
        L += ["bra.uni LFIRST;", "DISPATCH:"] + tail[:-1] + ["LFIRST:", "brx.idx.uni cd, ts;"]
    else:
        L.append("brx.idx.uni cd, ts;")
    back = ["bra.uni DISPATCH;"] if single else tail
    for code in range(NC):
        q, kh, kw = code // (K * K), (code // K) % K, code % K
        L.append("L%d:" % code)
        for ph in range(PH):
            for pw in range(PW):
                a = q * P + ph * PW + pw
                xi = x0 + (ph * S + kh) * XW + (pw * S + kw)
                L.append("fma.rn.f32 %%%d, w, %%%d, %%%d;" % (a, xi, a))
        L += back
    # NEXT: reload the window of the channel whose byte offset is in w
    L.append("LNEXT:")
    L.append("mov.b32 wa, w;")
    L.append("add.u32 wa, wa, %%%d;" % bidx)
    for r in range(XH):
        if vec:
            for v in range(XWV):
                regs = []
                for j in range(4):
                    c = 4 * v + j
                    regs.append("%%%d" % (x0 + r * XW + c) if c < XW else "d%d" % j)
                L.append("ld.shared.v4.f32 {%s}, [wa+%d];" % (", ".join(regs), 16 * v))
        else:
            for c in range(XW):
                L.append("ld.shared.f32 %%%d, [wa+%d];" % (x0 + r * XW + c, 4 * c))
        if r + 1 < XH:
            L.append("add.u32 wa, wa, %%%d;" % ridx)
    L += back
    L += ["LEND:", "}"]
    body = "\n".join('      "%s\\n"' % l for l in L)
    outs = ", ".join('"+f"(acc[%d])' % i for i in range(nacc)) + ", " + \
        ", ".join('"+f"(x[%d])' % i for i in range(nx)) + ', "+r"(p)'
    ins = '"r"(wbase), "r"(rowb)'
    return body, outs, ins


def chunk_loop2(K, S, PH, PW, Q):
    """FFMA2 variant of chunk_loop: output pixels are processed in horizontal
    pairs (pw, pw+1) with one fma.rn.f32x2 each; the window is held as pairs
    (x[r][c], x[r][c+1]) for every start column c, rebuilt on NEXT."""
    assert PW % 2 == 0 and S == 1
    P = PH * PW
    XH, XW = (PH - 1) * S + K, (PW - 1) * S + K
    XWV = (XW + 3) // 4
    NP = XW - 1                       # pair start columns per window row
    NC = Q * K * K
    nacc = Q * P // 2
    nx = XH * NP
    x0 = nacc
    pidx = nacc + nx
    bidx, ridx = pidx + 1, pidx + 2
    L = ["{",
         ".reg .b32 cd, wb, cn, wn, wa;",
         ".reg .f32 w, " + ", ".join("t%d" % i for i in range(4 * XWV)) + ";",
         ".reg .b64 w2;",
         "ld.shared.v2.b32 {cd, wb}, [%%%d];" % pidx,
         "ld.shared.v2.b32 {cn, wn}, [%%%d+8];" % pidx,
         "add.u32 %%%d, %%%d, 16;" % (pidx, pidx),
         "mov.b32 w, wb;",
         "ts: .branchtargets " + ", ".join(["L%d" % i for i in range(NC)] + ["LNEXT", "LEND"]) + ";"]
    tail = ["mov.b32 w, wn;", "mov.b32 cd, cn;",
            "ld.shared.v2.b32 {cn, wn}, [%%%d];" % pidx,
            "add.u32 %%%d, %%%d, 8;" % (pidx, pidx),
            "brx.idx.uni cd, ts;"]
    L += ["bra.uni LFIRST;", "DISPATCH:"] + tail[:-1] + ["LFIRST:", "brx.idx.uni cd, ts;"]
    for code in range(NC):
        q, kh, kw = code // (K * K), (code // K) % K, code % K
        L.append("L%d:" % code)
        L.append("mov.b64 w2, {w, w};")
        for ph in range(PH):
            for pw in range(0, PW, 2):
                a = q * (P // 2) + ph * (PW // 2) + pw // 2
                xi = x0 + (ph + kh) * NP + (pw + kw)
                L.append("fma.rn.f32x2 %%%d, w2, %%%d, %%%d;" % (a, xi, a))
        L.append("bra.uni DISPATCH;")
    L.append("LNEXT:")
    L.append("mov.b32 wa, w;")
    L.append("add.u32 wa, wa, %%%d;" % bidx)
    for r in range(XH):
        for v in range(XWV):
            L.append("ld.shared.v4.f32 {t%d, t%d, t%d, t%d}, [wa+%d];" % (4 * v, 4 * v + 1, 4 * v + 2, 4 * v + 3, 16 * v))
        for c in range(NP):
            L.append("mov.b64 %%%d, {t%d, t%d};" % (x0 + r * NP + c, c, c + 1))
        if r + 1 < XH:
            L.append("add.u32 wa, wa, %%%d;" % ridx)
    L.append("bra.uni DISPATCH;")
    L += ["LEND:", "}"]
    body = "\n".join('      "%s\\n"' % l for l in L)
    outs = ", ".join('"+l"(acc[%d])' % i for i in range(nacc)) + ", " + \
        ", ".join('"+l"(x[%d])' % i for i in range(nx)) + ', "+r"(p)'
    ins = '"r"(wbase), "r"(rowb)'
    return body, outs, ins


def chunk_loop_rel(K, S, PH, PW, Q, vec, D):
    """chunk_loop with SMALL per-site jump tables.

    ptxas emits one jump table per brx.idx site; with a site per case the
    tables (NC+2)^2 entries overflow the constant cache and every record's
    indexed LDC misses (measured: the top stall).  Here records are 16 bytes
    {idx, payload, abs, 0}: idx indexes the PREDECESSOR's site list.  Case c's
    list holds only the D codes after c (records of a bucket are sorted by
    code) plus NEXT, DONE and FAR; FAR re-reads the record's absolute code and
    dispatches through the one full list (the prologue / NEXT site's).
    """
    P = PH * PW
    XH, XW = (PH - 1) * S + K, (PW - 1) * S + K
    XWV = (XW + 3) // 4
    NC = Q * K * K
    nacc = Q * P
    nx = XH * XW
    x0 = nacc
    pidx = nacc + nx
    bidx, ridx = pidx + 1, pidx + 2
    full = ", ".join(["L%d" % i for i in range(NC)] + ["LNEXT", "LEND"])
    L = ["{",
         ".reg .b32 cd, wb, cn, wn, cnn, wnn, wa, ab;",
         ".reg .f32 w, d0, d1, d2, d3;",
         "ld.shared.v2.b32 {cd, wb}, [%%%d];" % pidx,
         "ld.shared.v2.b32 {cn, wn}, [%%%d+16];" % pidx,
         "ld.shared.v2.b32 {cnn, wnn}, [%%%d+32];" % pidx,
         "add.u32 %%%d, %%%d, 48;" % (pidx, pidx),
         "mov.b32 w, wb;",
         "tfull: .branchtargets " + full + ";",
         "brx.idx.uni cd, tfull;"]

    def tail(site):
        return ["mov.b32 w, wn;", "mov.b32 cd, cn;", "mov.b32 wn, wnn;", "mov.b32 cn, cnn;",
                "ld.shared.v2.b32 {cnn, wnn}, [%%%d];" % pidx,
                "add.u32 %%%d, %%%d, 16;" % (pidx, pidx),
                "brx.idx.uni cd, %s;" % site]

    for code in range(NC):
        q, kh, kw = code // (K * K), (code // K) % K, code % K
        L.append("L%d:" % code)
        for ph in range(PH):
            for pw in range(PW):
                a = q * P + ph * PW + pw
                xi = x0 + (ph * S + kh) * XW + (pw * S + kw)
                L.append("fma.rn.f32 %%%d, w, %%%d, %%%d;" % (a, xi, a))
        succ = ["L%d" % (code + 1 + i) if code + 1 + i < NC else "LFAR" for i in range(D)]
        L.append("t%d: .branchtargets %s;" % (code, ", ".join(succ + ["LNEXT", "LEND", "LFAR"])))
        L += tail("t%d" % code)
    L.append("LNEXT:")
    L.append("mov.b32 wa, w;")
    L.append("add.u32 wa, wa, %%%d;" % bidx)
    for r in range(XH):
        if vec:
            for v in range(XWV):
                regs = ["%%%d" % (x0 + r * XW + 4 * v + j) if 4 * v + j < XW else "d%d" % j for j in range(4)]
                L.append("ld.shared.v4.f32 {%s}, [wa+%d];" % (", ".join(regs), 16 * v))
        else:
            for c in range(XW):
                L.append("ld.shared.f32 %%%d, [wa+%d];" % (x0 + r * XW + c, 4 * c))
        if r + 1 < XH:
            L.append("add.u32 wa, wa, %%%d;" % ridx)
    L += tail("tfull")
    # FAR: the record being dispatched sits 3 records behind p; its abs field
    L += ["LFAR:", "ld.shared.b32 ab, [%%%d+-40];" % pidx, "brx.idx.uni ab, tfull;"]
    L += ["LEND:", "}"]
    body = "\n".join('      "%s\\n"' % l for l in L)
    outs = ", ".join('"+f"(acc[%d])' % i for i in range(nacc)) + ", " + \
        ", ".join('"+f"(x[%d])' % i for i in range(nx)) + ', "+r"(p)'
    ins = '"r"(wbase), "r"(rowb)'
    return body, outs, ins


def chunk_loop_link(K, S, PH, PW, Q, vec, D, depth=1):
    """Dispatch loop over LINKED records: record r = {idx(r+1), payload(r)}
    (plus {abs(r+1), 0} when D > 0), so the jump-table load for the next
    dispatch uses a register that is ready on entry to the case, and the
    record prefetch rotates only two registers (w, c).  Per record: LDS.64,
    pointer add, table index, LDC, 2 MOV, BRX (vs 4 MOV + 2 loads' worth of
    bookkeeping in chunk_loop).  The stream starts with a header {idx(first)}.

    D == 0: every case's jump list is the full list (idx = absolute code).
    D > 0 : case c's list is the D codes after c + NEXT, DONE, FAR (small
            constant-cache footprint); FAR re-dispatches via the full list from
            the absolute code stored in the record.
    """
    P = PH * PW
    XH, XW = (PH - 1) * S + K, (PW - 1) * S + K
    XWV = (XW + 3) // 4
    NC = Q * K * K
    nacc = Q * P
    nx = XH * XW
    x0 = nacc
    pidx = nacc + nx
    bidx, ridx = pidx + 1, pidx + 2
    RS = 16 if D > 0 else 8
    full = ", ".join(["L%d" % i for i in range(NC)] + ["LNEXT", "LEND"])
    L = ["{",
         ".reg .b32 c, lc, lw, lc2, lw2, wb, wa, t, ab;",
         ".reg .f32 w, d0, d1, d2, d3;",
         "ld.shared.b32 t, [%%%d];" % pidx,
         "ld.shared.v2.b32 {c, wb}, [%%%d+%d];" % (pidx, RS)]
    if depth == 2:  # also record 1: {idx(r2), w(r1)}
        L.append("ld.shared.v2.b32 {lc, lw}, [%%%d+%d];" % (pidx, 2 * RS))
    L += ["add.u32 %%%d, %%%d, %d;" % (pidx, pidx, (3 if depth == 2 else 2) * RS),
          "mov.b32 w, wb;",
          "tfull: .branchtargets " + full + ";",
          "brx.idx.uni t, tfull;"]

    def head():
        if depth == 2:  # depth 2 = depth 1 with the record load issued at the TAIL (after the
            return []   # moves that free its registers), so a whole dispatch hides its latency
        return ["ld.shared.v2.b32 {lc, lw}, [%%%d];" % pidx, "add.u32 %%%d, %%%d, %d;" % (pidx, pidx, RS)]

    def tail(site):
        mv = ["mov.b32 t, c;", "mov.b32 w, lw;", "mov.b32 c, lc;"]
        if depth == 2:
            mv += ["ld.volatile.shared.v2.b32 {lc, lw}, [%%%d];" % pidx, "add.u32 %%%d, %%%d, %d;" % (pidx, pidx, RS)]
        return mv + ["brx.idx.uni t, %s;" % site]

    for code in range(NC):
        q, kh, kw = code // (K * K), (code // K) % K, code % K
        L.append("L%d:" % code)
        L += head()
        for ph in range(PH):
            for pw in range(PW):
                a = q * P + ph * PW + pw
                xi = x0 + (ph * S + kh) * XW + (pw * S + kw)
                L.append("fma.rn.f32 %%%d, w, %%%d, %%%d;" % (a, xi, a))
        if D > 0:
            succ = ["L%d" % (code + 1 + i) if code + 1 + i < NC else "LFAR" for i in range(D)]
            L.append("t%d: .branchtargets %s;" % (code, ", ".join(succ + ["LNEXT", "LEND", "LFAR"])))
            L += tail("t%d" % code)
        else:
            L += tail("tfull")
    L.append("LNEXT:")
    L += head()
    L.append("mov.b32 wa, w;")
    L.append("add.u32 wa, wa, %%%d;" % bidx)
    for r in range(XH):
        if vec:
            for v in range(XWV):
                regs = ["%%%d" % (x0 + r * XW + 4 * v + j) if 4 * v + j < XW else "d%d" % j for j in range(4)]
                L.append("ld.shared.v4.f32 {%s}, [wa+%d];" % (", ".join(regs), 16 * v))
        else:
            for c in range(XW):
                L.append("ld.shared.f32 %%%d, [wa+%d];" % (x0 + r * XW + c, 4 * c))
        if r + 1 < XH:
            L.append("add.u32 wa, wa, %%%d;" % ridx)
    L += tail("tfull")
    if D > 0:
        # FAR: dispatching record r+1 from case r; p = &rec[r+2] (depth 1) or
        # &rec[r+3] (depth 2); abs(r+1) is in rec[r]
        L += ["LFAR:", "ld.shared.b32 ab, [%%%d+%d];" % (pidx, -(3 if depth == 2 else 2) * RS + 8), "brx.idx.uni ab, tfull;"]
    L += ["LEND:", "}"]
    body = "\n".join('      "%s\\n"' % l for l in L)
    outs = ", ".join('"+f"(acc[%d])' % i for i in range(nacc)) + ", " + \
        ", ".join('"+f"(x[%d])' % i for i in range(nx)) + ', "+r"(p)'
    ins = '"r"(wbase), "r"(rowb)'
    return body, outs, ins


def chunk_loop3(K, S, PH, PW, Q):
    """Image-pair variant: every lane holds its patch for two images; the
    window registers are (image 2g, image 2g+1) pairs loaded straight from the
    interleaved slab with ld.shared.v2.b64; one fma.rn.f32x2 per pixel, the
    weight a broadcast scalar operand."""
    assert S == 1
    P = PH * PW
    XH, XW = (PH - 1) * S + K, (PW - 1) * S + K
    assert XW % 2 == 0
    NC = Q * K * K
    nacc = Q * P
    nx = XH * XW
    x0 = nacc
    pidx = nacc + nx
    bidx, ridx = pidx + 1, pidx + 2
    L = ["{",
         ".reg .b32 cd, wb, cn, wn, cnn, wnn, wa;",
         ".reg .f32 w;",
         ".reg .b64 w2;",
         "ld.shared.v2.b32 {cd, wb}, [%%%d];" % pidx,
         "ld.shared.v2.b32 {cn, wn}, [%%%d+8];" % pidx,
         "ld.shared.v2.b32 {cnn, wnn}, [%%%d+16];" % pidx,
         "add.u32 %%%d, %%%d, 24;" % (pidx, pidx),
         "mov.b32 w, wb;",
         "ts: .branchtargets " + ", ".join(["L%d" % i for i in range(NC)] + ["LNEXT", "LEND"]) + ";"]
    tail = ["mov.b32 w, wn;", "mov.b32 cd, cn;", "mov.b32 wn, wnn;", "mov.b32 cn, cnn;",
            "ld.shared.v2.b32 {cnn, wnn}, [%%%d];" % pidx,
            "add.u32 %%%d, %%%d, 8;" % (pidx, pidx),
            "brx.idx.uni cd, ts;"]
    L += ["bra.uni LFIRST;", "DISPATCH:"] + tail[:-1] + ["LFIRST:", "brx.idx.uni cd, ts;"]
    for code in range(NC):
        q, kh, kw = code // (K * K), (code // K) % K, code % K
        L.append("L%d:" % code)
        L.append("mov.b64 w2, {w, w};")
        for ph in range(PH):
            for pw in range(PW):
                a = q * P + ph * PW + pw
                xi = x0 + (ph + kh) * XW + (pw + kw)
                L.append("fma.rn.f32x2 %%%d, w2, %%%d, %%%d;" % (a, xi, a))
        L.append("bra.uni DISPATCH;")
    L.append("LNEXT:")
    L.append("mov.b32 wa, w;")
    L.append("add.u32 wa, wa, %%%d;" % bidx)
    for r in range(XH):
        for v in range(XW // 2):
            L.append("ld.shared.v2.b64 {%%%d, %%%d}, [wa+%d];" % (x0 + r * XW + 2 * v, x0 + r * XW + 2 * v + 1, 16 * v))
        if r + 1 < XH:
            L.append("add.u32 wa, wa, %%%d;" % ridx)
    L.append("bra.uni DISPATCH;")
    L += ["LEND:", "}"]
    body = "\n".join('      "%s\\n"' % l for l in L)
    outs = ", ".join('"+l"(acc[%d])' % i for i in range(nacc)) + ", " + \
        ", ".join('"+l"(x[%d])' % i for i in range(nx)) + ', "+r"(p)'
    ins = '"r"(wbase), "r"(rowb)'
    return body, outs, ins


TEMPLATE_P3 = """// GENERATED by gen_sconv.py — do not edit.
// Variant {name}: K={K} stride={S} patch {PH}x{PW} Q={Q}, image-pair FFMA2 ({NC} dispatch cases).
#include "sconv_tiled.cuh"

namespace escoin {{

template <>
__device__ __forceinline__ void chunk_loop3<{K}, {S}, {PH}, {PW}, {Q}, {TAG}>(unsigned long long* acc, unsigned long long* x,
                                                                     unsigned& p, unsigned wbase, unsigned rowb) {{
  asm volatile(
{body}
      : {outs}
      : {ins}
      : "memory");
}}

int launch_{name}(const TiledArgs& a, cudaStream_t s) {{
  return launch_tiled<{K}, {S}, {PH}, {PW}, {Q}, {MINB}, 3, {TAG}>(a, s);
}}

}}  // namespace escoin
"""

VARIANTS_P3 = [
    ("p3s1_q4_2x4", 3, 1, 2, 4, 4),
]


def min_blocks_p3(K, S, PH, PW, Q):
    XH, XW = (PH - 1) * S + K, (PW - 1) * S + K
    return 2 if 2 * (Q * PH * PW + XH * XW) <= 112 else 1


TEMPLATE_F2 = """// GENERATED by gen_sconv.py — do not edit.
// Variant {name}: K={K} stride={S} patch {PH}x{PW} Q={Q}, FFMA2 pixel pairs ({NC} dispatch cases).
#include "sconv_tiled.cuh"

namespace escoin {{

template <>
__device__ __forceinline__ void chunk_loop2<{K}, {S}, {PH}, {PW}, {Q}, {TAG}>(unsigned long long* acc, unsigned long long* x,
                                                                     unsigned& p, unsigned wbase, unsigned rowb) {{
  asm volatile(
{body}
      : {outs}
      : {ins}
      : "memory");
}}

int launch_{name}(const TiledArgs& a, cudaStream_t s) {{
  return launch_tiled<{K}, {S}, {PH}, {PW}, {Q}, {MINB}, 2, {TAG}>(a, s);
}}

}}  // namespace escoin
"""

# 1x1 row-block variants (mode 4, sconv_1x1.cuh): name, R rows per warp, V pixels per lane
VARIANTS_1X1 = [
    ("d1_r4_v8", 4, 8),
    ("s1_r4_v8", 4, 8),
    ("s1_r1_v8", 1, 8),
    ("s1_r2_v2", 2, 2),
]

TEMPLATE_1X1 = """// GENERATED by gen_sconv.py — do not edit.
// Variant {name}: 1x1 {kind}, R={R} rows per warp, V={V} pixels per lane.
#include "sconv_1x1.cuh"

namespace escoin {{

int launch_{name}(const TiledArgs& a, cudaStream_t s) {{
  return launch_1x1<{R}, {V}, {MINB}, {TAG}, {SP}>(a, s);
}}

}}  // namespace escoin
"""

# Tap-record variants (mode 6, no dispatch): name, K, PH (rows per lane), Q
# (stride 1; the "s2" entries below are stride 2)
VARIANTS_TAP = [
    ("b3_q4_8x1", 3, 8, 4),
    ("b5_q2_16x1", 5, 16, 2),
    ("b3s2_q4_8x1", 3, 8, 4),
]

TEMPLATE_TAP = """// GENERATED by gen_sconv.py — do not edit.
// Variant {name}: K={K} stride={S} tap records (mode 6), column patches {PH}x1, Q={Q}.
#include "sconv_tiled.cuh"

namespace escoin {{

int launch_{name}(const TiledArgs& a, cudaStream_t s) {{
  return launch_tiled<{K}, {S}, {PH}, 1, {Q}, 2, 6, {TAG}>(a, s);
}}

}}  // namespace escoin
"""

# Row-record variants (mode 7, no dispatch; mosaic tiling, lanes over super-image rows,
# PW >= the (super-)row width): name, K, PW (row pixels), Q
VARIANTS_ROW = [
    ("c3_q4_1x13", 3, 13, 4),
    ("c5_q1_1x27", 5, 27, 1),
]

TEMPLATE_ROW = """// GENERATED by gen_sconv.py — do not edit.
// Variant {name}: K={K} row records (mode 7), full-row patches 1x{PW}, Q={Q}.
#include "sconv_tiled.cuh"

namespace escoin {{

int launch_{name}(const TiledArgs& a, cudaStream_t s) {{
  return launch_tiled<{K}, 1, 1, {PW}, {Q}, 2, 7, {TAG}>(a, s);
}}

}}  // namespace escoin
"""

VARIANTS_F2 = [
    ("f3s1_q3_4x4", 3, 1, 4, 4, 3),
]


def min_blocks_f2(K, S, PH, PW, Q):
    XH, XW = (PH - 1) * S + K, (PW - 1) * S + K
    return 2 if Q * PH * PW + 2 * XH * (XW - 1) <= 112 else 1


def bucket_mask(K, S, PH, PW, Q):
    """Dense-bucket sweep: weights [tap][q] (zeros = absent), slot s = tap*Q + q."""
    P = PH * PW
    XH, XW = (PH - 1) * S + K, (PW - 1) * S + K
    NS = Q * K * K
    NV = (NS + 3) // 4
    nacc = Q * P
    widx = nacc           # "r"(wp): shared address of the bucket's weights
    x0 = nacc + 1
    L = ["{", ".reg .pred p;", ".reg .f32 wa0, wa1, wa2, wa3, wb0, wb1, wb2, wb3;",
         "ld.shared.v4.f32 {wa0, wa1, wa2, wa3}, [%%%d];" % widx]
    for v in range(NV):
        cur, nxt = ("wa", "wb") if v % 2 == 0 else ("wb", "wa")
        if v + 1 < NV:
            L.append("ld.shared.v4.f32 {%s0, %s1, %s2, %s3}, [%%%d+%d];" % (nxt, nxt, nxt, nxt, widx, 16 * (v + 1)))
        for lane in range(4):
            sl = 4 * v + lane
            if sl >= NS:
                break
            t, q = sl // Q, sl % Q
            kh, kw = t // K, t % K
            L.append("setp.neu.f32 p, %s%d, 0f00000000;" % (cur, lane))
            L.append("@!p bra.uni SK%d;" % sl)
            for ph in range(PH):
                for pw in range(PW):
                    a = q * P + ph * PW + pw
                    xi = x0 + (ph * S + kh) * XW + (pw * S + kw)
                    L.append("fma.rn.f32 %%%d, %s%d, %%%d, %%%d;" % (a, cur, lane, xi, a))
            L.append("SK%d:" % sl)
    L.append("}")
    body = "\n".join('      "%s\\n"' % l for l in L)
    outs = ", ".join('"+f"(acc[%d])' % i for i in range(nacc))
    ins = '"r"(wp), ' + ", ".join('"f"(x[%d])' % i for i in range(XH * XW))
    return body, outs, ins


TEMPLATE_MASK = """// GENERATED by gen_sconv.py — do not edit.
// Variant {name}: K={K} stride={S} patch {PH}x{PW} Q={Q}, dense-bucket mask sweep ({NS} slots).
#include "sconv_tiled.cuh"

namespace escoin {{

template <>
__device__ __forceinline__ void bucket_mask<{K}, {S}, {PH}, {PW}, {Q}, {TAG}>(float* acc, const float* x, unsigned wp) {{
  asm volatile(
{body}
      : {outs}
      : {ins}
      : "memory");
}}

int launch_{name}(const TiledArgs& a, cudaStream_t s) {{
  return launch_tiled<{K}, {S}, {PH}, {PW}, {Q}, {MINB}, 1, {TAG}>(a, s);
}}

}}  // namespace escoin
"""

TEMPLATE = """// GENERATED by gen_sconv.py — do not edit.
// Variant {name}: K={K} stride={S} patch {PH}x{PW} Q={Q} ({NC} dispatch cases).
#include "sconv_tiled.cuh"

namespace escoin {{

template <>
__device__ __forceinline__ void chunk_loop<{K}, {S}, {PH}, {PW}, {Q}, {TAG}>(float* acc, float* x, unsigned& p,
                                                                    unsigned wbase, unsigned rowb) {{
  asm volatile(
{body}
      : {outs}
      : {ins}
      : "memory");
}}

int launch_{name}(const TiledArgs& a, cudaStream_t s) {{
  return launch_tiled<{K}, {S}, {PH}, {PW}, {Q}, {MINB}, 0, {TAG}>(a, s);
}}

}}  // namespace escoin
"""


def main(outdir):
    os.makedirs(outdir, exist_ok=True)
    table = []
    for name, K, S, PH, PW, Q in VARIANTS:
        # suffix letters: r = full-row tiling, s = single dispatch site,
        # x = relative (small) jump tables, n = linked records
        last = name.split("_")[-1]
        sfx = "" if re.match(r"^\d+x\d+$", last) else last
        full_row, rel, link = "r" in sfx, "x" in sfx, "n" in sfx
        dm = re.search(r"x(\d+)$", sfx)  # "_nx8": relative tables with D = 8 successors
        rel_d = int(dm.group(1)) if dm else REL_D
        vec = (PW * S) % 4 == 0 or full_row
        if link:
            body, outs, ins = chunk_loop_link(K, S, PH, PW, Q, vec=vec, D=rel_d if rel else 0,
                                              depth=2 if "2" in sfx else 1)
        elif rel:
            body, outs, ins = chunk_loop_rel(K, S, PH, PW, Q, vec=vec, D=rel_d)
        else:
            body, outs, ins = chunk_loop(K, S, PH, PW, Q, vec=vec, single="s" in sfx)
        src = TEMPLATE.format(TAG=zlib.crc32(name.encode()) & 0x7fffffff, name=name, K=K, S=S, PH=PH, PW=PW, Q=Q, NC=Q * K * K, body=body, outs=outs, ins=ins,
                              MINB=min_blocks(K, S, PH, PW, Q))
        path = os.path.join(outdir, "variant_%s.cu" % name)
        if not os.path.exists(path) or open(path).read() != src:
            open(path, "w").write(src)
        table.append((name, K, S, PH, PW, Q, min_blocks(K, S, PH, PW, Q), 0, 1 if full_row else 0,
                      rel_d if rel else 0, 1 if link else 0))
    for name, K, S, PH, PW, Q in VARIANTS_MASK:
        body, outs, ins = bucket_mask(K, S, PH, PW, Q)
        src = TEMPLATE_MASK.format(TAG=zlib.crc32(name.encode()) & 0x7fffffff, name=name, K=K, S=S, PH=PH, PW=PW, Q=Q, NS=Q * K * K, body=body, outs=outs,
                                   ins=ins, MINB=min_blocks(K, S, PH, PW, Q))
        path = os.path.join(outdir, "variant_%s.cu" % name)
        if not os.path.exists(path) or open(path).read() != src:
            open(path, "w").write(src)
        table.append((name, K, S, PH, PW, Q, min_blocks(K, S, PH, PW, Q), 1, 0, 0, 0))
    for name, K, S, PH, PW, Q in VARIANTS_F2:
        body, outs, ins = chunk_loop2(K, S, PH, PW, Q)
        mb = min_blocks_f2(K, S, PH, PW, Q)
        src = TEMPLATE_F2.format(TAG=zlib.crc32(name.encode()) & 0x7fffffff, name=name, K=K, S=S, PH=PH, PW=PW, Q=Q, NC=Q * K * K, body=body, outs=outs,
                                 ins=ins, MINB=mb)
        path = os.path.join(outdir, "variant_%s.cu" % name)
        if not os.path.exists(path) or open(path).read() != src:
            open(path, "w").write(src)
        table.append((name, K, S, PH, PW, Q, mb, 2, 0, 0, 0))
    for name, K, S, PH, PW, Q in VARIANTS_P3:
        body, outs, ins = chunk_loop3(K, S, PH, PW, Q)
        mb = min_blocks_p3(K, S, PH, PW, Q)
        src = TEMPLATE_P3.format(TAG=zlib.crc32(name.encode()) & 0x7fffffff, name=name, K=K, S=S, PH=PH, PW=PW, Q=Q, NC=Q * K * K, body=body, outs=outs,
                                 ins=ins, MINB=mb)
        path = os.path.join(outdir, "variant_%s.cu" % name)
        if not os.path.exists(path) or open(path).read() != src:
            open(path, "w").write(src)
        table.append((name, K, S, PH, PW, Q, mb, 3, 0, 0, 0))
    for name, R, V in VARIANTS_1X1:
        mb = 2 if R * V <= 64 else 1
        sp = 1 if name.startswith("s1") else 0
        src = TEMPLATE_1X1.format(TAG=zlib.crc32(name.encode()) & 0x7fffffff, name=name, R=R, V=V, MINB=mb, SP=sp,
                                  kind="exact row lists" if sp else "row blocks")
        path = os.path.join(outdir, "variant_%s.cu" % name)
        if not os.path.exists(path) or open(path).read() != src:
            open(path, "w").write(src)
        table.append((name, 1, 1, 1, V, R, mb, 5 if sp else 4, 0, 0, 0))
    for name, K, PH, Q in VARIANTS_TAP:
        S = 2 if "s2" in name else 1
        src = TEMPLATE_TAP.format(TAG=zlib.crc32(name.encode()) & 0x7fffffff, name=name, K=K, S=S, PH=PH, Q=Q)
        path = os.path.join(outdir, "variant_%s.cu" % name)
        if not os.path.exists(path) or open(path).read() != src:
            open(path, "w").write(src)
        table.append((name, K, S, PH, 1, Q, 2, 6, 0, 0, 0))
    for name, K, PW, Q in VARIANTS_ROW:
        src = TEMPLATE_ROW.format(TAG=zlib.crc32(name.encode()) & 0x7fffffff, name=name, K=K, PW=PW, Q=Q)
        path = os.path.join(outdir, "variant_%s.cu" % name)
        if not os.path.exists(path) or open(path).read() != src:
            open(path, "w").write(src)
        table.append((name, K, 1, 1, PW, Q, 2, 7, 0, 0, 0))
    keep = set("variant_%s.cu" % t[0] for t in table)
    for f in os.listdir(outdir):
        if f.startswith("variant_") and f.endswith(".cu") and f not in keep:
            os.remove(os.path.join(outdir, f))
    decl = "\n".join("int launch_%s(const TiledArgs&, cudaStream_t);" % t[0] for t in table)
    rows = "\n".join('  {"%s", %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, &launch_%s},' % (t + (t[0],)) for t in table)
    inc = "// GENERATED by gen_sconv.py — do not edit.\n%s\nstatic const TiledVariant kTiledVariants[] = {\n%s\n};\n" % (
        decl, rows)
    path = os.path.join(outdir, "variants_table.inc")
    if not os.path.exists(path) or open(path).read() != inc:
        open(path, "w").write(inc)
    return [os.path.join(outdir, "variant_%s.cu" % t[0]) for t in table]


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "generated"))
