"""Markdown tables from bench.py JSON lines (for DESIGN.md §10 / profiles/).

usage: python tools/bench_table.py BENCH.json [BENCH.json ...]
"""
import json
import sys

BL = [("im2col+cublas_sgemm", "cuBLAS/img"), ("im2col+cublas_sgemm_one_gemm_per_batch", "cuBLAS 1 GEMM"),
      ("im2col+cusparse_spmm", "cuSPARSE"), ("cudnn_fp32_dense", "cuDNN FP32"),
      ("cudnn_tf32_dense_tensorcore", "cuDNN TF32"), ("dense_tcgen05_3xtf32", "tcgen05 3xTF32"),
      ("escoin_paper_mapping", "paper mapping")]


def main(paths):
    rows = [json.load(open(p)) for p in paths]
    print("| workload | images/s | ms/step | stack TFLOP/s (frac of 74.45) | e2e images/s | dominant layer: kernel, frac | "
          + " | ".join("vs " + n for _, n in BL) + " | oracle (cores) |")
    print("|---" * (7 + len(BL)) + "|")
    for d in rows:
        st = d["roofline"].get("stack", {})
        bl = d.get("baselines", {})
        sp = []
        for k, _ in BL:
            v = bl.get(k, {})
            sp.append("%.2f×" % v["escoin_speedup"] if "escoin_speedup" in v else "—")
        cb = d.get("cpu_baseline") or {}
        print("| %s | %.0f | %.3f | %.1f (%.3f) | %.0f | %s: %s, %.3f | %s | %s |" % (
            d["config"]["workload"], d["value"], d["ms_per_step"], st.get("tflops_graph", 0), st.get("frac_graph", 0),
            d["e2e"]["value"], d["roofline"]["kernel"].split("(")[-1].rstrip(")"), d["roofline"]["kernel"].split()[1],
            d["roofline"]["frac"], " | ".join(sp),
            "%.1f (%s)" % (cb["value"], cb.get("cores")) if cb else "—"))
    print()
    for d in rows:
        print("%s per layer (ms, TFLOP/s, frac):" % d["config"]["workload"])
        print("; ".join("%s %.4f %.1f %.3f" % (l["layer"], l["ms"], l["tflops"], l["frac_fp32"]) for l in d["layers"]))
        print()


if __name__ == "__main__":
    main(sys.argv[1:])
