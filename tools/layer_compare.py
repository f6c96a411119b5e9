"""Per-layer comparison of the sparse path with the library baselines from bench.py JSON lines.

usage: python tools/layer_compare.py BENCH.json [...]
north_star: "beats im2col+cuBLAS and im2col+cuSPARSE on every pruned layer at batch 128".
"""
import json
import sys

KEYS = [("im2col+cublas_sgemm", "cuBLAS/img"), ("im2col+cublas_sgemm_one_gemm_per_batch", "cuBLAS 1 GEMM"),
        ("im2col+cusparse_spmm", "cuSPARSE"), ("cudnn_fp32_dense", "cuDNN FP32"),
        ("cudnn_tf32_dense_tensorcore", "cuDNN TF32")]


def main(paths):
    for p in paths:
        d = json.load(open(p))
        bl = d.get("baselines", {})
        print("### %s" % d["config"]["workload"])
        print()
        print("| layer | escoin ms | " + " | ".join("%s ms (speedup)" % n for _, n in KEYS) + " |")
        print("|---" * (2 + len(KEYS)) + "|")
        wins = {k: 0 for k, _ in KEYS}
        for l in d["layers"]:
            cells = []
            for k, _ in KEYS:
                ms = bl.get(k, {}).get("ms_per_layer", {}).get(l["layer"])
                if ms is None:
                    cells.append("—")
                    continue
                sp = ms / l["ms"]
                wins[k] += sp > 1.0
                cells.append("%.4f (%.2f×)" % (ms, sp))
            print("| %s | %.4f | %s |" % (l["layer"], l["ms"], " | ".join(cells)))
        n = len(d["layers"])
        print()
        print("escoin faster on: " + ", ".join("%s %d/%d layers" % (nm, wins[k], n) for k, nm in KEYS))
        print()


if __name__ == "__main__":
    main(sys.argv[1:])
