/*
 * escoin_oracle.c — CPU ORACLE for the Escoin direct sparse convolution.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the plain, slow, obviously
 * correct reference the CUDA path is checked against.  Only tests/,
 * __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
 * `--impl reference`) may load it.  The product library
 * (paper_1802_10280_b200/, libescoin.so) never includes, links or calls
 * anything in this directory, and this file includes nothing from there.
 *
 * Precision: every accumulation is in double (fp64).  A product of two
 * fp32 values is exact in fp64 (24+24 <= 53 mantissa bits).
 *
 * Citations: "P:n" is line n of the paper text (PAPER.md, arXiv 1802.10280),
 * "S:n" a line of SPEC.md.  Readings of ambiguous passages are numbered as in
 * SURVEY.md §8(c) and listed in DESIGN.md ("R#n").
 *
 * Parity pins (tests/test_oracle.py): every function below is pinned against
 * something other than itself — brute force (O-3 vs O-2), torch conv2d in
 * float64, closed forms, SPEC worked examples in tests/golden/, invariants.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ shapes
 * Output extent.  Eq.1 gives E = H - R + 1 for stride 1 and no pad;
 * the stride/pad generalisation is SPEC S:34 (reading R#1/R#2):
 *   E = floor((H + 2*pad - K)/stride) + 1.
 * Returns -1 when the shape is invalid (E < 1 or bad parameters). */
int oracle_output_dim(int H, int K, int stride, int pad) {
  if (H < 1 || K < 1 || stride < 1 || pad < 0) return -1;
  int span = H + 2 * pad - K;
  if (span < 0) return -1;
  return span / stride + 1;
}

/* Layout function f of §3.1: in CHW layout
 *   f(c, r, s) = (c * H_in + r) * W_in + s.
 * With H_in/W_in the PADDED extents (reading R#3). */
int64_t oracle_layout_f(int64_t c, int64_t y, int64_t x, int64_t Hin, int64_t Win) {
  return (c * Hin + y) * Win + x;
}

/* Thread count of the parallel loops (timing only: the per-output arithmetic does not depend on it). */
void oracle_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ O-1
 * Dense pruned weights -> CSR (§2.3, Fig.4) -> weight stretching
 * (§3.1).
 *
 * Step 1: "The data array value stores only the non-zero elements
 * row by row"; colidx[i] is the column of value[i]; rowptr[i] is the start of
 * row i in colidx, rowptr[i+1]-rowptr[i] its count.  Row m of the weight
 * matrix is filter m flattened in (c, r, s) order (the M x CRS matrix W of
 * §2.2), so the unstretched column is (c*K + r)*K + s.  "Non-zero"
 * means w != 0.0f (reading R#6).
 *
 * Step 2: "the weight matrix is stretched ... This operation only
 * modifies the column indices": the column (c, r, s) becomes the input offset
 * f(c, r, s) over the padded input, Hp = H + 2 pad, Wp = W + 2 pad (R#3/R#4).
 * rowptr and value are untouched.
 *
 * cap = capacity of colidx/value.  Returns 0 on success, -1 on bad shape,
 * -2 if cap is too small (nnz still written to *nnz_out). */
int oracle_csr_stretch(const float* w, int M, int C, int H, int W, int K, int stride, int pad,
                       int32_t* rowptr, int32_t* colidx, float* value, int64_t cap, int64_t* nnz_out) {
  if (M < 1 || C < 1) return -1;
  if (oracle_output_dim(H, K, stride, pad) < 1 || oracle_output_dim(W, K, stride, pad) < 1) return -1;
  const int64_t CRS = (int64_t)C * K * K;
  const int64_t Hp = H + 2 * pad, Wp = W + 2 * pad;
  /* step 1: dense -> CSR with unstretched columns */
  int64_t nnz = 0;
  rowptr[0] = 0;
  for (int m = 0; m < M; ++m) {
    for (int64_t col = 0; col < CRS; ++col) {
      float v = w[(int64_t)m * CRS + col];
      if (v != 0.0f) {
        if (nnz < cap) { colidx[nnz] = (int32_t)col; value[nnz] = v; }
        ++nnz;
      }
    }
    rowptr[m + 1] = (int32_t)nnz;
  }
  *nnz_out = nnz;
  if (nnz > cap) return -2;
  /* step 2: stretch — decode (c, r, s) from the CRS column, re-encode with f */
  for (int64_t j = 0; j < nnz; ++j) {
    int64_t col = colidx[j];
    int64_t s = col % K;
    int64_t r = (col / K) % K;
    int64_t c = col / ((int64_t)K * K);
    colidx[j] = (int32_t)oracle_layout_f(c, r, s, Hp, Wp);
  }
  return 0;
}

/* ------------------------------------------------------------------ padding
 * pad_in ("A 1-D array is used to hold the ifmaps, padded if
 * necessary"): X~[n][c][y][x] = X[n][c][y-p][x-p] inside, 0 outside. */
void oracle_pad_input(const float* in, int N, int C, int H, int W, int pad, double* out) {
  const int64_t Hp = H + 2 * pad, Wp = W + 2 * pad;
  for (int64_t nc = 0; nc < (int64_t)N * C; ++nc)
    for (int64_t y = 0; y < Hp; ++y)
      for (int64_t x = 0; x < Wp; ++x) {
        int64_t yi = y - pad, xi = x - pad;
        out[(nc * Hp + y) * Wp + x] =
            (yi >= 0 && yi < H && xi >= 0 && xi < W) ? (double)in[(nc * H + yi) * W + xi] : 0.0;
      }
}

/* ------------------------------------------------------------------ O-2
 * Algorithm 2 "Sequential Sparse Convolution", over the
 * materialised padded input, generalised with stride (reading R#1):
 *
 *   for n, for m, for j in [rowptr[m], rowptr[m+1]):
 *     off <- colidx[j]; val <- value[j]
 *     for h in [0,E), for w in [0,F):
 *       out[n][m][h][w] += val * in[n][off + f(0, h*s, w*s)]
 *
 * Accumulators start at 0; the epilogue (reading R#10) adds bias[m] and
 * applies ReLU if relu != 0.  scale[n][m][h][w] = sum |val * in| over the
 * same terms (reading R#21), the magnitude the tolerance is relative to.
 * Work is split over disjoint (n, m) pairs (OpenMP), each computed exactly as
 * the sequential loop nest, so the result is independent of thread count.
 * bias may be NULL (= 0).  out and scale are [N][M][E][F]; scale may be NULL. */
int oracle_sconv(int N, int C, int H, int W, int M, int K, int stride, int pad,
                 const int32_t* rowptr, const int32_t* colidx, const float* value,
                 const float* in, const float* bias, int relu, double* out, double* scale) {
  const int E = oracle_output_dim(H, K, stride, pad), F = oracle_output_dim(W, K, stride, pad);
  if (E < 1 || F < 1 || N < 0 || M < 1 || C < 1) return -1;
  const int64_t Hp = H + 2 * pad, Wp = W + 2 * pad;
  const int64_t img = (int64_t)C * Hp * Wp;
  const int64_t EF = (int64_t)E * F;
  double* xp = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1) * (size_t)img);
  if (!xp) return -3;
  oracle_pad_input(in, N, C, H, W, pad, xp);
  const int64_t NM = (int64_t)N * M;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t nm = 0; nm < NM; ++nm) {
    const int64_t n = nm / M, m = nm % M;
    double* o = out + nm * EF;
    double* sc = scale ? scale + nm * EF : NULL;
    for (int64_t i = 0; i < EF; ++i) { o[i] = 0.0; if (sc) sc[i] = 0.0; }
    const double* xn = xp + n * img;
    for (int64_t j = rowptr[m]; j < rowptr[m + 1]; ++j) {
      const int64_t off = colidx[j];
      const double val = (double)value[j];
      for (int64_t h = 0; h < E; ++h)
        for (int64_t w = 0; w < F; ++w) {
          const double t = val * xn[off + oracle_layout_f(0, h * stride, w * stride, Hp, Wp)];
          o[h * F + w] += t;
          if (sc) sc[h * F + w] += fabs(t);
        }
    }
    const double b = bias ? (double)bias[m] : 0.0;
    for (int64_t i = 0; i < EF; ++i) {
      double v = o[i] + b;
      o[i] = (relu && !(v > 0.0)) ? 0.0 : v;
    }
  }
  free(xp);
  return 0;
}

/* Same as oracle_sconv for an explicit list of output coordinates
 * (n, m, h, w) — used to check sampled outputs of full-size layers one by
 * one.  Unpadded input; padding applied per term (same definition as
 * oracle_pad_input).  coords is [npts][4]. */
int oracle_sconv_points(int N, int C, int H, int W, int M, int K, int stride, int pad,
                        const int32_t* rowptr, const int32_t* colidx, const float* value,
                        const float* in, const float* bias, int relu,
                        const int64_t* coords, int64_t npts, double* out, double* scale) {
  const int E = oracle_output_dim(H, K, stride, pad), F = oracle_output_dim(W, K, stride, pad);
  if (E < 1 || F < 1) return -1;
  const int64_t Hp = H + 2 * pad, Wp = W + 2 * pad;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < npts; ++i) {
    const int64_t n = coords[4 * i], m = coords[4 * i + 1], h = coords[4 * i + 2], w = coords[4 * i + 3];
    double acc = 0.0, sc = 0.0;
    if (n >= 0 && n < N && m >= 0 && m < M && h >= 0 && h < E && w >= 0 && w < F) {
      for (int64_t j = rowptr[m]; j < rowptr[m + 1]; ++j) {
        const int64_t idx = colidx[j] + oracle_layout_f(0, h * stride, w * stride, Hp, Wp);
        const int64_t c = idx / (Hp * Wp), y = (idx / Wp) % Hp - pad, x = idx % Wp - pad;
        const double xv = (y >= 0 && y < H && x >= 0 && x < W)
                              ? (double)in[((n * C + c) * H + y) * W + x] : 0.0;
        const double t = (double)value[j] * xv;
        acc += t;
        sc += fabs(t);
      }
      const double v = acc + (bias ? (double)bias[m] : 0.0);
      out[i] = (relu && !(v > 0.0)) ? 0.0 : v;
    } else {
      out[i] = NAN;
    }
    if (scale) scale[i] = sc;
  }
  return 0;
}

/* ------------------------------------------------------------------ O-3
 * Algorithm 1 "Sequential Convolution" / Eq.1: the
 * 7-deep loop nest over n, m, c, h, w, r, s on the DENSE pruned weights,
 * generalised with stride and zero padding (readings R#1/R#2):
 *   out[n][m][h][w] += in[n][c][h*s + r - p][w*s + q - p] * weight[m][c][r][q]
 * (terms falling in the padding read 0).  Brute force for tiny shapes. */
int oracle_conv_dense(int N, int C, int H, int W, int M, int K, int stride, int pad,
                      const float* weight, const float* in, const float* bias, int relu, double* out) {
  const int E = oracle_output_dim(H, K, stride, pad), F = oracle_output_dim(W, K, stride, pad);
  if (E < 1 || F < 1) return -1;
  for (int64_t i = 0; i < (int64_t)N * M * E * F; ++i) out[i] = 0.0;
  for (int n = 0; n < N; ++n)
    for (int m = 0; m < M; ++m)
      for (int c = 0; c < C; ++c)
        for (int h = 0; h < E; ++h)
          for (int w = 0; w < F; ++w)
            for (int r = 0; r < K; ++r)
              for (int s = 0; s < K; ++s) {
                const int y = h * stride + r - pad, x = w * stride + s - pad;
                const double iv = (y >= 0 && y < H && x >= 0 && x < W)
                                      ? (double)in[(((int64_t)n * C + c) * H + y) * W + x] : 0.0;
                out[(((int64_t)n * M + m) * E + h) * F + w] +=
                    iv * (double)weight[(((int64_t)m * C + c) * K + r) * K + s];
              }
  for (int64_t nm = 0; nm < (int64_t)N * M; ++nm) {
    const double b = bias ? (double)bias[nm % M] : 0.0;
    for (int64_t i = 0; i < (int64_t)E * F; ++i) {
      double v = out[nm * E * F + i] + b;
      out[nm * E * F + i] = (relu && !(v > 0.0)) ? 0.0 : v;
    }
  }
  return 0;
}
