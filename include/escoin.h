/*
 * escoin.h — C-ABI of the B200-native Escoin direct sparse convolution
 * (arXiv 1802.10280, "Escort"/"Escoin").
 *
 * The two calls of the method (BASELINE.json north_star):
 *   escoin_csr_stretch   — CSR build + weight stretching, run once per layer
 *                          (P:310-322 CSR format, P:437-442 weight stretching)
 *   escoin_sconv_forward — direct sparse convolution with dynamic indexing
 *                          (Alg.2, §3.1), bias + ReLU fused
 * plus handle management around them.  Citations "P:n" are lines of the
 * paper text; "R#n" are the readings listed in DESIGN.md.
 *
 * Conventions (all functions):
 *   - Return an escoin_status (0 = OK, < 0 = error).  No C++ exception or
 *     CUDA error ever crosses the ABI; nothing is printed.
 *   - Pointers are plain host or device pointers as stated per argument;
 *     "device" means memory of the CUDA device the handle lives on.
 *   - cuda_stream is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  All device work is asynchronous on that stream.
 *   - Tensors are fp32, row-major NCHW ("CHW layout"; batch outermost).
 *   - Weights are square K x K filters, one stride, symmetric zero padding
 *     (SPEC non-goals S:103: no dilation, no non-square shapes).
 */
#ifndef ESCOIN_H_
#define ESCOIN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ESCOIN_OK = 0,
  ESCOIN_ERR_NULL = -1,          /* a required pointer argument is NULL */
  ESCOIN_ERR_SHAPE = -2,         /* a dim < 1, stride < 1, pad < 0, or E < 1 / F < 1 */
  ESCOIN_ERR_CSR_MISMATCH = -3,  /* forward shape != shape recorded in the handle, or CSR arrays inconsistent */
  ESCOIN_ERR_NOT_ON_DEVICE = -4, /* forward on a handle with no device copy, or device mismatch */
  ESCOIN_ERR_OVERFLOW = -5,      /* nnz, C*Hp*Wp or an index exceeds INT32_MAX */
  ESCOIN_ERR_UNSUPPORTED = -6,   /* no compiled kernel for this (K, stride) / kernel id out of range */
  ESCOIN_ERR_ALLOC = -7,         /* host or device allocation failed */
  ESCOIN_ERR_CUDA = -8           /* a CUDA runtime call or kernel launch failed */
} escoin_status;

/* Opaque handle: one pruned, stretched CONV layer.  Immutable once on the
 * device, so concurrent forwards on different streams are safe. */
typedef struct escoin_csr escoin_csr;

/* ---------------------------------------------------------------- stretch
 * Build the stretched CSR of one layer from its dense pruned weights.
 *   w      host, caller-owned, read-only, not retained: [M][C][K][K] fp32.
 *          Grouped convolutions pass the block-diagonal expansion (C = all
 *          input channels, zeros outside the group; reading R#18).
 *   M,C    output / input channels; H, W the UNPADDED input extent;
 *   K      square filter size; stride, pad as in the forward.
 * Semantics (readings R#3-R#7):
 *   - entries with w != 0.0f are kept (+0 and -0 dropped), row m in order,
 *     inside a row ascending (c, kh, kw) — equivalently ascending colidx;
 *   - colidx = c*Hp*Wp + kh*Wp + kw with Hp = H + 2*pad, Wp = W + 2*pad
 *     (the offset f(c, kh, kw) into the padded input);
 *   - rowptr[M+1] prefix counts (int32); value copied bitwise.
 *   stride is used only to validate E, F >= 1 and is recorded in the handle
 *   (M is added to the north_star signature, reading R#8).
 * On success *out owns host copies of rowptr/colidx/value (no device memory
 * yet).  Errors: NULL, SHAPE, OVERFLOW (nnz or C*Hp*Wp > INT32_MAX), ALLOC. */
int escoin_csr_stretch(const float* w, int M, int C, int H, int W, int K, int stride, int pad,
                       escoin_csr** out);

/* Same stretch computed ON THE DEVICE (NEXT-4): d_w is a device pointer to
 * the dense pruned weights [M][C][K][K] fp32 (caller-owned, read-only, not
 * retained).  Count / scan / order-preserving compaction kernels on
 * cuda_stream; the result is bit-identical to escoin_csr_stretch.  The handle
 * owns the device CSR, also keeps host copies (one D2H), and is returned
 * already on `device` (derived format built).  Synchronous.
 * Errors: NULL, SHAPE, OVERFLOW, ALLOC, CUDA. */
int escoin_csr_stretch_device(const float* d_w, int M, int C, int H, int W, int K, int stride, int pad,
                              int device, void* cuda_stream, escoin_csr** out);

/* Shape and nnz recorded in the handle (any output pointer may be NULL). */
int escoin_csr_info(const escoin_csr* csr, int* M, int* C, int* H, int* W, int* K, int* stride,
                    int* pad, int64_t* nnz);

/* Borrow the handle's host arrays (valid until escoin_csr_free): rowptr[M+1],
 * colidx[nnz], value[nnz].  For bit-exact checks of the stretch.  A handle
 * made by escoin_csr_wrap_device has host copies too (copied at wrap time). */
int escoin_csr_host_arrays(const escoin_csr* csr, const int32_t** rowptr, const int32_t** colidx,
                           const float** value);

/* Upload the CSR to `device` and build the kernel-side derived format
 * (DS-6: records bucketed by output-channel group and input channel; built
 * once from the stretched CSR, never part of the bit-exact contract).
 * Synchronises cuda_stream before returning.  Idempotent.
 * Errors: NULL, CUDA, ALLOC. */
int escoin_csr_to_device(escoin_csr* csr, int device, void* cuda_stream);

/* Make a handle around device CSR arrays that already hold a stretched CSR
 * (e.g. received by an NCCL broadcast on another rank).  The arrays are
 * BORROWED: the caller keeps them alive and unmodified while the handle
 * lives.  The handle copies them to the host once (synchronously on
 * cuda_stream) and builds its own derived format on `device`.
 * Errors: NULL, SHAPE, CSR_MISMATCH (rowptr[0] != 0, rowptr[M] != nnz, a
 * decreasing rowptr, or a colidx outside [0, C*Hp*Wp)), OVERFLOW, CUDA, ALLOC. */
int escoin_csr_wrap_device(const int32_t* d_rowptr, const int32_t* d_colidx, const float* d_value,
                           int64_t nnz, int M, int C, int H, int W, int K, int stride, int pad,
                           int device, void* cuda_stream, escoin_csr** out);

/* Free host memory and every device allocation the handle owns.  NULL-safe.
 * Synchronises the device first (pending forwards may still read it). */
void escoin_csr_free(escoin_csr* csr);

/* ---------------------------------------------------------------- forward
 * out[n][m][oh][ow] = act( bias[m] + sum_{j in row m} value[j] *
 *                          X~[n][colidx[j] + oh*stride*Wp + ow*stride] )
 * with X~ the zero-padded input (Alg.2 P:389-410 with stride, reading R#1;
 * padding virtual, R#9), act = ReLU if relu else identity, E/F from
 * E = (H + 2 pad - K)/stride + 1.
 *   in    device, [N][C][H][W] fp32, UNPADDED (padding is synthesised on chip).
 *   out   device, [N][M][E][F] fp32; must not alias in.
 *   bias  device [M] fp32, or NULL (= 0).      relu  0 or 1.
 * Shape args must equal those recorded in the handle (else CSR_MISMATCH);
 * N may be 0 (no-op).  Asynchronous on cuda_stream; no host sync, no
 * allocation, no workspace.  Returns the launch status; device faults
 * surface at the caller's next synchronisation.
 * Numerics: fp32 FMA accumulation from 0 in ascending colidx order per output
 * channel, then + bias, then ReLU (reading R#10/R#22; no fast-math).
 * Deterministic: bitwise identical for the same inputs whatever N, the grid,
 * the kernel variant or the number of GPUs the batch is sharded over. */
int escoin_sconv_forward(int N, int C, int H, int W, int M, int K, int stride, int pad,
                         const escoin_csr* csr, const float* in, float* out, const float* bias,
                         int relu, void* cuda_stream);

/* End-to-end variant for HOST buffers (bench e2e leg): copies h_in
 * ([N][C][H][W], host; pinned for asynchrony) to d_in, runs the forward into
 * d_out, copies d_out back to h_out ([N][M][E][F], host).  d_in / d_out are
 * caller-provided device scratch of those sizes; bias is a DEVICE pointer or
 * NULL.  Asynchronous on cuda_stream when the host buffers are pinned. */
int escoin_sconv_forward_hostio(int N, int C, int H, int W, int M, int K, int stride, int pad,
                                const escoin_csr* csr, const float* h_in, float* h_out,
                                float* d_in, float* d_out, const float* bias, int relu,
                                void* cuda_stream);

/* ---------------------------------------------------------------- kernel variants
 * "Kernel customization" (§3.4): the compiled variants of the
 * sconv kernel.  Variant 0 is the paper's own mapping (one CTA per (image,
 * output channel), one thread per output element, CSR row in shared memory,
 * inputs through the read-only cache, P:491-500 / P:541-556) and accepts
 * every (K, stride).  The other variants are register-tiled sm_100a kernels
 * specialised for one (K, stride).  ESCOIN_KERNEL_AUTO lets the library pick.
 * All variants compute bitwise-identical outputs. */
#define ESCOIN_KERNEL_AUTO (-1)
int escoin_kernel_count(void);
/* Name and (K, stride) of variant id; K = stride = 0 for "any". Strings are static. */
int escoin_kernel_info(int id, const char** name, int* K, int* stride);
/* Select the variant used by this handle's forwards (rebuilds the derived
 * format if needed; synchronous).  Errors: NULL, UNSUPPORTED, CUDA, ALLOC. */
int escoin_csr_set_kernel(escoin_csr* csr, int id);
/* The variant the handle currently uses (after AUTO resolution). */
int escoin_csr_get_kernel(const escoin_csr* csr, int* id);

/* Measured kernel customization (§3.4 P:563-564 "the optimization space we
 * explore includes the grid shape and thread block size"): time every
 * compiled variant that accepts the handle's (K, stride) — including the
 * paper mapping and every specialised kernel compiled by escoin_csr_jit —
 * and, per variant, its best four modelled tilings (CTA
 * shape, mosaic width, channel chunk), on the caller's buffers (same meaning as
 * escoin_sconv_forward; `out` is overwritten), `reps` timed forwards each
 * after one warm-up, and keep the fastest.  Synchronous on cuda_stream.
 * *best_id (may be NULL) receives the chosen variant, *best_ms its mean time.
 * All variants give bitwise-identical outputs, so this never changes results.
 * Errors: as escoin_sconv_forward, plus CUDA/ALLOC from the rebuilds. */
int escoin_csr_autotune(escoin_csr* csr, int N, const float* in, float* out, const float* bias, int relu,
                        int reps, void* cuda_stream, int* best_id, float* best_ms);
/* escoin_csr_autotune under the caller's measurement conditions:
 *   flush_buf / flush_bytes  device scratch (or NULL / 0) memset before EVERY timed rep, outside the
 *              timing events, so candidates are timed with a cold L2 like a flushed benchmark step
 *              (give >= 2x the L2 size, e.g. 256 MB on B200);
 *   flags      ESCOIN_TUNE_VARIANTS (the compiled variants and the paper mapping) and/or
 *              ESCOIN_TUNE_JIT (every specialised kernel compiled by escoin_csr_jit).
 * Each candidate: one warm-up forward, then `reps` single forwards each between its own events;
 * the candidate's time is the median (*best_ms).  The label of the winner is
 * escoin_csr_kernel_label.  Errors: as escoin_csr_autotune; NULL (flush_bytes > 0, no buffer),
 * UNSUPPORTED (no flag, or no candidate). */
#define ESCOIN_TUNE_VARIANTS 1
#define ESCOIN_TUNE_JIT 2
int escoin_csr_autotune_ex(escoin_csr* csr, int N, const float* in, float* out, const float* bias, int relu,
                           int reps, void* cuda_stream, void* flush_buf, int64_t flush_bytes, int flags,
                           int* best_id, float* best_ms);
/* Full label of the handle's current kernel, every tunable included, into buf (NUL-terminated,
 * truncated to cap): specialised kernels "jit_q<Q>_p<P>_cc<CC>_ns<NS>_w<warps>_b<CTAs/SM>_pf<prefetch>
 * _mb<mbarrier>_u<units>_sw<staged row stride>", variants "<name>_wm.._wp.._nb.._tr.._cc.._ns.._mos.._scs..",
 * "paper_mapping".  Errors: NULL; OVERFLOW if truncated. */
int escoin_csr_kernel_label(const escoin_csr* csr, char* buf, int cap);

/* ---------------------------------------------------------------- pattern-specialised kernel
 * Kernel customisation (§3.4) taken to the layer's weights: the
 * paper specialises its kernel per filter size / ofmap size / batch / stride
 * with C++ templates; weights are fixed once stretched ("only run once",
 * P:437-442), so this call compiles the handle's nonzero PATTERN and VALUES
 * into a kernel (generated PTX, one `fma.rn.f32 acc, x, <weight>, acc` per
 * nonzero and output pixel, compiled in-process for sm_100a and loaded into
 * the current context).  Results are bitwise identical to every other variant
 * (same fp32 terms in the same ascending (c, kh, kw) order, R#10).
 *   n_hint     batch size the mosaic geometry is planned for (<= 0: 128);
 *              forwards accept any N.
 *   tunables   NULL or ntunables (<= 18) ints {Q output channels per CTA,
 *              P pixels per lane, CC channels per stage, NS stages, warps per
 *              CTA, CTAs per SM, instruction-prefetch pass (< 0 = off),
 *              mbarrier pipeline (> 0 = on: warps drift up to NS-2 chunks
 *              instead of one CTA barrier per chunk), units (separately
 *              compiled modules the output-channel groups are split into,
 *              compiled in parallel host threads (relocatable)
 *              and linked into one kernel; <= 0: one per 500k nonzeros or 1536 chunk blocks,
 *              <= 32), vec (input words per staging copy: <= 0 = the widest
 *              the input row allows, 4 / 2 / 1), reorder (output
 *              channels regrouped so every group of Q rows holds about the
 *              same number of nonzeros — load balance under skewed per-row
 *              sparsity: 0 = when the heaviest group of
 *              consecutive rows exceeds the mean by > 5%, > 0 always, < 0
 *              never; results are bitwise identical either way), sws (row
 *              stride of the staged input in words: 0 = W + 2*pad, < 0 =
 *              the bank-conflict model's pick (larger strides spread a
 *              warp's lanes over the 32 shared-memory banks), > 0 = this),
 *              perm (> 0: lanes take the tile's pixels dealt by shared-
 *              memory bank instead of consecutively — conflict-free window
 *              loads — and the accumulators are transposed through shared
 *              memory for coalesced stores; same bits), split (> 1: the
 *              CTA's warps form that many independent sub-tiles, each with
 *              its own stage ring and named barrier, all running the same
 *              m-group's code — one sub-tile's barrier wait is covered by the
 *              others' work), pair (> 0 or 0 = default: with P even, pixel
 *              slots j, j+1 of a lane share one fma.rn.f32x2 per nonzero —
 *              two exact fp32 FMAs, the weight an immediate broadcast to both
 *              halves — halving the issued FMA instructions and the code
 *              bytes; < 0: one fma.rn.f32 per slot; same bits either way),
 *              hp (> 0, stride 1, K <= 5, P even, FFMA2 on: a lane's pixel
 *              pairs are horizontal neighbours (ow, ow+1) of one output row,
 *              whose taps of one filter row are K+1 consecutive staged words
 *              read with 8-byte ld.shared.v2 — fewer shared-memory loads;
 *              1 = pair alignment by rule, 2 = pairs (2i-pad%2, 2i+1-pad%2)
 *              keeping vector staging; same bits), pw (> 0: one extra warp
 *              per CTA runs the output-channel group's code one chunk ahead
 *              of the compute warps on stale data — no copies, no stores —
 *              so their instruction fetches hit the L1.5 cache; replaces the
 *              prefetch pass; not with mbarrier / split / perm / units > 1;
 *              same bits; measured slower, r02y),
 *              ks (> 1: each output-channel group's input channels are
 *              split into ks contiguous chunk ranges, one CTA each, for
 *              layers with too few CTAs (small planes, few output channels):
 *              partial sums go to a workspace owned by the handle ([ks][N][M]
 *              [E][F] fp32, allocated by the first forward that needs it —
 *              run one forward before capturing a graph) and a reduce kernel
 *              adds them in a fixed order, then bias and ReLU.  Deterministic
 *              and independent of the batch slice, within the R#11 tolerance,
 *              but NOT bitwise equal to the one-range kernels; < 0: as many
 *              parts as fill one wave of 148 x CTAs/SM, 1 if the grid does;
 *              <= -2: the same, but UNSUPPORTED when no split is needed — a
 *              tuning list entry that only compiles where it splits)};
 *              <= 0 entries take the defaults.
 * Compilation uses at most ESCOIN_JIT_THREADS (default: all host cores) concurrent
 * compiler threads across the process; if the environment variable ESCOIN_JIT_CACHE
 * names a writable directory, cubins are stored there keyed by a hash of their PTX
 * and reused by later calls and other processes (the ranks of a node compile once).
 * On success the new kernel is added to the handle's specialised kernels
 * and selected (the handle's kernel becomes ESCOIN_KERNEL_JIT); earlier ones
 * stay compiled until escoin_csr_free, and escoin_csr_autotune times all of
 * them.  Thread-safe per handle (several tunings may compile concurrently);
 * not concurrent with forwards on the same handle.  Compile time grows with
 * nnz (about 45 s for 180k nonzeros on one host core).  Filters up to 11x11,
 * any stride and padding (K > 11 returns UNSUPPORTED).
 * Errors: NULL, NOT_ON_DEVICE, UNSUPPORTED (shape, tunables, compile), CUDA (load). */
#define ESCOIN_KERNEL_JIT 1000
int escoin_csr_jit(escoin_csr* csr, int n_hint, const int* tunables, int ntunables);
/* Parameters of the handle's specialised kernel: tunables6 (6 ints, as above,
 * defaults resolved), units, registers per thread (max over units), cubin bytes
 * (sum over units).  Any output pointer may be NULL.  Errors: NULL, UNSUPPORTED
 * (no specialised kernel). */
int escoin_csr_jit_info(const escoin_csr* csr, int* tunables6, int* units, int* regs, int64_t* code_bytes);
/* Build statistics of the handle's selected specialised kernel: units, units loaded from
 * ESCOIN_JIT_CACHE, wall seconds of the build (generate + compile + load), PTX bytes.  Any
 * output pointer may be NULL.  Errors: NULL, UNSUPPORTED (no specialised kernel). */
int escoin_csr_jit_stats(const escoin_csr* csr, int* units, int* cache_hits, double* compile_s,
                         int64_t* ptx_bytes);

/* ---------------------------------------------------------------- engine selection
 * "Specifically optimized for convolutions in certain parts of the parameter space" (§3.4,
 * P:558-560): below some sparsity a dense tensor-core convolution of the pruned weights
 * (zeros included) is faster than the direct sparse kernel.  Deterministic rule
 * (SPEC select_engine): SPARSE when sparsity = 1 - nnz/(M*C*K*K) >= threshold
 * (ties -> SPARSE), else DENSE_TC.  The default threshold is the measured crossover of this
 * library's two engines on B200 (profiles/*density_sweep*), overridable per call
 * or process-wide with ESCOIN_SPARSE_THRESHOLD=<0..1>.  Grouped layers count the zeros of the
 * block-diagonal expansion (the dense engine computes them).
 * ESCOIN_KERNEL_DENSE_TC selects the dense engine on a handle (escoin_csr_set_kernel): the
 * handle's CSR is scattered back into dense [M][C][K][K] weights on its device (kept until
 * free) and forwards run the tcgen05 3xTF32 implicit GEMM (FP32-level accuracy, within the
 * method's 1e-5*sum|w*x| tolerance; not bitwise equal to the sparse kernels). */
#define ESCOIN_ENGINE_SPARSE 0
#define ESCOIN_ENGINE_DENSE_TC 1
#define ESCOIN_KERNEL_DENSE_TC 2000
#define ESCOIN_DEFAULT_SPARSE_THRESHOLD 0.35
/* Active threshold: ESCOIN_SPARSE_THRESHOLD if set to a number in [0, 1], else the default. */
double escoin_sparse_threshold(void);
/* The rule; threshold outside [0, 1] (e.g. -1) = escoin_sparse_threshold().  Returns the
 * engine (>= 0) or SHAPE (< 0). */
int escoin_select_engine(int M, int C, int K, int64_t nnz, double threshold);
/* Apply the rule to a handle on its device: DENSE_TC -> escoin_csr_set_kernel(DENSE_TC);
 * SPARSE -> leaves the handle's sparse kernel (from DENSE_TC: back to AUTO).  *engine (may be
 * NULL) receives the decision.  Errors: NULL, as escoin_csr_set_kernel. */
int escoin_csr_select_engine(escoin_csr* csr, double threshold, int* engine);

/* ---- Benchmark-only comparison point (NOT the method; SURVEY 8(b) "escoin_bench_*",
 * north_star: "a dense tcgen05 implicit-GEMM is kept only as a measured comparison point").
 * Dense convolution of the pruned weights INCLUDING their zeros on the 5th-generation
 * tensor cores: out = act(conv(in, w) + bias), implicit im2col, virtual padding.
 *   w     device fp32 [M][C][K][K] dense (block-diagonal expanded for grouped layers);
 *   in    device fp32 [N][C][H][W]; out device fp32 [N][M][E][F]; bias device [M] or NULL.
 *   nsplit 1: TF32 operands (~1e-3 relative error; NOT within the method's tolerance);
 *          3: 3xTF32 split (hi*hi + hi*lo + lo*hi), FP32-level accuracy.
 * Asynchronous on cuda_stream, no allocation.  Errors: NULL, SHAPE, UNSUPPORTED (nsplit), CUDA. */
int escoin_bench_dense_tc_forward(int N, int C, int H, int W, int M, int K, int stride, int pad, const float* w,
                                  const float* in, float* out, const float* bias, int relu, int nsplit,
                                  void* cuda_stream);

const char* escoin_status_string(int status);
/* Library version string, e.g. "escoin-b200 0.1 sm_100a". */
const char* escoin_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ESCOIN_H_ */
