// jit_sconv.h — pattern-specialised sconv kernels (jit_sconv.cpp). Internal, not ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace escoin {

struct JitPlan {
  // tunables (<= 0: default)
  int Q = 0;      // output channels per CTA (rows of one m-group)
  int P = 0;      // pixels per lane (slots 32 apart)
  int CC = 0;     // input channels per pipeline stage
  int NS = 0;     // pipeline stages
  int warps = 0;  // warps per CTA
  int minb = 0;   // CTAs per SM the register budget is compiled for
  int pf = 0;     // instruction prefetch pass: 0 = default (on), < 0 = off
  int mb = 0;     // > 0: mbarrier pipeline (warps drift up to NS-2 chunks) instead of a CTA barrier per chunk
  int split = 0;    // > 1: CTA = `split` independent sub-tiles (own stage ring + named barrier), same m-group
  int perm = 0;     // > 0: lane -> pixel deal by shared-memory bank (perm_table), accumulators transposed via smem
  int reorder = 0;  // output-channel grouping: 0 = balance groups by nonzeros if skewed, > 0 always, < 0 never
  int sws = 0;    // staged row stride request (0: W + 2*pad rounded to V; < 0: bank-conflict model; > 0: this)
  int vec = 0;    // staging vector width request (<= 0: widest the input row allows; 1 = 4-byte copies)
  int units = 0;  // separately compiled modules the m-groups are split into (<= 0: by nnz, jit_build)
  int pair = 0;   // > 0: slot pairs (j, j+1) share one fma.rn.f32x2 (FFMA2, weight immediate broadcast) — needs
                  // P even; 0 = default (on when P is even), < 0 = one fma.rn.f32 per slot
  int pw = 0;     // > 0: one extra "prefetch warp" per CTA walks the m-group's code one chunk ahead of the compute
                  // warps (garbage data, no copies, no stores) so their instruction fetches hit the L1.5 cache
                  // (straight-line barrier mode only; not with split / deal / mbarrier)
  int ks = 0;     // > 1: the group's channel chunks are split into ks contiguous ranges (split points on multiples of
                  // NS), one CTA each (grid z); partial sums go to a workspace and a reduce kernel adds them in
                  // z order + bias + ReLU — deterministic, within R#11, NOT bitwise equal to the one-range kernels
  int hp = 0;     // > 0: horizontal pixel pairs (stride 1, K <= 5, P even): a lane's pixel pair is (ow, ow+1) of one
                  // row, its taps come from ld.shared.v2 (K+1 words per filter row instead of 2K); 1 = pair origin
                  // parity by rule, 2 = origins at odd columns kept for vector staging
  // layer
  int C = 0, H = 0, W = 0, M = 0, K = 0, pad = 0, E = 0, F = 0, S = 1;
  // derived
  int mos = 1;    // images per staged row: always 1 (stacked layout, jit_sconv.cpp header)
  int SWs = 0;    // super-image row stride (words)
  int T = 0;      // slots per CTA
  int L = 0, Ls = 0;  // staged words per channel (and padded stride)
  int V = 1, Lv = 0;  // staging vector width (words per cp.async) and V-chunks per channel
  int nphase = 0;     // tile phases of the lane -> pixel deal (0 = off)
  int sp = 1;         // sub-tiles per CTA in effect (split)
  int f2 = 0;         // FFMA2 slot pairs in effect (pair)
  // items: what a lane slot holds — a pixel, or (hp) a horizontal pixel pair.  Item (n, oh, i) of a row of Fi
  // items has its window origin at stacked column i*cs + co; Pi items per lane (P, or P/2 pairs)
  int Fi = 0, cs = 1, co = 0, Pi = 1;
  int cpr = 0, rows_win = 0;  // data chunks per input row, stacked rows a window touches
  int KS = 0;     // staging slots per thread
  int nmg = 0, nch = 0;
  int smem_bytes = 0;
};

// One separately compiled unit: the code of m-groups [g_lo, g_hi).  Several units are compiled
// in parallel as relocatable device functions and linked behind one entry kernel (one launch).
struct JitUnit {
  int g_lo = 0, g_hi = 0;
  int64_t nnz = 0;
  size_t ptx_bytes = 0, cubin_bytes = 0;
  bool cache_hit = false;
};

struct JitModule {
  JitPlan plan;
  std::vector<JitUnit> units;
  void* module = nullptr;          // CUmodule
  void* func = nullptr;            // CUfunction escoin_jit_sconv
  int regs = 0;
  int local_bytes = 0;             // local memory per thread (call-saved registers of linked units)
  size_t ptx_bytes = 0, cubin_bytes = 0;
  double compile_s = 0.0;          // wall time of jit_build (all units, parallel)
  int cache_hits = 0;              // units loaded from ESCOIN_JIT_CACHE instead of compiled
  bool reordered = false;          // output channels regrouped for load balance (row_order)
  void* d_perm = nullptr;          // device lane -> pixel deal table (uint16 [nphase][T]) or null
  float* d_ws = nullptr;           // split-channel partial sums (ks > 1): [ks][N][M][E][F]
  int64_t ws_elems = 0;
};

// 0 = supported (plan filled), < 0 = this layer has no JIT form (stride != 1, 2*pad != K-1, smem).
int jit_plan(JitPlan& p, int C, int H, int W, int M, int K, int stride, int pad, int n_hint, double density);
// Generate, compile (units in parallel host threads, bounded by ESCOIN_JIT_THREADS or the
// host's cores; cubins reused from / stored in the directory ESCOIN_JIT_CACHE when set) and
// load; 0 = OK. log receives the compiler error log on failure.
int jit_build(JitModule& jm, const JitPlan& p, const int32_t* rowptr, const int32_t* colidx, const float* value,
              std::string* log);
// Host only (no device): generate, compile and (several units) link the cubin jit_build loads.
int jit_cubin(JitModule& jm, const JitPlan& p, const int32_t* rowptr, const int32_t* colidx, const float* value,
              std::vector<char>* cubin, std::string* log);
// The m-group ranges of the units jit_build would compile (balanced by nonzeros).
std::vector<std::pair<int, int>> jit_units(const JitPlan& p, const int32_t* rowptr);
// PTX of one unit (m-groups [g_lo, g_hi); g_hi <= 0: all groups).
std::string jit_ptx_text(const JitPlan& p, const int32_t* rowptr, const int32_t* colidx, const float* value,
                         int g_lo = 0, int g_hi = 0);
// Human-readable label of the plan, every tunable included (e.g. "jit_q32_p1_cc8_ns3_w32_b1_pf1_mb0_u4_sw15").
std::string jit_label(const JitModule& jm);
void jit_free(JitModule& jm);
// Compile PTX for sm_100a in-process without loading it (host only); 0 = OK.
int jit_compile_only(const char* ptx, size_t* cubin_bytes);
// ks > 1: writes the partial sums to ws ([ks][N][M][E][F], caller-sized) instead of out; the caller reduces.
int jit_launch(const JitModule& jm, const float* in, float* out, const float* bias, int relu, int N,
               cudaStream_t s, float* ws = nullptr);

}  // namespace escoin
