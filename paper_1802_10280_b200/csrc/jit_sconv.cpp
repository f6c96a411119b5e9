// jit_sconv.cpp — pattern-specialised direct sparse convolution (kernel
// customisation, §3.4, carried to its limit).
//
// The paper customises its kernel per (filter size, ofmap size, batch,
// stride) with C++ templates.  Weights are fixed once a layer is pruned and
// stretched ("only run once"), so this file goes one step further
// and compiles the layer's nonzero PATTERN and VALUES into the instruction
// stream: for every (output-channel group, input channel) the generated PTX
// loads the input taps the group uses from the shared-memory slab and issues
// one `fma.rn.f32 acc, x, <weight immediate>, acc` per (nonzero, pixel) — or,
// with P even, one `fma.rn.f32x2` (FFMA2, the weight broadcast as a 32-bit
// immediate) per (nonzero, pixel pair).  There is no per-nonzero dispatch, no
// record stream and no weight load at all (the weight is an immediate), which
// is what the register-tiled interpreter kernels (sconv_tiled.cuh) spend most
// of their issue slots on.
//
// Semantics are exactly escoin_sconv_forward's (Alg.2 P:389-410 with the
// stride/pad generalisation R#1, R#9, R#10): each accumulator starts at 0.0f
// and receives its CSR terms in ascending (c, kh, kw) = colidx order with
// fma.rn.f32, then acc + bias[m] and ReLU — bit-identical to every other
// variant (tested).  Exception: split channels (JitPlan::ks > 1) add per-range
// partial sums in a fixed order (deterministic, within R#11).
//
// Geometry: a CTA owns T consecutive output pixels g = (n*E + oh)*F + ow (tile
// blockIdx.y; lane l of warp w: g0 + (w*P + j)*32 + l, no idle lanes) and
// blockIdx.x selects the output-channel group of Q rows whose code it runs (the
// groups of a tile are consecutive CTAs: they share the tile's input through L2).  The input is staged in a stacked layout — images one above
// the other, separated by `pad` zero rows shared by neighbours, row stride
// SWs = W + 2*pad — where pixel g sits at pos(g) = (n*(H+pad) + oh)*SWs + ow and
// reads tap (kh, kw) at pos(g) + kh*SWs + kw: the stretched offset f(0, kh, kw)
// of P:428 with the stacked row stride, an immediate offset from the lane's
// base register.  Per pipeline stage CC channels of the window
// [pos(g0), pos(g0) + L) are staged: data chunks with 16/8/4-byte cp.async,
// the padding words zeroed once per CTA (the virtual padding, R#9).
//
// Compilation: PTX text -> nvPTXCompiler (static, in-process) -> cubin ->
// driver module (entry points via cudaGetDriverEntryPoint, so the library
// has no link-time dependency on libcuda).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvJitLink.h>
#include <nvPTXCompiler.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <dlfcn.h>
#include <unistd.h>
#include <string>
#include <vector>

#include "jit_sconv.h"

namespace escoin {
namespace {

typedef CUresult (*PFN_ModuleLoadData)(CUmodule*, const void*);
typedef CUresult (*PFN_ModuleGetFunction)(CUfunction*, CUmodule, const char*);
typedef CUresult (*PFN_ModuleUnload)(CUmodule);
typedef CUresult (*PFN_FuncSetAttribute)(CUfunction, CUfunction_attribute, int);
typedef CUresult (*PFN_FuncGetAttribute)(int*, CUfunction_attribute, CUfunction);
typedef CUresult (*PFN_LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                     unsigned, CUstream, void**, void**);

struct Driver {
  PFN_ModuleLoadData load = nullptr;
  PFN_ModuleGetFunction get = nullptr;
  PFN_ModuleUnload unload = nullptr;
  PFN_FuncSetAttribute setattr = nullptr;
  PFN_FuncGetAttribute getattr = nullptr;
  PFN_LaunchKernel launch = nullptr;
  bool ok = false;
};

template <typename T>
bool entry(const char* name, T* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p)
    return false;
  *fn = reinterpret_cast<T>(p);
  return true;
}

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry("cuModuleLoadData", &d.load) && entry("cuModuleGetFunction", &d.get) &&
           entry("cuModuleUnload", &d.unload) && entry("cuFuncSetAttribute", &d.setattr) &&
           entry("cuFuncGetAttribute", &d.getattr) && entry("cuLaunchKernel", &d.launch);
  });
  return d;
}

int cdiv(int a, int b) { return (a + b - 1) / b; }

constexpr int kMaxK = 11;  // largest filter with a specialised form (AlexNet conv1)

// ---------------------------------------------------------------- geometry
// Stacked staging layout: images one above the other, separated by `pad` shared zero rows, row
// stride SWs >= W + 2*pad (extra columns are zeros too); output pixel g = (n*E + oh)*F + ow has
// its window origin at pos(g) = (n*(H+pad) + oh*S)*SWs + ow*S and reads tap (kh, kw) at
// pos(g) + kh*SWs + kw — the stretched offset f(0, kh, kw) of P:428 with the stacked row stride.
// Items (hp): a lane slot holds item g = (n*E + oh)*Fi + i — a pixel (Fi = F, column i*S) or a horizontal
// pixel pair (ow, ow+1) = (2i + co, 2i + co + 1) (Fi pairs per row, co = 0 or -1) — with window origin at
// stacked column i*cs + co.
int64_t stacked_pos(const JitPlan& p, int sws, int64_t g) {
  const int64_t EF = int64_t(p.E) * p.Fi, n = g / EF, r = g % EF;
  return (n * (p.H + p.pad) + (r / p.Fi) * p.S) * sws + (r % p.Fi) * p.cs + p.co;
}

// Shared-memory wavefronts per warp-wide LDS (1 = conflict-free) of the lane -> pixel mapping
// (warp w, slot j, lane l -> pixel g0 + (w*P + j)*32 + l) for row stride sws: the mean over the
// first tiles of the n_hint-image grid of the largest number of lanes on one bank.
double lds_wavefronts(const JitPlan& p, int sws, int n_hint) {
  const int64_t EF = int64_t(p.E) * p.Fi, total = int64_t(std::max(1, n_hint)) * EF;
  const int64_t tiles = std::min<int64_t>((total + p.T - 1) / p.T, 12);
  double sum = 0;
  int64_t groups = 0;
  for (int64_t t = 0; t < tiles; ++t)
    for (int grp = 0; grp < p.T / 32; ++grp) {
      int cnt[32] = {};
      int mx = 0;
      for (int l = 0; l < 32; ++l) {
        const int64_t g = std::min(total - 1, t * p.T + grp * 32 + l);
        mx = std::max(mx, ++cnt[stacked_pos(p, sws, g) & 31]);
      }
      sum += mx;
      ++groups;
    }
  return groups ? sum / groups : 1.0;
}

void plan_geometry(JitPlan& p, int /*n_hint*/) {
  // horizontal pixel pairs: stride 1, filters up to 5x5 (one filter row of words live), P even, no deal
  const bool hp = p.hp > 0 && p.f2 && p.S == 1 && p.K <= 5 && p.P % 2 == 0 && p.perm <= 0;
  p.Pi = hp ? p.P / 2 : p.P;
  p.cs = hp ? 2 : p.S;
  const int T = p.warps * 32 * p.Pi;
  if (!hp) {
    p.co = 0;
    p.Fi = p.F;
  }
  p.mos = 1;
  p.T = T;
  // split > 1: the CTA's warps form `split` independent sub-tiles of T/split pixels (own stage
  // ring, own named barrier) running the same m-group's code
  p.sp = (p.split > 1 && !p.mb && p.perm <= 0 && p.warps % p.split == 0) ? p.split : 1;
  const int Th = T / p.sp;
  // Staging vector width: V input words per cp.async when an input row is a whole number of
  // V-word (16 / 8 byte) chunks (W % V == 0); with a row stride that is a multiple of V and a
  // per-CTA shift of the buffer (bo, gen_ptx) the data chunks are aligned in global AND shared
  // memory.  Only data chunks are copied: the padding words of the stage buffers are zeroed once
  // per CTA (they are the same positions for every channel and chunk).
  if (p.vec <= 0) p.V = p.W % 4 == 0 ? 4 : p.W % 2 == 0 ? 2 : 1;
  else p.V = (p.vec >= 4 && p.W % 4 == 0) ? 4 : (p.vec >= 2 && p.W % 2 == 0) ? 2 : 1;
  if (hp) {
    // Pair origins must be even words of the stage buffer (ld.shared.v2).  With vector staging the
    // first data word of a row (column pad) sits on a V-word boundary, so origins (column 2i + co)
    // are even iff co = pad mod 2 (co = -1: pairs (-1, 0), (1, 2), ...; a phantom pixel at -1).
    // co = 0 with an odd pad needs 4-byte staging.  hp = 1: co = 0 when F is even and the pad odd
    // only on planes up to 28 wide (no phantom column, 4-byte copies); else co = -(pad mod 2).
    const bool keep_v = p.pad % 2 == 0 || p.hp == 2 || p.F % 2 == 1 || p.F > 28;
    p.co = keep_v ? -(p.pad % 2) : 0;
    if (!keep_v) p.V = 1;
    p.Fi = (p.F - p.co + 1) / 2;
  }
  const int VA = hp && p.V == 1 ? 2 : p.V;  // row stride alignment (even for pairs)
  const int base = (p.W + 2 * p.pad + VA - 1) / VA * VA;
  p.SWs = p.sws > 0 ? std::max(base, (p.sws + VA - 1) / VA * VA) : base;
  const int EF = p.E * p.Fi;  // items per image
  int64_t span = 0;  // max pos(g0 + Th - 1) - pos(g0); periodic in g0 with period EF
  for (int64_t g0 = 0; g0 < EF; ++g0)
    span = std::max(span, stacked_pos(p, p.SWs, g0 + Th - 1) - stacked_pos(p, p.SWs, g0));
  p.L = int(span + int64_t(p.K - 1) * (p.SWs + 1) + 1 + (hp ? 2 : 0));  // pairs: one more column (+1: v2 of K odd)
  p.Lv = cdiv(p.L + p.V - 1, p.V);  // V-word chunks per channel (the window shifted by bo < V)
  p.Ls = (p.Lv * p.V + 3) & ~3;
  p.nmg = cdiv(p.M, p.Q);
  p.nch = cdiv(p.C, p.CC);
  p.cpr = p.W / p.V;                                  // data chunks per input row
  p.rows_win = (p.Lv * p.V + p.SWs - 1) / p.SWs + 1;  // stacked rows the window can touch
  p.KS = cdiv(p.rows_win * p.cpr, p.warps * 32 / p.sp);  // data-chunk slots per thread
  // + the m-group's Q bias values (staged once per CTA, read by the epilogue)
  p.smem_bytes = p.sp * p.NS * p.CC * p.Ls * 4 + (p.mb ? 128 : 0) + ((p.Q * 4 + 15) & ~15);
  // lane -> pixel deal (perm > 0): the bank pattern of a tile repeats every EF / gcd(T, EF) tiles
  p.nphase = 0;
  if (p.perm > 0) {
    int a = T, b = EF;
    while (b) { const int t = a % b; a = b; b = t; }
    const int64_t nph = EF / a;
    if (nph * T <= (int64_t(1) << 22) && T <= 65536) p.nphase = int(nph);
  }
}

// Geometry with the channel chunk halved until the stage ring fits shared memory (strided
// layers stage S*S times more input per output pixel).
bool plan_fit_sws(JitPlan& p, int n_hint) {
  for (;;) {
    plan_geometry(p, n_hint);
    if (p.smem_bytes <= 227 * 1024 / p.minb) return true;
    if (p.CC == 1) return false;
    p.CC = (p.CC + 1) / 2;
  }
}

// Row stride: the base W + 2*pad (rounded to V) unless requested.  sws < 0 asks for the
// bank-conflict model: a warp's 32 pixels wrap across row ends of the stacked layout, and with the
// base stride two of them land 32 words apart (2-way conflicts on most LDS, ncu r01z/r02b); among
// SWs = base .. base + 48 (multiples of V) take the fewest modelled wavefronts (ties: the smaller
// stride) that fits shared memory at the requested channel chunk.  Measured (r02f A/B): -4% time on
// ResNet res3 at 24 warps, +4% on res2 (the larger stage ring), neutral on res4/res5 — so it is an
// autotune candidate, not the default.
bool plan_fit(JitPlan& p, int n_hint) {
  if (p.sws >= 0) return plan_fit_sws(p, n_hint);
  JitPlan t = p;
  plan_geometry(t, n_hint);
  const int base = t.SWs;
  std::vector<std::pair<double, int>> cands;
  for (int sws = base; sws <= base + 48; sws += t.V)
    cands.emplace_back(std::round(lds_wavefronts(t, sws, n_hint) * 100.0) / 100.0, sws);
  std::sort(cands.begin(), cands.end());
  for (const auto& c : cands) {
    JitPlan q = p;
    q.sws = c.second;
    plan_geometry(q, n_hint);
    if (q.smem_bytes <= 227 * 1024 / q.minb) {
      q.sws = -1;  // keep the request "model" (plan equality compares SWs itself)
      p = q;
      return true;
    }
  }
  p.sws = 0;
  if (!plan_fit_sws(p, n_hint)) return false;
  p.sws = -1;
  return true;
}

// ---------------------------------------------------------------- PTX text
struct Out {
  std::string s;
  char buf[256];
  void operator()(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
    va_list ap;
    va_start(ap, fmt);
    va_list ap2;
    va_copy(ap2, ap);
    const int n = vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (n < int(sizeof buf)) {
      s.append(buf, n);
    } else {  // long line (branch-target lists)
      std::string big(size_t(n) + 1, '\0');
      vsnprintf(&big[0], big.size(), fmt, ap2);
      s.append(big.data(), n);
    }
    va_end(ap2);
    s.push_back('\n');
  }
};

struct Nz {
  int t, q;
  uint32_t bits;
};

// Lane -> pixel deal of the tiles (perm > 0), per tile phase ph (tile mod nphase): the T pixels of
// the tile sorted by the shared-memory bank of their window origin (pos(g) mod 32; every tap adds
// the same offset to all lanes, so the banks of any LDS are this pattern shifted) and dealt
// round-robin to the T/32 (warp, slot) groups: a group receives at most one pixel per bank unless a
// bank holds more than T/32 of the tile's pixels (row ends of the stacked layout make the
// consecutive-pixel assignment 2-way conflicted, ncu r01z/r02b).  table[ph*T + s*32 + l] = pixel
// offset in the tile of slot s = warp*P + j, lane l.
std::vector<uint16_t> perm_table(const JitPlan& p) {
  const int T = p.T, G = T / 32;
  std::vector<uint16_t> tab(size_t(p.nphase) * T);
  std::vector<int> idx(T);
  std::vector<int> bank(T);
  for (int ph = 0; ph < p.nphase; ++ph) {
    const int64_t g0 = int64_t(ph) * T;
    for (int i = 0; i < T; ++i) {
      idx[i] = i;
      bank[i] = int(stacked_pos(p, p.SWs, g0 + i) & 31);
    }
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return bank[a] < bank[b]; });
    for (int i = 0; i < T; ++i) tab[size_t(i % G) * 32 + i / G + size_t(ph) * T] = uint16_t(idx[i]);
  }
  return tab;
}

// Output-channel order of the m-groups (slot g*Q + q -> CSR row, -1 = empty slot).  Identity unless
// p.reorder > 0, or p.reorder == 0 and the densest group of consecutive rows holds > 5% more
// nonzeros per row than the layer's mean (skewed per-row sparsity, "adaptively tile the output channel"):
// then rows are dealt longest-first to the group with the fewest nonzeros so far (LPT), so every
// group's CTAs do about the same work.  Only the grouping changes: each channel still accumulates
// its own CSR row in ascending (c, kh, kw) order, so the output bits are identical.
std::vector<int> row_order(const JitPlan& p, const int32_t* rowptr, bool* reordered) {
  const int Q = p.Q, G = p.nmg;
  std::vector<int> ord(size_t(G) * Q, -1);
  for (int m = 0; m < p.M; ++m) ord[m] = m;
  *reordered = false;
  if (p.reorder < 0 || G < 2) return ord;
  std::vector<int64_t> gn(G, 0);
  int64_t tot = 0;
  for (int m = 0; m < p.M; ++m) {
    gn[m / Q] += rowptr[m + 1] - rowptr[m];
    tot += rowptr[m + 1] - rowptr[m];
  }
  // imbalance = the densest group's nonzeros per row over the layer's mean (a partial last group
  // has fewer rows, not less work per row)
  double mx = 0.0;
  for (int g = 0; g < G; ++g) mx = std::max(mx, double(gn[g]) / double(std::min(Q, p.M - g * Q)));
  if (p.reorder == 0 && (tot == 0 || mx <= 1.05 * double(tot) / p.M)) return ord;
  std::vector<int> rows(p.M);
  for (int m = 0; m < p.M; ++m) rows[m] = m;
  std::stable_sort(rows.begin(), rows.end(), [&](int a, int b) {
    return rowptr[a + 1] - rowptr[a] > rowptr[b + 1] - rowptr[b];
  });
  std::vector<int64_t> load(G, 0);
  std::vector<std::vector<int>> members(G);
  for (int m : rows) {
    int best = -1;
    for (int g = 0; g < G; ++g) {
      const int cap = g < G - 1 ? Q : p.M - (G - 1) * Q;
      if (int(members[g].size()) < cap && (best < 0 || load[g] < load[best])) best = g;
    }
    members[best].push_back(m);
    load[best] += rowptr[m + 1] - rowptr[m];
  }
  for (int g = 0; g < G; ++g) {
    std::sort(members[g].begin(), members[g].end());
    for (size_t q = 0; q < members[g].size(); ++q) ord[size_t(g) * Q + q] = members[g][q];
  }
  *reordered = true;
  return ord;
}

// PTX of the m-groups [g_lo, g_hi).  unit < 0: a complete kernel `escoin_jit_sconv` (blockIdx.y =
// g - g_lo).  unit >= 0: the device function `escoin_unit_<unit>` of a linked multi-unit kernel
// (gen_entry below calls it with the local group index), compiled relocatable on its own.
std::string gen_ptx(const JitPlan& p, const int32_t* rowptr, const int32_t* colidx, const float* value, int g_lo,
                    int g_hi, int unit) {
  // NT = threads of the CTA, NTc = compute threads (the prefetch warp, if any, is warp p.warps)
  const int KK = p.K * p.K, Q = p.Q, P = p.P, NTc = p.warps * 32, NT = NTc + (p.pw ? 32 : 0);
  const int ng = g_hi - g_lo;  // groups of this unit
  const int Hpd = p.H + 2 * p.pad, Wpd = p.W + 2 * p.pad;  // stretched geometry (R#3)
  const int hp = p.H + p.pad;
  const int HW = p.H * p.W, EF = p.E * p.F;
  // items (stacked_pos): pixels, or horizontal pixel pairs (hpair: Pi = P/2 pairs per lane, slots
  // j = 2*ji + h are pixel h of pair ji)
  const int EFi = p.E * p.Fi, Pi = p.Pi;
  const bool hpair = Pi != P;
  // nonzeros per (m-group, channel), ascending tap then row
  bool reordered = false;
  const std::vector<int> ord = row_order(p, rowptr, &reordered);
  const bool permuted = p.perm > 0 && !reordered && p.nphase > 0;  // lane -> pixel deal (perm_table)
  std::vector<std::vector<Nz>> lists(size_t(ng) * p.C);
  for (int slot = g_lo * Q; slot < g_hi * Q; ++slot) {
    const int m = ord[slot];
    if (m < 0) continue;
    const int g = slot / Q - g_lo, q = slot % Q;
    for (int j = rowptr[m]; j < rowptr[m + 1]; ++j) {
      const int col = colidx[j];
      const int c = col / (Hpd * Wpd), r = col % (Hpd * Wpd);
      const int kh = r / Wpd, kw = r % Wpd;
      uint32_t bits;
      std::memcpy(&bits, &value[j], 4);
      lists[size_t(g) * p.C + c].push_back({kh * p.K + kw, q, bits});
    }
  }
  for (auto& l : lists)
    std::stable_sort(l.begin(), l.end(), [](const Nz& a, const Nz& b) { return a.t < b.t; });

  Out o;
  o(".version 8.7");
  o(".target sm_100a");
  o(".address_size 64");
  o(".extern .shared .align 16 .b8 smem[];");
  const size_t table_pos = o.s.size();
  std::string mgr_table;
  const std::string mgr = unit < 0 ? std::string("mgr") : "mgr" + std::to_string(unit);
  if (unit < 0) {
    o(".visible .entry escoin_jit_sconv(.param .u64 p_in, .param .u64 p_out, .param .u64 p_bias, "
      ".param .u32 p_relu, .param .u32 p_N, .param .u64 p_perm, .param .u64 p_ws)");
    o(".maxntid %d, 1, 1", NT);
    o(".minnctapersm %d", p.minb);
  } else {
    o(".visible .func escoin_unit_%d(.param .u64 p_in, .param .u64 p_out, .param .u64 p_bias, "
      ".param .u32 p_relu, .param .u32 p_N, .param .u32 p_gy, .param .u64 p_perm, .param .u64 p_ws)", unit);
  }
  o("{");
  o(".reg .pred %%p<%d>;", 16 + 2 * p.KS + P);
  o(".reg .b32 %%r<%d>;", 64 + 4 * p.KS + 8 * P);
  o(".reg .b64 %%rd<%d>;", 32 + 2 * p.KS + 2 * P + p.KS);
  o(".reg .f32 %%a<%d>;", Q * P);
  o(".reg .f32 %%x<%d>;", KK * P);
  if (hpair) o(".reg .f32 %%y<%d>;", p.K * (p.K + 2) * Pi);  // words of one filter row per pair: (kh, w, ji)
  const int P2 = P / 2;  // slot pairs (FFMA2): %A<q*P2 + jp> = {%a<q*P + 2jp>, %a<q*P + 2jp + 1>}, same for %X
  if (p.f2) {
    o(".reg .b64 %%A<%d>;", Q * P2);
    o(".reg .b64 %%X<%d>;", KK * P2);
    o(".reg .b64 %%W;");
  }
  auto zero_acc = [&] {
    if (p.f2)
      for (int i = 0; i < Q * P2; ++i) o("mov.b64 %%A%d, 0;", i);
    else
      for (int q = 0; q < Q * P; ++q) o("mov.f32 %%a%d, 0f00000000;", q);
  };
  o(".reg .f32 %%v<8>;");
  o(".reg .b16 %%rs<2>;");
  o(".reg .b32 %%s<5>;");
  o(".reg .b32 %%bb;");  // shared-memory address of the group's staged bias
  if (p.ks > 1) {
    o(".reg .b32 %%kz<4>;");
    o(".reg .b64 %%rdz;");
    o(".reg .pred %%pz<2>;");
  }
  if (p.pw) {
    o(".reg .pred %%pw<2>;");
  }
  // params, ids
  o("ld.param.u64 %%rd0, [p_in];");
  o("cvta.to.global.u64 %%rd0, %%rd0;");
  o("ld.param.u64 %%rd1, [p_out];");
  o("cvta.to.global.u64 %%rd1, %%rd1;");
  o("ld.param.u64 %%rd2, [p_bias];");
  o("ld.param.u32 %%r0, [p_relu];");
  o("ld.param.u32 %%r1, [p_N];");
  if (p.ks > 1) o("cvt.u64.u32 %%rd13, %%r1;");
  o("ld.param.u64 %%rd11, [p_perm];");
  if (p.ks > 1) {
    // split channels: this CTA (grid z) writes raw partial sums — no bias, no ReLU — to its slice
    // ws + z*N*M*E*F of the workspace, same layout as the output
    o("ld.param.u64 %%rd1, [p_ws];");
    o("cvta.to.global.u64 %%rd1, %%rd1;");
    o("mov.u32 %%kz0, %%ctaid.z;");
    o("mul.lo.u32 %%kz1, %%kz0, %d;", p.M * p.E * p.F);
    o("mul.wide.u32 %%rdz, %%kz1, 4;");
    o("mul.lo.u64 %%rdz, %%rdz, %%rd13;");
    o("add.s64 %%rd1, %%rd1, %%rdz;");
    o("mov.u64 %%rd2, 0;");
    o("mov.u32 %%r0, 0;");
  }
  o("mov.u32 %%r2, %%tid.x;");
  // grid = (m-groups, pixel tiles): the m-groups of one tile are consecutive CTAs, so they run
  // together and read the tile's input from L2 instead of re-reading it from HBM
  o("mov.u32 %%r3, %%ctaid.y;");
  if (unit < 0)
    o("mov.u32 %%r4, %%ctaid.x;");
  else
    o("ld.param.u32 %%r4, [p_gy];");     // local m-group (the entry subtracted g_lo)
  const int NTh = NTc / p.sp, WH = p.warps / p.sp;
  o("and.b32 %%r7, %%r2, 31;");           // lane
  o("shr.u32 %%r8, %%r2, 5;");            // warp
  // sub-tile registers: %s0 = tid in the sub-tile, %s1 = sub-tile h = warp / WH, %s2 = warp in the
  // sub-tile, %s3 = its named barrier, %s4 = base of the whole stage area
  if (p.sp > 1) {
    o("div.u32 %%s1, %%r8, %d;", WH);
    o("mul.lo.u32 %%s0, %%s1, %d;", NTh);
    o("sub.u32 %%s0, %%r2, %%s0;");
    o("mul.lo.u32 %%s2, %%s1, %d;", WH);
    o("sub.u32 %%s2, %%r8, %%s2;");
    o("add.u32 %%s3, %%s1, 1;");
  } else {
    o("mov.u32 %%s0, %%r2;");
    o("mov.u32 %%s1, 0;");
    o("mov.u32 %%s2, %%r8;");
  }
  o("mul.lo.u32 %%r28, %%r3, %d;", p.T);  // g0: first output pixel of the tile
  if (p.sp > 1) o("mad.lo.u32 %%r28, %%s1, %d, %%r28;", p.T / p.sp);  // ... of the sub-tile
  o("mul.lo.u32 %%r29, %%r1, %d;", EFi);
  o("sub.u32 %%r29, %%r29, 1;");           // last item N*E*Fi - 1
  // window origin of item (n, oh, i): stacked row oh*S, column i*cs + co (pixels: ow*S, R#1)
  auto origin_cols = [&] {
    if (p.S > 1) o("mul.lo.u32 %%r32, %%r32, %d;", p.S);
    if (p.cs > 1) o("mul.lo.u32 %%r33, %%r33, %d;", p.cs);
    if (p.co) o("add.s32 %%r33, %%r33, %d;", p.co);
  };
  // q0 = pos(g0): staged window start
  o("div.u32 %%r30, %%r28, %d;", EFi);
  o("mul.lo.u32 %%r31, %%r30, %d;", EFi);
  o("sub.u32 %%r31, %%r28, %%r31;");
  o("div.u32 %%r32, %%r31, %d;", p.Fi);
  o("mul.lo.u32 %%r33, %%r32, %d;", p.Fi);
  o("sub.u32 %%r33, %%r31, %%r33;");
  origin_cols();
  o("mad.lo.u32 %%r34, %%r30, %d, %%r32;", hp);
  o("mad.lo.u32 %%r5, %%r34, %d, %%r33;", p.SWs);
  // bo = (q0 - pad) mod V: word q of the window is stored at buffer word q - q0 + bo, which puts
  // every data chunk (input column x = 0 mod V) on a V-word boundary
  o("add.u32 %%r10, %%r5, %d;", p.V - p.pad % p.V);
  o("and.b32 %%r10, %%r10, %d;", p.V - 1);
  o("mov.u32 %%r6, smem;");
  if (p.mb) {  // mbarriers full[NS], empty[NS] in the first 128 bytes, stage buffers after
    o("mov.u32 %%r36, %%r6;");
    o("add.u32 %%r6, %%r6, 128;");
  }
  o("mov.u32 %%s4, %%r6;");               // whole stage area (all sub-tiles), for the padding fill
  if (p.sp > 1) o("mad.lo.u32 %%r6, %%s1, %d, %%r6;", p.NS * p.CC * p.Ls * 4);  // this sub-tile's ring
  o("mul.lo.u32 %%r9, %%s2, %d;", 32 * Pi);
  o("add.u32 %%r9, %%r9, %%r7;");
  o("add.u32 %%r9, %%r9, %%r28;");        // item g of slot j = 0 (item slot ji adds 32 ji)
  if (p.pw) {
    // prefetch warp (warp p.warps): its lanes read the tile's first items' windows (valid words of the
    // stage buffers; garbage is fine) and, after the lane bases, take items far past the last one so
    // none of its stores is enabled; %pw1 = compute warp
    o("setp.eq.u32 %%pw0, %%r8, %d;", p.warps);
    o("not.pred %%pw1, %%pw0;");
    o("selp.b32 %%r9, %%r28, %%r9, %%pw0;");
  }
  if (permuted) {
    // lane -> pixel deal (perm_table): slot (warp*P + j, lane) of tile phase ph = tile mod nphase
    // takes pixel g0 + perm[ph][(warp*P + j)*32 + lane]; r(56+j) = that offset
    o("rem.u32 %%r54, %%r3, %d;", p.nphase);
    o("mul.lo.u32 %%r55, %%r54, %d;", p.T);
    o("mad.lo.u32 %%r55, %%r8, %d, %%r55;", 32 * P);
    o("add.u32 %%r55, %%r55, %%r7;");
    for (int j = 0; j < P; ++j) {
      o("add.u32 %%r54, %%r55, %d;", 32 * j);
      o("mul.wide.u32 %%rd12, %%r54, 2;");
      o("add.s64 %%rd12, %%rd12, %%rd11;");
      o("ld.global.nc.u16 %%rs0, [%%rd12];");
      o("cvt.u32.u16 %%r%d, %%rs0;", 56 + j);
    }
  }
  for (int j = 0; j < Pi; ++j) {         // lane smem base of item slot j: smem + 4 (pos(g) - q0)
    if (permuted)
      o("add.u32 %%r35, %%r28, %%r%d;", 56 + j);
    else
      o("add.u32 %%r35, %%r9, %d;", 32 * j);
    o("min.u32 %%r35, %%r35, %%r29;");     // tail lanes read in range, never store
    o("div.u32 %%r30, %%r35, %d;", EFi);
    o("mul.lo.u32 %%r31, %%r30, %d;", EFi);
    o("sub.u32 %%r31, %%r35, %%r31;");
    o("div.u32 %%r32, %%r31, %d;", p.Fi);
    o("mul.lo.u32 %%r33, %%r32, %d;", p.Fi);
    o("sub.u32 %%r33, %%r31, %%r33;");
    origin_cols();
    o("mad.lo.u32 %%r34, %%r30, %d, %%r32;", hp);
    o("mad.lo.u32 %%r34, %%r34, %d, %%r33;", p.SWs);
    o("sub.u32 %%r34, %%r34, %%r5;");
    o("add.u32 %%r34, %%r34, %%r10;");
    o("shl.b32 %%r34, %%r34, 2;");
    o("add.u32 %%r%d, %%r34, %%r6;", 40 + j);
  }
  if (p.pw) o("selp.b32 %%r9, %d, %%r9, %%pw0;", 0x7FFF0000);  // prefetch warp: no output item
  // Data-chunk staging slots k < KS: chunk d = tid + k*NT of the window's rows x (W/V) chunks;
  // d -> stacked row R = R_lo + d / cpr, chunk c = d % cpr, buffer word R*SWs + pad + c*V - q0 + bo.
  // Valid (predicate p(16+k)) iff R is an image row of an image < N and the V words lie inside the
  // buffer; only valid chunks are ever copied (the padding words were zeroed once).  regs: rd(32+k)
  // source pointer, r(64+k) buffer byte offset.
  o("sub.s32 %%r37, %%r5, %%r10;");                   // q0 - bo (>= -3)
  o("add.s32 %%r38, %%r37, %d;", p.SWs);
  o("div.s32 %%r38, %%r38, %d;", p.SWs);
  o("sub.s32 %%r38, %%r38, 1;");                      // R_lo = floor((q0 - bo) / SWs)
  for (int k = 0; k < p.KS; ++k) {
    const int rs = 64 + k, t0 = 64 + 2 * p.KS;  // t0.. scratch
    o("add.u32 %%r%d, %%s0, %d;", t0, k * NTh);                // d
    o("setp.lt.u32 %%p0, %%r%d, %d;", t0, p.rows_win * p.cpr);
    o("div.u32 %%r%d, %%r%d, %d;", t0 + 1, t0, p.cpr);         // row in window
    o("mul.lo.u32 %%r%d, %%r%d, %d;", t0 + 2, t0 + 1, p.cpr);
    o("sub.u32 %%r%d, %%r%d, %%r%d;", t0 + 2, t0, t0 + 2);     // c
    o("add.s32 %%r%d, %%r%d, %%r38;", t0 + 1, t0 + 1);         // R
    o("mul.lo.s32 %%r%d, %%r%d, %d;", t0 + 3, t0 + 1, p.SWs);
    o("mad.lo.s32 %%r%d, %%r%d, %d, %%r%d;", t0 + 3, t0 + 2, p.V, t0 + 3);
    o("add.s32 %%r%d, %%r%d, %d;", t0 + 3, t0 + 3, p.pad);
    o("sub.s32 %%r%d, %%r%d, %%r37;", t0 + 3, t0 + 3);         // buffer word
    o("setp.ge.and.s32 %%p0, %%r%d, 0, %%p0;", t0 + 3);
    o("setp.le.and.s32 %%p0, %%r%d, %d, %%p0;", t0 + 3, p.Lv * p.V - p.V);
    o("sub.s32 %%r%d, %%r%d, %d;", t0 + 1, t0 + 1, p.pad);     // rr
    o("setp.ge.and.s32 %%p0, %%r%d, 0, %%p0;", t0 + 1);
    o("max.s32 %%r%d, %%r%d, 0;", t0 + 1, t0 + 1);
    o("div.u32 %%r%d, %%r%d, %d;", t0 + 4, t0 + 1, hp);        // n
    o("mul.lo.u32 %%r%d, %%r%d, %d;", t0 + 5, t0 + 4, hp);
    o("sub.u32 %%r%d, %%r%d, %%r%d;", t0 + 5, t0 + 1, t0 + 5); // y
    o("setp.lt.and.u32 %%p0, %%r%d, %d, %%p0;", t0 + 5, p.H);
    o("setp.lt.and.u32 %%p0, %%r%d, %%r1, %%p0;", t0 + 4);
    o("selp.b32 %%r%d, 1, 0, %%p0;", 64 + p.KS + k);            // slot valid (kept as a register)
    o("max.s32 %%r%d, %%r%d, 0;", t0 + 3, t0 + 3);
    o("shl.b32 %%r%d, %%r%d, 2;", rs, t0 + 3);
    o("add.u32 %%r%d, %%r%d, %%r6;", rs, rs);                  // dst
    o("mul.lo.u32 %%r%d, %%r%d, %d;", t0 + 4, t0 + 4, p.C * HW);
    o("mad.lo.u32 %%r%d, %%r%d, %d, %%r%d;", t0 + 4, t0 + 5, p.W, t0 + 4);
    o("mad.lo.u32 %%r%d, %%r%d, %d, %%r%d;", t0 + 4, t0 + 2, p.V, t0 + 4);  // src element
    o("selp.u32 %%r%d, %%r%d, 0, %%p0;", t0 + 4, t0 + 4);
    o("mul.wide.u32 %%rd%d, %%r%d, 4;", 32 + k, t0 + 4);
    o("add.s64 %%rd%d, %%rd%d, %%rd0;", 32 + k, 32 + k);
    o("setp.ne.u32 %%p%d, %%r%d, 0;", 16 + k, 64 + p.KS + k);
    if (p.pw) o("and.pred %%p%d, %%p%d, %%pw1;", 16 + k, 16 + k);  // the prefetch warp never copies
  }
  // the padding words of every stage buffer: zero once (16-byte stores), before any copy lands
  {
    const int words = p.sp * p.NS * p.CC * p.Ls;  // multiple of 4
    o("shl.b32 %%r39, %%r2, 4;");
    o("add.u32 %%r39, %%r39, %%s4;");
    o("mov.b32 %%r23, 0;");
    if (p.pw) o("@%%pw0 bra.uni ZF_DONE;");
    for (int w0 = 0; w0 < words; w0 += 4 * NTc) {
      if (w0 + 4 * NTc > words) {
        o("setp.lt.u32 %%p2, %%r2, %d;", (words - w0) / 4);
        o("@%%p2 st.shared.v4.b32 [%%r39+%d], {%%r23, %%r23, %%r23, %%r23};", w0 * 4);
      } else {
        o("st.shared.v4.b32 [%%r39+%d], {%%r23, %%r23, %%r23, %%r23};", w0 * 4);
      }
    }
    if (p.pw) o("ZF_DONE:");
    // the group's bias values (0 past M or without bias) into shared memory behind the stage area now,
    // so the epilogue does not wait on a global load (ncu r03b: the bias loads' long-scoreboard stalls)
    o("add.u32 %%bb, %%s4, %d;", words * 4);
    if (!reordered) {
      o("setp.lt.u32 %%p13, %%r2, %d;", Q);
      o("@%%p13 add.u32 %%r24, %%r4, %d;", g_lo);
      o("@%%p13 mad.lo.u32 %%r24, %%r24, %d, %%r2;", Q);       // m = m0 + tid
      o("@%%p13 setp.lt.u32 %%p13, %%r24, %d;", p.M);
      o("mov.f32 %%v2, 0f00000000;");
      o("setp.ne.and.u64 %%p14, %%rd2, 0, %%p13;");
      o("@%%p14 mul.wide.u32 %%rd12, %%r24, 4;");
      o("@%%p14 add.s64 %%rd12, %%rd12, %%rd2;");
      o("@%%p14 ld.global.nc.f32 %%v2, [%%rd12];");
      o("setp.lt.u32 %%p13, %%r2, %d;", Q);
      o("shl.b32 %%r24, %%r2, 2;");
      o("add.u32 %%r24, %%r24, %%bb;");
      o("@%%p13 st.shared.f32 [%%r24], %%v2;");
    }
    o("bar.sync 0;");
  }
  // stage(chunk register rc, buffer byte offset register rb): r11 = chunk, r12 = buffer offset
  // Per (channel, slot) one cp.async; the channel offset and the stage offset are immediates
  // or hoisted per slot, predicates only where a chunk or the slot range is ragged.
  const bool ragged_c = p.C % p.CC != 0;
  auto stage = [&](const char* rc, const char* rb) {
    o("mul.wide.u32 %%rd3, %s, %d;", rc, p.CC * HW * 4);
    if (ragged_c) {
      o("mul.lo.u32 %%r13, %s, %d;", rc, p.CC);
      o("sub.s32 %%r13, %d, %%r13;", p.C);  // channels left
    }
    for (int k = 0; k < p.KS; ++k) {
      o("add.u32 %%r%d, %%r%d, %s;", 64 + 2 * p.KS + k, 64 + k, rb);
      o("add.s64 %%rd%d, %%rd%d, %%rd3;", 32 + p.KS + P + k, 32 + k);
    }
    for (int cc = 0; cc < p.CC; ++cc) {
      if (ragged_c) o("setp.gt.s32 %%p1, %%r13, %d;", cc);
      for (int k = 0; k < p.KS; ++k) {
        std::string pred = "@%p" + std::to_string(16 + k) + " ";
        if (ragged_c) {
          o("and.pred %%p2, %%p1, %%p%d;", 16 + k);
          pred = "@%p2 ";
        }
        o("%scp.async.%s.shared.global [%%r%d+%d], [%%rd%d+%d], %d;", pred.c_str(), p.V == 4 ? "cg" : "ca",
          64 + 2 * p.KS + k, cc * p.Ls * 4, 32 + p.KS + P + k, cc * HW * 4, 4 * p.V);
      }
    }
  };
  zero_acc();
  // Active chunk range per m-group (grouped layers: an m-group touches only its group's
  // channels; empty groups run no chunk at all and store bias only).
  std::vector<int> klo(ng, 0), khi(ng, 0);
  for (int g = 0; g < ng; ++g) {
    int lo = p.nch, hi = 0;
    for (int c = 0; c < p.C; ++c)
      if (!lists[size_t(g) * p.C + c].empty()) {
        lo = std::min(lo, c / p.CC);
        hi = std::max(hi, c / p.CC + 1);
      }
    if (lo < hi) { klo[g] = lo; khi[g] = hi; }
  }
  {
    std::string tbl;
    for (int g = 0; g < ng; ++g) tbl += (g ? ", " : "") + std::to_string(klo[g]) + ", " + std::to_string(khi[g]);
    // (declared at module scope below via a placeholder replaced after generation)
    mgr_table = tbl;
  }
  o("mov.u64 %%rd8, %s;", mgr.c_str());
  o("mul.wide.u32 %%rd9, %%r4, 8;");
  o("add.s64 %%rd8, %%rd8, %%rd9;");
  o("ld.global.nc.u32 %%r20, [%%rd8];");    // k_lo
  o("ld.global.nc.u32 %%r21, [%%rd8+4];");  // k_hi
  if (p.ks > 1) {
    // this CTA's part of the active chunks [k_lo, k_hi): [k_lo + a, k_lo + b), a = floor(z*n/ks) and b =
    // floor((z+1)*n/ks) rounded down to multiples of NS (b = n for the last z) — every part starts on
    // stage buffer 0, like the whole range, so the compile-time buffer offsets hold; a part may be empty
    o("sub.u32 %%kz2, %%r21, %%r20;");
    o("mov.u32 %%kz0, %%ctaid.z;");
    o("mul.lo.u32 %%kz1, %%kz0, %%kz2;");
    o("div.u32 %%kz1, %%kz1, %d;", p.ks);
    o("div.u32 %%kz1, %%kz1, %d;", p.NS);
    o("mul.lo.u32 %%kz1, %%kz1, %d;", p.NS);
    o("add.u32 %%kz3, %%kz0, 1;");
    o("mul.lo.u32 %%kz3, %%kz3, %%kz2;");
    o("div.u32 %%kz3, %%kz3, %d;", p.ks);
    o("div.u32 %%kz3, %%kz3, %d;", p.NS);
    o("mul.lo.u32 %%kz3, %%kz3, %d;", p.NS);
    o("setp.eq.u32 %%pz0, %%kz0, %d;", p.ks - 1);
    o("selp.b32 %%kz3, %%kz2, %%kz3, %%pz0;");
    o("add.u32 %%r21, %%r20, %%kz3;");
    o("add.u32 %%r20, %%r20, %%kz1;");
  }
  // Copy-ahead distance D: chunks staged before the one being computed. Bar mode: NS - 1
  // (one cp.async group per chunk, wait_group + CTA barrier per chunk). mbarrier mode: NS - 2,
  // so a warp may run one chunk ahead of the slowest (a buffer is refilled only after every
  // warp arrived on its `empty` barrier; data readiness is the `full` barrier's phase).
  const int D = p.mb ? std::max(1, p.NS - 2) : p.NS - 1;
  if (p.mb) {
    o("setp.eq.u32 %%p15, %%r2, 0;");
    for (int b = 0; b < p.NS; ++b) {
      o("@%%p15 mbarrier.init.shared::cta.b64 [%%r36+%d], %d;", 8 * b, NT);
      o("@%%p15 mbarrier.init.shared::cta.b64 [%%r36+%d], %d;", 8 * (p.NS + b), p.warps);
    }
    o("bar.sync 0;");
  }
  for (int s = 0; s < D; ++s) {
    o("add.u32 %%r11, %%r20, %d;", s);
    o("setp.ge.u32 %%p3, %%r11, %%r21;");
    o("@%%p3 bra.uni PRO%d;", s);
    o("mov.u32 %%r12, %d;", s * p.CC * p.Ls * 4);
    stage("%r11", "%r12");
    if (p.mb) o("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%%r36+%d];", 8 * s);
    o("PRO%d:", s);
    if (!p.mb) o("cp.async.commit_group;");
  }
  o("mov.u32 %%r15, %%r20;");  // k
  o("setp.ge.u32 %%p3, %%r15, %%r21;");
  o("@%%p3 bra.uni EPI;");
  o("mov.u32 %%r16, %d;", D * p.CC * p.Ls * 4);  // buffer offset of chunk k + D
  // branch targets
  std::string tg = "ts: .branchtargets ";
  for (int g = 0; g < ng; ++g)
    for (int k = 0; k < p.nch; ++k) {
      char b[32];
      snprintf(b, sizeof b, "%sB%d_%d", (g || k) ? ", " : "", g, k);
      tg += b;
    }
  tg += ";";
  // Instruction prefetch pass (p.pf): the code of one m-group is hundreds of KB and, after
  // an L2 flush, every CTA running that group would stall on the same sequential i-cache
  // misses (ncu: no_instructions dominates). Before the main loop, warp w < ceil(chunks /
  // gridDim.x) of each CTA runs ONE chunk block of its group — chunk k_lo + (blockIdx.x +
  // w * gridDim.x) mod (active chunks) — on whatever the stage buffers hold, then the
  // accumulators are reset: the CTAs of a group pull all parts of its code into L2 in
  // parallel, nothing computed is kept. (Guard predicates instead would make ptxas
  // if-convert every FFMA into FFMA + FSEL; one chunk per warp in EVERY warp measured slower
  // when L2 is warm: 16 streams per SM.)
  if (p.pf) {
    std::string tp = tg;
    tp[1] = 'p';  // "tp: .branchtargets ..."
    o("setp.eq.u32 %%p12, %%r1, 0;");              // false at run time (N >= 1), opaque to ptxas
    o("sub.u32 %%r23, %%r21, %%r20;");             // active chunks (>= 1 here)
    o("mov.u32 %%r22, %%nctaid.y;");
    o("add.u32 %%r24, %%r23, %%r22;");
    o("sub.u32 %%r24, %%r24, 1;");
    o("div.u32 %%r24, %%r24, %%r22;");             // warps needed so the group's CTAs cover every chunk
    o("mov.u32 %%r27, 0;");
    o("setp.ge.u32 %%p14, %%r8, %%r24;");
    o("@%%p14 bra.uni PF_DONE;");
    o("mad.lo.u32 %%r26, %%r8, %%r22, %%r3;");     // tile + warp * tiles
    o("rem.u32 %%r26, %%r26, %%r23;");
    o("add.u32 %%r26, %%r26, %%r20;");
    // The block reads stage buffer (k - k_lo) mod NS; shift the lane bases so it reads buffer NS-1
    // instead: that one holds only the zeros of the padding fill until the main loop's first
    // refill (after a CTA barrier), so the pass never reads words the prologue's copies are writing.
    o("sub.u32 %%r27, %%r26, %%r20;");
    o("rem.u32 %%r27, %%r27, %d;", p.NS);
    o("sub.u32 %%r27, %d, %%r27;", p.NS - 1);
    o("mul.lo.u32 %%r27, %%r27, %d;", p.CC * p.Ls * 4);
    for (int j = 0; j < Pi; ++j) o("add.u32 %%r%d, %%r%d, %%r27;", 40 + j, 40 + j);
    o("mad.lo.u32 %%r17, %%r4, %d, %%r26;", p.nch);
    o("%s", tp.c_str());
    o("brx.idx.uni %%r17, tp;");
    o("PF_DONE:");
    for (int j = 0; j < Pi; ++j) o("sub.u32 %%r%d, %%r%d, %%r27;", 40 + j, 40 + j);
    o("setp.ne.u32 %%p12, %%r1, 0;");              // true from here on
    zero_acc();
  }
  // one chunk block: per channel of the chunk, the taps the group uses, then its FFMAs
  auto block_body = [&](int g, int k) {
    const int buf = (k - klo[g]) % p.NS;
    for (int cc = 0; cc < p.CC; ++cc) {
      const int c = k * p.CC + cc;
      if (c >= p.C) break;
      const auto& l = lists[size_t(g) * p.C + c];
      if (l.empty()) continue;
      bool used[kMaxK * kMaxK] = {};
      for (const Nz& z : l) used[z.t] = true;
      // K <= 5: every used tap of the channel is loaded, then its FFMAs (ptxas schedules); larger
      // filters (AlexNet conv1 11x11) row by row — load a filter row's taps, run their FFMAs —
      // so at most one row of taps is live.  Either way the list is sorted by tap, so every
      // accumulator still receives its terms in ascending (kh, kw) order.
      const int rows_per_pass = p.K <= 5 ? p.K : 1;
      size_t zi = 0;
      // the FFMAs of the list's taps below t_end (the list is sorted by tap)
      auto emit_fmas = [&](int t_end) {
        for (; zi < l.size() && l[zi].t < t_end; ++zi) {
          const Nz& z = l[zi];
          if (p.f2) {
            // FFMA2: both halves x_j * w + acc_j, each rounded once (fma.rn) — the same two fp32
            // FMAs as the scalar form; the 64-bit immediate {w, w} becomes FFMA2's broadcast
            // 32-bit immediate operand
            for (int jp = 0; jp < P2; ++jp)
              o("mov.b64 %%W, 0x%08X%08X; fma.rn.f32x2 %%A%d, %%X%d, %%W, %%A%d;", z.bits, z.bits,
                z.q * P2 + jp, z.t * P2 + jp, z.q * P2 + jp);
          } else {
            for (int j = 0; j < P; ++j)
              o("fma.rn.f32 %%a%d, %%x%d, 0f%08X, %%a%d;", z.q * P + j, z.t * P + j, z.bits, z.q * P + j);
          }
        }
      };
      if (hpair) {
        // Horizontal pairs: pixel h of the pair reads tap (kh, kw) at word kw + h of filter row kh,
        // so a row's K taps of both pixels are the K + 1 words [0, K] — ld.shared.v2 of word pairs
        // (2r, 2r+1) from the (even) pair origin; tap kw's operand pair is {word kw, word kw + 1}
        // (a loaded pair for even kw, two moves for odd kw).  y index = (kh*(K+2) + w)*Pi + ji.
        const int K = p.K, YW = K + 2;
        for (int kh = 0; kh < K; ++kh)
          for (int r = 0; 2 * r <= K; ++r) {
            bool need = false;
            for (int kw = 2 * r - 1; kw <= 2 * r + 1; ++kw) need |= kw >= 0 && kw < K && used[kh * K + kw];
            if (!need) continue;
            for (int ji = 0; ji < Pi; ++ji)
              o("ld.shared.v2.f32 {%%y%d, %%y%d}, [%%r%d+%d];", (kh * YW + 2 * r) * Pi + ji,
                (kh * YW + 2 * r + 1) * Pi + ji, 40 + ji, ((buf * p.CC + cc) * p.Ls + kh * p.SWs + 2 * r) * 4);
          }
        for (int t = 0; t < KK; ++t) {
          if (!used[t]) continue;
          const int kh = t / K, kw = t % K;
          for (int ji = 0; ji < Pi; ++ji)
            o("mov.b64 %%X%d, {%%y%d, %%y%d};", t * Pi + ji, (kh * YW + kw) * Pi + ji, (kh * YW + kw + 1) * Pi + ji);
        }
        emit_fmas(KK);
      }
      for (int kh0 = 0; kh0 < p.K && !hpair; kh0 += rows_per_pass) {
        const int t_end = std::min(p.K, kh0 + rows_per_pass) * p.K;
        for (int t = kh0 * p.K; t < t_end; ++t) {
          if (!used[t]) continue;
          const int kh = t / p.K, kw = t % p.K;
          for (int j = 0; j < P; ++j)
            o("ld.shared.f32 %%x%d, [%%r%d+%d];", t * P + j, 40 + j,
              ((buf * p.CC + cc) * p.Ls + kh * p.SWs + kw) * 4);
          for (int jp = 0; jp < P2 && p.f2; ++jp)
            o("mov.b64 %%X%d, {%%x%d, %%x%d};", t * P2 + jp, t * P + 2 * jp, t * P + 2 * jp + 1);
        }
        emit_fmas(t_end);
      }
    }
  };
  if (!p.mb) {
    // Straight-line schedule: each m-group's chunks follow each other in the instruction stream,
    // with the per-chunk control (wait for this chunk's copies, CTA barrier, stage chunk k + D into
    // its buffer — both compile-time) inline between the blocks, so a group's code is one
    // sequential stream from its entry to the epilogue: no per-chunk jump back to a shared loop
    // head (the jumps restarted the sequential instruction prefetch three times per chunk; ncu
    // r02l: no_instructions was the top stall of the large-code layers).
    if (p.ks > 1) {  // enter the group's code at this CTA's first chunk
      std::string tk = "tks: .branchtargets ";
      for (int g = 0; g < ng; ++g)
        for (int k = 0; k < p.nch; ++k) tk += std::string(g || k ? ", " : "") + "E" + std::to_string(g) + "_" + std::to_string(k);
      o("%s;", tk.c_str());
      o("mad.lo.u32 %%kz1, %%r4, %d, %%r20;", p.nch);
      o("brx.idx.uni %%kz1, tks;");
    } else {
      std::string tgg = "tgg: .branchtargets ";
      for (int g = 0; g < ng; ++g) tgg += std::string(g ? ", " : "") + "G" + std::to_string(g);
      o("%s;", tgg.c_str());
      o("brx.idx.uni %%r4, tgg;");
    }
    for (int g = 0; g < ng; ++g) {
      o("G%d:", g);
      // prefetch warp: barrier 2 pairs the compute warps at chunk k with the prefetch warp at chunk k+1
      // (compute warps sync on it at every chunk but the last, the prefetch warp at every chunk but the
      // first), so the prefetch warp runs exactly one chunk ahead — the next chunk's code is in the L1.5
      // instruction cache when the compute warps get there — and the compute warps wait if it lags.
      // (A non-blocking arrive instead would let fast compute warps arrive twice in one phase.)
      for (int k = klo[g]; k < khi[g]; ++k) {
        if (p.ks > 1) {
          if (k > klo[g]) {  // this CTA's part ends here
            o("setp.le.u32 %%pz0, %%r21, %d;", k);
            o("@%%pz0 bra.uni EPI;");
          }
          o("E%d_%d:", g, k);
        }
        o("cp.async.wait_group %d;", p.NS - 2);
        if (p.pw) {
          o("@%%pw1 bar.sync 1, %d;", NTc);  // compute warps: this chunk's copies landed
          const bool cw = k + 1 < khi[g], pf = k > klo[g];
          if (cw && pf) o("bar.sync 2, %d;", NT);
          else if (cw) o("@%%pw1 bar.sync 2, %d;", NT);
          else if (pf) o("@%%pw0 bar.sync 2, %d;", NT);
        } else if (p.sp > 1) {
          o("bar.sync %%s3, %d;", NTh);
        } else {
          o("bar.sync 0;");
        }
        if (k + D < khi[g]) {
          if (p.ks > 1) {  // not past this CTA's part
            o("setp.le.u32 %%pz1, %%r21, %d;", k + D);
            o("@%%pz1 bra.uni SK%d_%d;", g, k);
          }
          o("mov.u32 %%r11, %d;", k + D);
          o("mov.u32 %%r12, %d;", ((k + D - klo[g]) % p.NS) * p.CC * p.Ls * 4);
          stage("%r11", "%r12");
          if (p.ks > 1) o("SK%d_%d:", g, k);
        }
        o("cp.async.commit_group;");
        o("B%d_%d:", g, k);
        block_body(g, k);
        if (p.pf) o("@!%%p12 bra.uni PF_DONE;");
      }
      o("bra.uni EPI;");
    }
    // entries of the prefetch / split tables for chunks a group never runs (not taken)
    for (int g = 0; g < ng; ++g)
      for (int k = 0; k < p.nch; ++k)
        if (k < klo[g] || k >= khi[g]) {
          o("B%d_%d:", g, k);
          if (p.ks > 1) o("E%d_%d:", g, k);
          o("bra.uni EPI;");
        }
  } else {
    o("LOOP:");
    if (!p.mb) {
      o("cp.async.wait_group %d;", p.NS - 2);
      if (p.sp > 1)
        o("bar.sync %%s3, %d;", NTh);         // only this sub-tile's warps
      else
        o("bar.sync 0;");
    }
    o("add.u32 %%r11, %%r15, %d;", D);
    o("setp.ge.u32 %%p3, %%r11, %%r21;");
    o("@%%p3 bra.uni NOSTAGE;");
    if (p.mb) {
      // buffer b = (j + D) % NS (byte offset r16); before refilling it, every warp must have
      // finished chunk j + D - NS: wait empty[b] with parity ((j + D) / NS + 1) & 1
      o("sub.u32 %%r48, %%r11, %%r20;");             // jj = j + D
      o("setp.lt.u32 %%p3, %%r48, %d;", p.NS);       // first use of the buffer: nothing to wait for
      o("@%%p3 bra.uni EMPTY_OK;");
      o("rem.u32 %%r49, %%r48, %d;", p.NS);
      o("div.u32 %%r50, %%r48, %d;", p.NS);
      o("add.u32 %%r50, %%r50, 1;");
      o("and.b32 %%r50, %%r50, 1;");
      o("mad.lo.u32 %%r51, %%r49, 8, %%r36;");
      o("add.u32 %%r51, %%r51, %d;", 8 * p.NS);
      o("WAIT_EMPTY:");
      o("mbarrier.try_wait.parity.shared::cta.b64 %%p15, [%%r51], %%r50;");
      o("@!%%p15 bra WAIT_EMPTY;");
      o("EMPTY_OK:");
    }
    stage("%r11", "%r16");
    if (p.mb) {
      o("sub.u32 %%r48, %%r11, %%r20;");
      o("rem.u32 %%r49, %%r48, %d;", p.NS);
      o("mad.lo.u32 %%r51, %%r49, 8, %%r36;");
      o("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%%r51];");
    }
    o("NOSTAGE:");
    if (!p.mb) o("cp.async.commit_group;");
    if (p.mb) {  // data of chunk j: full[j % NS], parity (j / NS) & 1
      o("sub.u32 %%r48, %%r15, %%r20;");
      o("rem.u32 %%r52, %%r48, %d;", p.NS);
      o("div.u32 %%r50, %%r48, %d;", p.NS);
      o("and.b32 %%r50, %%r50, 1;");
      o("mad.lo.u32 %%r51, %%r52, 8, %%r36;");
      o("WAIT_FULL:");
      o("mbarrier.try_wait.parity.shared::cta.b64 %%p15, [%%r51], %%r50;");
      o("@!%%p15 bra WAIT_FULL;");
      o("mad.lo.u32 %%r53, %%r52, 8, %%r36;");
      o("add.u32 %%r53, %%r53, %d;", 8 * p.NS);     // empty[j % NS], arrived on after the block
    }
    o("add.u32 %%r16, %%r16, %d;", p.CC * p.Ls * 4);
    o("setp.ge.u32 %%p4, %%r16, %d;", p.NS * p.CC * p.Ls * 4);
    o("@%%p4 mov.u32 %%r16, 0;");
    o("mad.lo.u32 %%r17, %%r4, %d, %%r15;", p.nch);
    o("%s", tg.c_str());
    o("brx.idx.uni %%r17, ts;");
    for (int g = 0; g < ng; ++g)
      for (int k = 0; k < p.nch; ++k) {
        o("B%d_%d:", g, k);
        if (k < klo[g] || k >= khi[g]) {  // never entered
          o("bra.uni NEXT;");
          continue;
        }
        block_body(g, k);
        o("bra.uni NEXT;");
      }
    o("NEXT:");
    if (p.pf) o("@!%%p12 bra.uni PF_DONE;");
    if (p.mb) {
      o("setp.eq.u32 %%p15, %%r7, 0;");
      o("@%%p15 mbarrier.arrive.shared::cta.b64 %%rd10, [%%r53];");
    }
    o("add.u32 %%r15, %%r15, 1;");
    o("setp.lt.u32 %%p5, %%r15, %%r21;");
    o("@%%p5 bra.uni LOOP;");

  }
  o("EPI:");
  for (int i = 0; i < Q * P2 && p.f2; ++i)  // unpack the pairs: the epilogues below read %a
    o("mov.b64 {%%a%d, %%a%d}, %%A%d;", 2 * i, 2 * i + 1, i);
  // Output slot j of this lane: predicate p(pv) = stored, rd(rdo) = out + 4*(n*M*E*F + oh*F + ow) (the
  // channel is added by the caller); t0..t0+4 scratch.  Item slot ji = j (pixels) or j / 2 (pairs,
  // pixel h = j % 2 of the pair: ow = 2i + co + h, stored only inside the row).
  auto slot_out = [&](int j, int pv, int rdo, int t0) {
    const int ji = hpair ? j / 2 : j, h = hpair ? j % 2 : 0;
    o("add.u32 %%r%d, %%r9, %d;", t0, 32 * ji);                // item g
    o("setp.le.u32 %%p%d, %%r%d, %%r29;", pv, t0);
    o("div.u32 %%r%d, %%r%d, %d;", t0 + 1, t0, EFi);          // n
    o("mul.lo.u32 %%r%d, %%r%d, %d;", t0 + 2, t0 + 1, EFi);
    o("sub.u32 %%r%d, %%r%d, %%r%d;", t0 + 2, t0, t0 + 2);    // item in image (pixels: oh*F + ow)
    if (hpair) {
      o("div.u32 %%r%d, %%r%d, %d;", t0 + 3, t0 + 2, p.Fi);   // oh
      o("mul.lo.u32 %%r%d, %%r%d, %d;", t0 + 4, t0 + 3, p.Fi);
      o("sub.u32 %%r%d, %%r%d, %%r%d;", t0 + 4, t0 + 2, t0 + 4);  // i
      o("mad.lo.s32 %%r%d, %%r%d, 2, %d;", t0 + 4, t0 + 4, p.co + h);  // ow (-1: phantom)
      o("setp.lt.and.u32 %%p%d, %%r%d, %d, %%p%d;", pv, t0 + 4, p.F, pv);
      o("mad.lo.u32 %%r%d, %%r%d, %d, %%r%d;", t0 + 2, t0 + 3, p.F, t0 + 4);  // oh*F + ow
    }
    o("mul.wide.u32 %%rd%d, %%r%d, %d;", rdo, t0 + 1, p.M * EF);
    o("cvt.u64.u32 %%rd7, %%r%d;", t0 + 2);
    o("add.s64 %%rd%d, %%rd%d, %%rd7;", rdo, rdo);
    o("shl.b64 %%rd%d, %%rd%d, 2;", rdo, rdo);
    o("add.s64 %%rd%d, %%rd%d, %%rd1;", rdo, rdo);
  };
  if (reordered) {
    // per-group epilogues: each group's rows are scattered output channels, so the channel of
    // (group, q) is an immediate (bias + 4m, out + 4m*EF); one brx on the group picks the block
    o("setp.ne.u64 %%p6, %%rd2, 0;");
    o("setp.ne.u32 %%p7, %%r0, 0;");
    for (int j = 0; j < P; ++j) slot_out(j, 16 + 2 * p.KS + j, 32 + p.KS + j, 64 + 4 * p.KS + 8 * j);
    std::string et = "te: .branchtargets ";
    for (int g = 0; g < ng; ++g) et += std::string(g ? ", " : "") + "EG" + std::to_string(g);
    o("%s;", et.c_str());
    o("brx.idx.uni %%r4, te;");
    for (int g = 0; g < ng; ++g) {
      o("EG%d:", g);
      for (int relu = 1; relu >= 0; --relu) {
        if (relu) o("@!%%p7 bra.uni EG%d_LIN;", g);
        else o("EG%d_LIN:", g);
        for (int q = 0; q < Q; ++q) {
          const int m = ord[size_t(g_lo + g) * Q + q];
          if (m < 0) continue;
          o("mov.f32 %%v0, 0f00000000;");
          o("@%%p6 ld.global.nc.f32 %%v0, [%%rd2+%d];", m * 4);
          for (int j = 0; j < P; ++j) {
            const int pv = 16 + 2 * p.KS + j, rdo = 32 + p.KS + j;
            o("add.rn.f32 %%v1, %%a%d, %%v0;", q * P + j);
            if (relu) {
              o("setp.gt.f32 %%p10, %%v1, 0f00000000;");
              o("selp.f32 %%v1, %%v1, 0f00000000, %%p10;");
            }
            o("@%%p%d st.global.f32 [%%rd%d+%lld], %%v1;", pv, rdo, (long long)m * EF * 4);
          }
        }
        o("ret;");
      }
    }
  } else {
    // epilogue
    o("setp.ne.u64 %%p6, %%rd2, 0;");
    o("setp.ne.u32 %%p7, %%r0, 0;");
    o("add.u32 %%r18, %%r4, %d;", g_lo);          // global m-group
    o("mul.lo.u32 %%r18, %%r18, %d;", Q);          // m0
    o("mul.wide.u32 %%rd5, %%r18, 4;");
    o("add.s64 %%rd5, %%rd5, %%rd2;");             // bias + m0
    o("mul.wide.u32 %%rd6, %%r18, %d;", EF * 4);   // m0 * EF bytes
    o("sub.s32 %%r19, %d, %%r18;", p.M);           // rows left
    for (int j = 0; j < P; ++j) {
      const int pv = 16 + 2 * p.KS + j, rdo = 32 + p.KS + j, t0 = 64 + 4 * p.KS + 8 * j;
      if (permuted) {  // stores in natural pixel order g0 + tid + j*NT (the accumulators go through smem)
        o("add.u32 %%r%d, %%r28, %%r2;", t0);
        o("add.u32 %%r%d, %%r%d, %d;", t0, t0, j * NTc);
        o("setp.le.u32 %%p%d, %%r%d, %%r29;", pv, t0);
        o("div.u32 %%r%d, %%r%d, %d;", t0 + 1, t0, EF);           // n
        o("mul.lo.u32 %%r%d, %%r%d, %d;", t0 + 2, t0 + 1, EF);
        o("sub.u32 %%r%d, %%r%d, %%r%d;", t0 + 2, t0, t0 + 2);    // oh*F + ow
        o("mul.wide.u32 %%rd%d, %%r%d, %d;", rdo, t0 + 1, p.M * EF);
        o("cvt.u64.u32 %%rd7, %%r%d;", t0 + 2);
        o("add.s64 %%rd%d, %%rd%d, %%rd7;", rdo, rdo);
        o("shl.b64 %%rd%d, %%rd%d, 2;", rdo, rdo);
        o("add.s64 %%rd%d, %%rd%d, %%rd1;", rdo, rdo);
      } else {
        slot_out(j, pv, rdo, t0);
      }
      o("add.s64 %%rd%d, %%rd%d, %%rd6;", rdo, rdo);
    }
    // acc + bias[m] (one fp32 add), then ReLU v > 0 ? v : 0 (R#10); relu is uniform, so the two
    // forms are separate straight-line blocks.  Row predicates only where a group can be partial
    // (M % Q != 0, last group); pixel predicates only matter in the tail CTA.
    const bool full_rows = p.M % Q == 0 || g_hi * Q <= p.M;
    if (permuted) {
      // Lanes hold dealt (non-consecutive) pixels: the accumulators are transposed through the
      // (now idle) stage ring, QB channels at a time, and stored in natural pixel order — every
      // warp store still writes 32 consecutive pixels of one channel (128 B).
      const int QB = std::max(1, std::min(Q, p.NS * p.CC * p.Ls / p.T));
      o("bar.sync 0;");                                 // every warp is done with the stage ring
      for (int j = 0; j < P; ++j) {
        o("shl.b32 %%r%d, %%r%d, 2;", 56 + j, 56 + j);
        o("add.u32 %%r%d, %%r%d, %%r6;", 56 + j, 56 + j);  // smem byte address of this slot's pixel
      }
      o("shl.b32 %%r54, %%r2, 2;");
      o("add.u32 %%r54, %%r54, %%r6;");                // natural pixel tid of the tile
      for (int b0 = 0; b0 < Q; b0 += QB) {
        const int qb = std::min(QB, Q - b0);
        for (int q = b0; q < b0 + qb; ++q)
          for (int j = 0; j < P; ++j)
            o("st.shared.f32 [%%r%d+%d], %%a%d;", 56 + j, (q - b0) * p.T * 4, q * P + j);
        o("bar.sync 0;");
        for (int relu = 1; relu >= 0; --relu) {
          if (relu) o("@!%%p7 bra.uni EPB%d_LIN;", b0);
          else o("EPB%d_LIN:", b0);
          for (int q = b0; q < b0 + qb; ++q) {
            if (!full_rows) o("setp.gt.s32 %%p8, %%r19, %d;", q);
            o("ld.shared.f32 %%v0, [%%bb+%d];", q * 4);  // staged bias
            for (int j = 0; j < P; ++j) {
              const int pv = 16 + 2 * p.KS + j, rdo = 32 + p.KS + j;
              o("ld.shared.f32 %%v1, [%%r54+%d];", ((q - b0) * p.T + j * NTc) * 4);
              o("add.rn.f32 %%v1, %%v1, %%v0;");
              if (relu) {
                o("setp.gt.f32 %%p10, %%v1, 0f00000000;");
                o("selp.f32 %%v1, %%v1, 0f00000000, %%p10;");
              }
              if (full_rows) {
                o("@%%p%d st.global.f32 [%%rd%d+%d], %%v1;", pv, rdo, q * EF * 4);
              } else {
                o("and.pred %%p11, %%p8, %%p%d;", pv);
                o("@%%p11 st.global.f32 [%%rd%d+%d], %%v1;", rdo, q * EF * 4);
              }
            }
          }
          if (relu) o("bra.uni EPB%d_END;", b0);
        }
        o("EPB%d_END:", b0);
        o("bar.sync 0;");
      }
      o("ret;");
    }
    for (int relu = 1; relu >= 0 && !permuted; --relu) {
      if (relu) o("@!%%p7 bra.uni EPI_LIN;");
      else o("EPI_LIN:");
      for (int q = 0; q < Q; ++q) {
        if (!full_rows) o("setp.gt.s32 %%p8, %%r19, %d;", q);
        o("ld.shared.f32 %%v0, [%%bb+%d];", q * 4);  // staged bias (0 past M / no bias)
        for (int j = 0; j < P; ++j) {
          const int pv = 16 + 2 * p.KS + j, rdo = 32 + p.KS + j;
          o("add.rn.f32 %%v1, %%a%d, %%v0;", q * P + j);
          if (relu) {
            o("setp.gt.f32 %%p10, %%v1, 0f00000000;");
            o("selp.f32 %%v1, %%v1, 0f00000000, %%p10;");
          }
          if (full_rows) {
            o("@%%p%d st.global.f32 [%%rd%d+%d], %%v1;", pv, rdo, q * EF * 4);
          } else {
            o("and.pred %%p11, %%p8, %%p%d;", pv);
            o("@%%p11 st.global.f32 [%%rd%d+%d], %%v1;", rdo, q * EF * 4);
          }
        }
      }
      if (relu) o("ret;");
    }

  }
  o("ret;");
  o("}");
  o.s.insert(table_pos, ".global .align 8 .u32 " + mgr + "[" + std::to_string(2 * ng) + "] = {" + mgr_table + "};\n");
  return o.s;
}

// Entry of a linked multi-unit kernel: picks the unit of blockIdx.y and calls its function with the
// local group index (one call per CTA); the units are compiled separately and linked (nvJitLink).
std::string gen_entry(const JitPlan& p, const std::vector<std::pair<int, int>>& ranges) {
  Out o;
  o(".version 8.7");
  o(".target sm_100a");
  o(".address_size 64");
  const char* sig = "(.param .u64 p_in, .param .u64 p_out, .param .u64 p_bias, .param .u32 p_relu, "
                    ".param .u32 p_N, .param .u32 p_gy, .param .u64 p_perm, .param .u64 p_ws)";
  for (size_t u = 0; u < ranges.size(); ++u) o(".extern .func escoin_unit_%d%s;", int(u), sig);
  o(".visible .entry escoin_jit_sconv(.param .u64 p_in, .param .u64 p_out, .param .u64 p_bias, "
    ".param .u32 p_relu, .param .u32 p_N, .param .u64 p_perm, .param .u64 p_ws)");
  o(".maxntid %d, 1, 1", (p.warps + (p.pw ? 1 : 0)) * 32);
  o(".minnctapersm %d", p.minb);
  o("{");
  o(".reg .pred %%p<2>;");
  o(".reg .b32 %%r<8>;");
  o(".reg .b64 %%rd<5>;");
  o("ld.param.u64 %%rd0, [p_in];");
  o("ld.param.u64 %%rd1, [p_out];");
  o("ld.param.u64 %%rd2, [p_bias];");
  o("ld.param.u32 %%r0, [p_relu];");
  o("ld.param.u32 %%r1, [p_N];");
  o("ld.param.u64 %%rd3, [p_perm];");
  o("ld.param.u64 %%rd4, [p_ws];");
  o("mov.u32 %%r2, %%ctaid.x;");
  for (size_t u = 0; u < ranges.size(); ++u) {
    o("setp.lt.u32 %%p0, %%r2, %d;", ranges[u].second);
    o("@%%p0 bra.uni U%d;", int(u));
  }
  o("ret;");
  for (size_t u = 0; u < ranges.size(); ++u) {
    o("U%d:", int(u));
    o("sub.u32 %%r3, %%r2, %d;", ranges[u].first);
    o("{");
    o(".param .u64 a0;");
    o(".param .u64 a1;");
    o(".param .u64 a2;");
    o(".param .u32 a3;");
    o(".param .u32 a4;");
    o(".param .u32 a5;");
    o(".param .u64 a6;");
    o(".param .u64 a7;");
    o("st.param.u64 [a0], %%rd0;");
    o("st.param.u64 [a1], %%rd1;");
    o("st.param.u64 [a2], %%rd2;");
    o("st.param.u32 [a3], %%r0;");
    o("st.param.u32 [a4], %%r1;");
    o("st.param.u32 [a5], %%r3;");
    o("st.param.u64 [a6], %%rd3;");
    o("st.param.u64 [a7], %%rd4;");
    o("call.uni escoin_unit_%d, (a0, a1, a2, a3, a4, a5, a6, a7);", int(u));
    o("}");
    o("ret;");
  }
  o("}");
  return o.s;
}

}  // namespace

int jit_plan(JitPlan& p, int C, int H, int W, int M, int K, int stride, int pad, int n_hint, double density) {
  // Any stride and padding: the stacked layout shares `pad` zero rows between neighbouring
  // images (image n's bottom padding is image n+1's top padding) and every window an output
  // reads lies inside its own image's padded extent, rows [oh*S, oh*S + K) of H + 2*pad.
  if (stride < 1 || pad < 0 || K > kMaxK) return -1;
  const int E = (H + 2 * pad - K) / stride + 1, F = (W + 2 * pad - K) / stride + 1;
  if (H + 2 * pad < K || W + 2 * pad < K || E < 1 || F < 1) return -1;
  p.C = C; p.H = H; p.W = W; p.M = M; p.K = K; p.pad = pad;
  p.E = E; p.F = F; p.S = stride;
  if (p.P <= 0) p.P = 1;
  p.f2 = (p.pair >= 0 && p.P % 2 == 0) ? 1 : 0;
  // channel chunk / stages: 5x5 (and larger) filters stage a wider halo per channel and run
  // 2.8x the FFMAs per staged word; measured best with 4 channels x 4 stages (AlexNet conv2
  // +5% over 8 x 3), 3x3 and 1x1 with 8 x 3 (conv3 -14% with 4 x 4).
  if (p.CC <= 0) p.CC = K >= 5 ? 4 : 8;
  if (p.NS <= 1) p.NS = K >= 5 ? 4 : 3;
  p.mb = p.mb > 0 ? 1 : 0;
  // the instruction-prefetch pass reads the last stage buffer, free until the first CTA barrier of
  // the main loop; the mbarrier pipeline has no such barrier, so it runs without the pass
  const bool ks_auto = p.ks < 0;  // resolved below, once the grid is known
  const bool ks_only = p.ks <= -2;  // ... and no kernel at all when no split is needed
  p.ks = (p.ks > 1 && !p.mb) ? std::min(p.ks, 64) : 1;
  if (p.ks > 1) {  // split channels: plain straight-line barrier mode, identity grouping
    p.perm = 0;
    p.reorder = -1;
  }
  p.pw = (p.pw > 0 && !p.mb && p.split <= 1 && p.perm <= 0 && p.ks == 1) ? 1 : 0;
  p.pf = (p.pf < 0 || p.mb || p.pw || p.ks > 1) ? 0 : 1;  // the prefetch warp replaces the prefetch pass
  n_hint = std::max(1, n_hint);
  if (p.Q <= 0 && p.warps <= 0 && p.minb <= 0 && p.f2) {
    // FFMA2 shapes (P even): a lane's work is pipe-bound by its FFMA2s (2 FMA-pipe cycles each) as long
    // as the issue slots (FFMA2 + tap loads + pair moves) and the shared-memory wavefronts of the 4
    // SMSPs keep up; the grid (tiles x m-groups) is sized so the last wave is nearly full — every warp
    // count 4..32 and 1-4 CTAs per SM are candidates (waves are few at batch 128: res5 = 16 groups x
    // 7-14 tiles), the partial last tile and group counted as lost work.
    double best = -1;
    JitPlan keep = p;
    const double pixels = double(n_hint) * E * F;
    for (int Qc : {16, 24, 32, 48, 64})
      for (int mb = 1; mb <= 4; ++mb)
        for (int wc = 4; wc <= 32 && wc * mb <= 64; ++wc) {
          JitPlan t = keep;
          t.Q = std::min(Qc, M); t.warps = wc; t.minb = mb;
          const int regs = std::min(255, 65536 / (wc * 32 * mb)) & ~7;
          if (!plan_fit(t, n_hint)) continue;
          const bool hpair = t.Pi != t.P;
          const int KK = K * K, taps_regs = hpair ? t.Pi * (K * (K + 2) + 2 * K) : KK * t.P;
          if (t.Q * t.P + taps_regs + 24 > regs) continue;
          const double items = double(n_hint) * E * t.Fi;
          const double work = items / t.T * (double(M) / t.Q);  // CTA-equivalents of real work
          const double ctas = std::ceil(items / t.T) * t.nmg, per_wave = 148.0 * mb;
          const double wave_eff = work / (std::ceil(ctas / per_wave) * per_wave);
          const double phantom = pixels / (items * (hpair ? 2.0 : 1.0));  // pair slots holding real pixels
          const double fma_cyc = t.Q * KK * density * t.P;
          const double used = 1.0 - std::pow(1.0 - density, t.Q);  // tap-use probability
          const double lds = hpair ? t.Pi * K * ((K + 2) / 2) : KK * used * t.P;
          const double movs = hpair ? t.Pi * K * (K / 2) * 2.0 : 0.0;
          const double issue = fma_cyc / 2 + lds + movs + 2.0 * t.L / t.T * t.P;
          const double wavefronts = 4.0 * lds * (hpair ? 2.0 : 1.0);
          const double eff = fma_cyc / std::max(fma_cyc, std::max(issue / 0.85, wavefronts / 0.8));
          const double fetch = std::pow(t.warps / 32.0, 0.25);
          const double score = wave_eff * phantom * eff * fetch;
          if (score > best) { best = score; p = t; }
        }
    if (best < 0) return -1;
  } else if (p.Q <= 0 && p.warps <= 0 && p.minb <= 0) {
    // Shape choice by a small model (escoin_csr_autotune_ex measures the real choice among the
    // compiled tunings).  Registers: Q accumulators + K*K taps + ~20 <= 65536 / (threads * CTAs/SM).
    // Terms: wave fill of the tiles x m-groups grid over 148 SMs x CTAs/SM (grids are often only
    // 1-3 waves at batch 128; 7x7 and 14x14 layers need small Q / several CTAs per SM to cover the
    // SMs), FFMA share (one LDS per used tap feeds Q*density FFMAs), and instruction-fetch
    // sharing (warps of one CTA run the same code; measured ~0.85x at 16 warps vs 32).
    double best = -1;
    JitPlan keep = p;
    static const int shapes[][2] = {{32, 1}, {28, 1}, {24, 1}, {20, 1}, {16, 1}, {16, 2}, {12, 2}, {8, 2},
                                    {10, 3}, {8, 3}, {8, 4}, {6, 4}, {4, 4}};
    for (int Qc : {16, 32, 64})
      for (const auto& sh : shapes) {
        const int wc = sh[0], mb = sh[1];
        const int regs = std::min(255, 65536 / (wc * 32 * mb)) & ~7;
        const int tap_regs = K <= 5 ? K * K : 2 * K;  // live taps (row-wise passes above 5x5)
        if (std::min(Qc, M) + tap_regs + 20 > regs && !(Qc == 32 && wc == 32 && K <= 5)) continue;
        JitPlan t = keep;
        t.Q = std::min(Qc, M); t.warps = wc; t.minb = mb;
        if (!plan_fit(t, n_hint)) continue;
        const double pixels = double(n_hint) * E * F;
        const double ctas = std::ceil(pixels / t.T) * t.nmg, per_wave = 148.0 * mb;
        const double wave_eff = ctas / (std::ceil(ctas / per_wave) * per_wave);
        const double fma = t.Q * K * K * density;
        const double taps = K * K * (1.0 - std::pow(1.0 - density, t.Q));
        const double instr_eff = fma / (fma + taps + 2.0 * t.L / t.T);
        const double fetch = std::pow(t.warps / 32.0, 0.25);
        const double score = wave_eff * instr_eff * fetch;
        if (score > best) { best = score; p = t; }
      }
    if (best < 0) return -1;
  } else {
    if (p.Q <= 0) p.Q = 64;
    if (p.minb <= 0) p.minb = 1;
    p.Q = std::min(p.Q, M);
    if (p.warps <= 0) {
      // Warps for the given Q and CTAs/SM: the tile size that fills the last wave of the (tiles x
      // groups) grid best — time ~ waves x CTAs/SM x (rows per group) x (pixels per CTA), discounted
      // mildly for few warps per SM (latency hiding, shared instruction fetch) — within the register
      // budget.
      const int G = cdiv(M, p.Q), Qb = cdiv(M, G), tap_regs = K <= 5 ? K * K * p.P : 2 * K * p.P;
      double best = -1;
      int bw = 16;
      for (int wc = 8; wc <= 32 && wc * p.minb <= 64; ++wc) {
        const int regs = std::min(255, 65536 / (wc * 32 * p.minb)) & ~7;
        if (Qb * p.P + tap_regs / 2 + 16 > regs) continue;  // (taps are not all live at once)
        JitPlan t = p;
        t.warps = wc;
        if (!plan_fit(t, n_hint)) continue;
        const double items = double(n_hint) * E * t.Fi;
        const double ctas = std::ceil(items / t.T) * G, waves = std::ceil(ctas / (148.0 * t.minb));
        // minb CTAs share an SM (one's barrier wait is covered by the other's work: ~10%, r03a)
        const double eff = std::pow(std::min(1.0, wc * t.minb / 32.0), 0.25) * (t.minb >= 2 ? 1.1 : 1.0);
        const double time = waves * t.minb * t.T * Qb / eff;
        if (best < 0 || time < best * 0.999) { best = time; bw = wc; }
      }
      p.warps = bw;
    }
    if (!plan_fit(p, n_hint)) return -1;
  }
  {
    // Balanced groups: the ceil(M/Q) m-groups take ceil(M/groups) rows each instead of Q (+ a short last
    // group) — the CTAs of the fullest group set the layer time (ResNet res4: Q 48 -> 43, 6 groups).
    const int G = cdiv(M, p.Q), Qb = cdiv(M, G);
    if (Qb != p.Q) {
      p.Q = Qb;
      if (!plan_fit(p, n_hint)) return -1;
    }
  }
  if (ks_auto && !p.mb) {
    // ks < 0: split the channels when the (tiles x groups) grid covers less than one wave of
    // 148 x CTAs/SM: enough parts to fill it, at least NS chunks each
    // time ~ waves(ctas * ks) / ks, + 4% per extra part (partial-sum traffic, the reduce)
    const double ctas = std::ceil(double(n_hint) * E * p.Fi / p.T) * p.nmg, slots = 148.0 * p.minb;
    const int maxp = std::max(1, std::min(p.nch / p.NS, 64));
    double best_t = 1e30;
    for (int k = 1; k <= maxp; ++k) {
      const double t = std::ceil(ctas * k / slots) / k * (1.0 + 0.04 * (k - 1));
      if (t < best_t * 0.999) { best_t = t; p.ks = k; }
    }
    if (p.ks > 1) {
      p.perm = 0;
      p.reorder = -1;
      p.pw = 0;
      p.pf = 0;
    } else if (ks_only) {
      return -1;
    }
  }
  if (p.smem_bytes > 227 * 1024 / p.minb) return -1;
  return 0;
}

namespace {

// ---------------------------------------------------------------- compile pool
// nvPTXCompiler runs single-threaded per call; the units of every jit_build in the process share
// one bound on concurrent compiles (ESCOIN_JIT_THREADS, else the host's cores), so callers may
// compile many layers at once without oversubscribing the host.
class CompileSlots {
 public:
  CompileSlots() {
    const char* e = std::getenv("ESCOIN_JIT_THREADS");
    n_ = e ? std::atoi(e) : int(std::thread::hardware_concurrency());
    if (n_ < 1) n_ = 1;
  }
  void acquire() {
    std::unique_lock<std::mutex> lk(m_);
    cv_.wait(lk, [&] { return n_ > 0; });
    --n_;
  }
  void release() {
    { std::lock_guard<std::mutex> lk(m_); ++n_; }
    cv_.notify_one();
  }

 private:
  std::mutex m_;
  std::condition_variable cv_;
  int n_;
};

CompileSlots& slots() {
  static CompileSlots s;
  return s;
}

const char* const kOpts[] = {"--gpu-name=sm_100a", "-O3"};
typedef std::vector<std::string> Opts;

// ---------------------------------------------------------------- cubin cache
// ESCOIN_JIT_CACHE=<dir>: cubins keyed by two 64-bit FNV-1a hashes (different offset bases) of the
// PTX text, the compile options and the compiler version.  Files are written to a temporary name
// and renamed, so concurrent processes (the ranks of one node) never read a partial cubin.
uint64_t fnv1a(const std::string& s, uint64_t h) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001B3ULL;
  }
  return h;
}

std::string cache_key(const std::string& ptx, const Opts& opts) {
  unsigned maj = 0, min = 0;
  nvPTXCompilerGetVersion(&maj, &min);
  std::string salt = "escoin-jit-v3|" + std::to_string(maj) + "." + std::to_string(min);
  for (const std::string& o : opts) salt += "|" + o;
  char b[64];
  snprintf(b, sizeof b, "%016llx%016llx", (unsigned long long)fnv1a(salt + ptx, 0xCBF29CE484222325ULL),
           (unsigned long long)fnv1a(ptx + salt, 0x84222325CBF29CE4ULL));
  return b;
}

std::string cache_dir() {
  const char* e = std::getenv("ESCOIN_JIT_CACHE");
  return e ? std::string(e) : std::string();
}

bool cache_get(const std::string& dir, const std::string& key, std::vector<char>* out) {
  FILE* f = std::fopen((dir + "/" + key + ".cubin").c_str(), "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  bool ok = n > 0;
  if (ok) {
    out->resize(size_t(n));
    ok = std::fread(out->data(), 1, size_t(n), f) == size_t(n);
  }
  std::fclose(f);
  return ok;
}

void cache_put(const std::string& dir, const std::string& key, const std::vector<char>& cubin) {
  static std::atomic<unsigned> seq{0};
  char tmpn[64];
  snprintf(tmpn, sizeof tmpn, ".tmp.%d.%u", int(getpid()), seq.fetch_add(1));
  const std::string fin = dir + "/" + key + ".cubin", tmp = fin + tmpn;
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return;  // unwritable cache: compile-only behaviour
  const bool ok = std::fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
  std::fclose(f);
  if (!ok || std::rename(tmp.c_str(), fin.c_str()) != 0) std::remove(tmp.c_str());
}

// PTX -> cubin (or relocatable object with --compile-only) (cache first); 0 = OK, -2 = compile error.
int compile_ptx(const std::string& ptx, const Opts& opts, std::vector<char>* cubin, std::string* log, bool* hit) {
  const std::string dir = cache_dir();
  const std::string key = dir.empty() ? std::string() : cache_key(ptx, opts);
  if (!dir.empty() && cache_get(dir, key, cubin)) {
    *hit = true;
    return 0;
  }
  *hit = false;
  slots().acquire();
  nvPTXCompilerHandle c = nullptr;
  int rc = 0;
  if (nvPTXCompilerCreate(&c, ptx.size(), ptx.c_str()) != NVPTXCOMPILE_SUCCESS) {
    rc = -2;
  } else if ([&] {
               std::vector<const char*> o;
               for (const std::string& x : opts) o.push_back(x.c_str());
               return nvPTXCompilerCompile(c, int(o.size()), o.data());
             }() != NVPTXCOMPILE_SUCCESS) {
    if (log) {
      size_t n = 0;
      nvPTXCompilerGetErrorLogSize(c, &n);
      std::string e(n, '\0');
      if (n) nvPTXCompilerGetErrorLog(c, &e[0]);
      *log = e;
    }
    rc = -2;
  } else {
    size_t n = 0;
    nvPTXCompilerGetCompiledProgramSize(c, &n);
    cubin->resize(n);
    nvPTXCompilerGetCompiledProgram(c, cubin->data());
  }
  if (c) nvPTXCompilerDestroy(&c);
  slots().release();
  if (rc == 0 && !dir.empty()) cache_put(dir, key, *cubin);
  return rc;
}

// nvJitLink, loaded at first use from the CUDA toolkit by path (its static archive would add
// ~100 MB to the library; a process may also hold an older libnvJitLink.so.12 of its own, e.g.
// torch's, so the library is opened by full path, RTLD_LOCAL, and the 12.9 entry points used).
struct JitLinkApi {
  nvJitLinkResult (*create)(nvJitLinkHandle*, uint32_t, const char**) = nullptr;
  nvJitLinkResult (*destroy)(nvJitLinkHandle*) = nullptr;
  nvJitLinkResult (*add)(nvJitLinkHandle, nvJitLinkInputType, const void*, size_t, const char*) = nullptr;
  nvJitLinkResult (*complete)(nvJitLinkHandle) = nullptr;
  nvJitLinkResult (*cubin_size)(nvJitLinkHandle, size_t*) = nullptr;
  nvJitLinkResult (*cubin)(nvJitLinkHandle, void*) = nullptr;
  nvJitLinkResult (*log_size)(nvJitLinkHandle, size_t*) = nullptr;
  nvJitLinkResult (*log)(nvJitLinkHandle, char*) = nullptr;
  bool ok = false;
};

const JitLinkApi& jitlink() {
  static JitLinkApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    std::vector<std::string> cands;
    if (const char* e = std::getenv("ESCOIN_NVJITLINK")) cands.push_back(e);
    cands.push_back("/usr/local/cuda/lib64/libnvJitLink.so.12");
    cands.push_back("libnvJitLink.so.12");
    for (const std::string& c : cands) {
      void* h = dlopen(c.c_str(), RTLD_NOW | RTLD_LOCAL);
      if (!h) continue;
      auto sym = [&](const char* n) { return dlsym(h, n); };
      a.create = reinterpret_cast<decltype(a.create)>(sym("__nvJitLinkCreate_12_9"));
      a.destroy = reinterpret_cast<decltype(a.destroy)>(sym("__nvJitLinkDestroy_12_9"));
      a.add = reinterpret_cast<decltype(a.add)>(sym("__nvJitLinkAddData_12_9"));
      a.complete = reinterpret_cast<decltype(a.complete)>(sym("__nvJitLinkComplete_12_9"));
      a.cubin_size = reinterpret_cast<decltype(a.cubin_size)>(sym("__nvJitLinkGetLinkedCubinSize_12_9"));
      a.cubin = reinterpret_cast<decltype(a.cubin)>(sym("__nvJitLinkGetLinkedCubin_12_9"));
      a.log_size = reinterpret_cast<decltype(a.log_size)>(sym("__nvJitLinkGetErrorLogSize_12_9"));
      a.log = reinterpret_cast<decltype(a.log)>(sym("__nvJitLinkGetErrorLog_12_9"));
      a.ok = a.create && a.destroy && a.add && a.complete && a.cubin_size && a.cubin && a.log_size && a.log;
      if (a.ok) return;
      dlclose(h);
    }
  });
  return a;
}

// Link relocatable objects (the units + the entry) into one cubin; 0 = OK.
int link_objects(const std::vector<std::vector<char>>& objs, std::vector<char>* cubin, std::string* log) {
  const JitLinkApi& L = jitlink();
  if (!L.ok) {
    if (log) *log = "nvJitLink (libnvJitLink.so.12, CUDA 12.9) not found: set ESCOIN_NVJITLINK";
    return -2;
  }
  nvJitLinkHandle h = nullptr;
  const char* lo[] = {"-arch=sm_100a"};
  if (L.create(&h, 1, lo) != NVJITLINK_SUCCESS) return -2;
  int rc = 0;
  for (size_t i = 0; i < objs.size() && rc == 0; ++i) {
    const std::string name = "unit" + std::to_string(i);
    if (L.add(h, NVJITLINK_INPUT_CUBIN, objs[i].data(), objs[i].size(), name.c_str()) != NVJITLINK_SUCCESS) rc = -2;
  }
  if (rc == 0 && L.complete(h) != NVJITLINK_SUCCESS) rc = -2;
  if (rc != 0 && log) {
    size_t n = 0;
    L.log_size(h, &n);
    std::string e(n, '\0');
    if (n) L.log(h, &e[0]);
    *log = e;
  }
  if (rc == 0) {
    size_t n = 0;
    L.cubin_size(h, &n);
    cubin->resize(n);
    L.cubin(h, cubin->data());
  }
  L.destroy(&h);
  return rc;
}

}  // namespace

std::vector<std::pair<int, int>> jit_units(const JitPlan& p, const int32_t* rowptr) {
  // nonzeros per m-group; units are contiguous group ranges of about equal nonzeros, about
  // kUnitNnz each (ptxas time grows with the code: ~0.25 ms per FFMA on one host core), so
  // the largest layers compile in parallel; never more units than groups or than 32.  A linked
  // unit runs 2-12% slower than the same code compiled as one kernel (measured, r02c: function
  // ABI around the staging code), so only layers whose single compile would take minutes split.
  constexpr int64_t kUnitNnz = 500000;
  constexpr int64_t kUnitBlocks = 1536;  // chunk blocks (brx targets): ptxas time also grows with these
  std::vector<int64_t> gn(p.nmg, 0);
  int64_t tot = 0;
  bool reordered = false;
  const std::vector<int> ord = row_order(p, rowptr, &reordered);
  for (int g = 0; g < p.nmg; ++g) {
    for (int q = 0; q < p.Q; ++q) {
      const int m = ord[size_t(g) * p.Q + q];
      if (m >= 0) gn[g] += rowptr[m + 1] - rowptr[m];
    }
    tot += gn[g];
  }
  int U = p.units > 0 ? p.units
                      : int(std::max((tot + kUnitNnz - 1) / kUnitNnz,
                                     (int64_t(p.nmg) * p.nch + kUnitBlocks - 1) / kUnitBlocks));
  U = std::max(1, std::min(U, std::min(p.nmg, 32)));
  std::vector<std::pair<int, int>> r;
  int g = 0;
  int64_t acc = 0;
  for (int u = 0; u < U; ++u) {
    const int lo = g;
    const int64_t target = (tot * (u + 1) + U - 1) / U;  // cumulative share of units 0..u
    while (g < p.nmg && (g == lo || acc + gn[g] <= target) && p.nmg - g > U - 1 - u) acc += gn[g++];
    if (u == U - 1) while (g < p.nmg) acc += gn[g++];
    r.emplace_back(lo, g);
  }
  return r;
}

int jit_cubin(JitModule& jm, const JitPlan& p, const int32_t* rowptr, const int32_t* colidx, const float* value,
              std::vector<char>* cubin_out, std::string* log) {
  jm.plan = p;
  row_order(p, rowptr, &jm.reordered);
  const auto ranges = jit_units(p, rowptr);
  const int U = int(ranges.size());
  jm.units.assign(U, JitUnit());
  // One unit: a complete kernel.  Several: each unit is the device function of its m-groups,
  // compiled relocatable in its own host thread (register budget of the kernel's occupancy),
  // then linked with a small entry kernel that calls the unit of blockIdx.y — ONE launch.
  if (U > 1 && p.pw) {  // a unit function with the prefetch warp's barriers exceeds the entry's register cap
    if (log) *log = "the prefetch warp (pw) is not supported with linked units";
    jm.units.clear();
    return -2;
  }
  const int maxreg = std::min(255, 65536 / (p.warps * 32 * p.minb)) & ~7;
  Opts uopts = {kOpts[0], kOpts[1]};
  if (U > 1) {
    uopts.push_back("--compile-only");
    uopts.push_back("--maxrregcount=" + std::to_string(maxreg));
  }
  std::vector<std::vector<char>> objs(U + (U > 1 ? 1 : 0));
  std::vector<int> rcs(U + 1, 0);
  std::vector<std::string> logs(U + 1);
  auto work = [&](int u) {
    JitUnit& ju = jm.units[u];
    ju.g_lo = ranges[u].first;
    ju.g_hi = ranges[u].second;
    const std::string ptx = gen_ptx(p, rowptr, colidx, value, ju.g_lo, ju.g_hi, U > 1 ? u : -1);
    ju.ptx_bytes = ptx.size();
    rcs[u] = compile_ptx(ptx, uopts, &objs[u], &logs[u], &ju.cache_hit);
    (void)ju;
    ju.cubin_bytes = objs[u].size();
  };
  if (U == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int u = 0; u < U; ++u) th.emplace_back(work, u);
    bool hit = false;
    rcs[U] = compile_ptx(gen_entry(p, ranges), Opts{kOpts[0], kOpts[1], "--compile-only"}, &objs[U], &logs[U],
                         &hit);
    for (auto& t : th) t.join();
  }
  for (int u = 0; u <= U; ++u)
    if (rcs[u] != 0) {
      if (log) *log = logs[u];
      jm.units.clear();
      return -2;
    }
  std::vector<char> linked;
  if (U > 1 && link_objects(objs, &linked, log) != 0) {
    jm.units.clear();
    return -2;
  }
  *cubin_out = U > 1 ? std::move(linked) : std::move(objs[0]);
  if (const char* dump = std::getenv("ESCOIN_JIT_DUMP")) {  // inspection only (cuobjdump -sass)
    if (FILE* f = std::fopen(dump, "wb")) {
      std::fwrite(cubin_out->data(), 1, cubin_out->size(), f);
      std::fclose(f);
    }
  }
  jm.ptx_bytes = jm.cubin_bytes = 0;
  jm.cache_hits = 0;
  for (const JitUnit& ju : jm.units) {
    jm.ptx_bytes += ju.ptx_bytes;
    jm.cache_hits += ju.cache_hit ? 1 : 0;
  }
  jm.cubin_bytes = cubin_out->size();
  return 0;
}

int jit_build(JitModule& jm, const JitPlan& p, const int32_t* rowptr, const int32_t* colidx, const float* value,
              std::string* log) {
  const Driver& d = driver();
  if (!d.ok) return -1;
  // the driver-API module calls below need the device's primary context current in THIS host
  // thread (callers may compile from worker threads); a runtime call binds it
  if (cudaFree(nullptr) != cudaSuccess) return -3;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<char> cubin;
  const int rc = jit_cubin(jm, p, rowptr, colidx, value, &cubin, log);
  if (rc != 0) return rc;
  CUmodule mod = nullptr;
  CUfunction f = nullptr;
  if (d.load(&mod, cubin.data()) != CUDA_SUCCESS) {
    jm.units.clear();
    return -3;
  }
  jm.module = mod;
  if (d.get(&f, mod, "escoin_jit_sconv") != CUDA_SUCCESS ||
      d.setattr(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, p.smem_bytes) != CUDA_SUCCESS) {
    jit_free(jm);
    return -3;
  }
  jm.func = f;
  if (p.perm > 0 && !jm.reordered && p.nphase > 0) {
    const std::vector<uint16_t> tab = perm_table(p);
    if (cudaMalloc(&jm.d_perm, tab.size() * 2) != cudaSuccess ||
        cudaMemcpy(jm.d_perm, tab.data(), tab.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess) {
      jit_free(jm);
      return -3;
    }
  }
  d.getattr(&jm.regs, CU_FUNC_ATTRIBUTE_NUM_REGS, f);
  d.getattr(&jm.local_bytes, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, f);
  jm.compile_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return 0;
}

int jit_compile_only(const char* ptx, size_t* cubin_bytes) {
  std::vector<char> cubin;
  bool hit = false;
  if (compile_ptx(std::string(ptx), Opts{kOpts[0], kOpts[1]}, &cubin, nullptr, &hit) != 0) return -2;
  *cubin_bytes = cubin.size();
  return 0;
}

std::string jit_ptx_text(const JitPlan& p, const int32_t* rowptr, const int32_t* colidx, const float* value,
                         int g_lo, int g_hi) {
  if (g_hi <= 0) g_hi = p.nmg;
  return gen_ptx(p, rowptr, colidx, value, g_lo, g_hi, -1);
}

std::string jit_label(const JitModule& jm) {
  const JitPlan& p = jm.plan;
  char b[160];
  snprintf(b, sizeof b, "jit_q%d_p%d%s%s_cc%d_ns%d_w%d%s_b%d_pf%d_mb%d_u%d_sw%d_v%d%s%s%s%s", p.Q, p.P,
           p.f2 ? "x2" : "", p.Pi != p.P ? (p.co ? "h1" : "h0") : "", p.CC, p.NS, p.warps, p.pw ? "p" : "", p.minb, p.pf, p.mb, int(jm.units.size()), p.SWs, p.V, jm.reordered ? "_ro" : "",
           (p.perm > 0 && !jm.reordered && p.nphase > 0) ? "_dl" : "", p.sp > 1 ? ("_s" + std::to_string(p.sp)).c_str() : "",
           p.ks > 1 ? ("_k" + std::to_string(p.ks)).c_str() : "");
  return b;
}

void jit_free(JitModule& jm) {
  if (jm.d_perm) cudaFree(jm.d_perm);
  jm.d_perm = nullptr;
  if (jm.d_ws) cudaFree(jm.d_ws);
  jm.d_ws = nullptr;
  jm.ws_elems = 0;
  if (jm.module && driver().ok) driver().unload(static_cast<CUmodule>(jm.module));
  jm.module = nullptr;
  jm.func = nullptr;
  jm.units.clear();
}

int jit_launch(const JitModule& jm, const float* in, float* out, const float* bias, int relu, int N,
               cudaStream_t s, float* ws) {
  const JitPlan& p = jm.plan;
  const int64_t pixels = int64_t(N) * p.E * p.Fi;  // items (pixels or horizontal pairs)
  const int64_t tiles = (pixels + p.T - 1) / p.T;
  const int64_t last_pos = (int64_t(N) * (p.H + p.pad) + p.pad) * p.SWs + p.L;  // staged positions stay int32
  if (!jm.func) return -1;
  if (pixels > 0x7fffffff || last_pos > 0x7fffffff || tiles > 65535) return -2;  // int32 positions, grid.y
  unsigned relu_u = relu ? 1u : 0u, n_u = unsigned(N);
  const void* a_in = in;
  void* a_out = out;
  const void* a_bias = bias;
  const void* a_perm = jm.d_perm;
  void* a_ws = ws;
  if (p.ks > 1 && !ws) return -1;
  void* args[] = {&a_in, &a_out, &a_bias, &relu_u, &n_u, &a_perm, &a_ws};
  const CUresult r = driver().launch(static_cast<CUfunction>(jm.func), unsigned(p.nmg), unsigned(tiles), unsigned(p.ks),
                                     unsigned((p.warps + (p.pw ? 1 : 0)) * 32), 1, 1, unsigned(p.smem_bytes), (CUstream)s, args,
                                     nullptr);
  return r == CUDA_SUCCESS ? 0 : -1;
}

}  // namespace escoin
