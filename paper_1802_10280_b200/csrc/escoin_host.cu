// escoin_host.cu — the C-ABI of include/escoin.h: weight stretching, handle
// lifetime, the kernel-side derived format (DS-6), tiling choice and the
// forward dispatch.  No exceptions or CUDA errors cross the ABI.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "escoin.h"
#include "escoin_internal.h"
#include "jit_sconv.h"

using namespace escoin;

struct escoin_csr {
  int M = 0, C = 0, H = 0, W = 0, K = 0, stride = 0, pad = 0, E = 0, F = 0;
  int64_t nnz = 0;
  std::vector<int32_t> rowptr, colidx;
  std::vector<float> value;
  // device side
  int device = -1;
  bool on_device = false;
  bool borrowed = false;  // CSR arrays borrowed (escoin_csr_wrap_device)
  int32_t* d_rowptr = nullptr;
  int32_t* d_colidx = nullptr;
  float* d_value = nullptr;
  // selected variant + derived format
  int kernel = -1;  // 0 = paper mapping, 1.. = tiled variant (index + 1)
  int2* d_recs = nullptr;
  int* d_sched = nullptr;
  int* d_sched_off = nullptr;
  TiledArgs targs{};  // pointers/tiling filled at DS-6 build; tensors per forward
  std::vector<JitModule*> jits;  // pattern-specialised kernels compiled for this handle (escoin_csr_jit)
  JitModule* jit = nullptr;      // the selected one
  float* d_dense = nullptr;      // dense [M][C][K][K] weights of the dense engine (ESCOIN_KERNEL_DENSE_TC)
  std::mutex jit_mu;             // escoin_csr_jit may be called from several host threads
};

namespace {

constexpr int64_t kInt32Max = 2147483647LL;
// ESCOIN_DEBUG_CODES=1|2: timing experiments only (wrong results) — collapses
// the dispatch codes to isolate branch-target / instruction-cache effects.
const int g_debug_kernel = [] {
  const char* e = std::getenv("ESCOIN_DEBUG_KERNEL");
  return e ? std::atoi(e) : 0;
}();
const int g_debug_code_mode = [] {
  const char* e = std::getenv("ESCOIN_DEBUG_CODES");
  return e ? std::atoi(e) : 0;
}();

int ceil_div(int a, int b) { return (a + b - 1) / b; }

int out_dim(int H, int K, int stride, int pad) {
  if (H < 1 || K < 1 || stride < 1 || pad < 0) return -1;
  const int span = H + 2 * pad - K;
  return span < 0 ? -1 : span / stride + 1;
}

void free_ds6(escoin_csr* h) {
  if (h->d_recs) cudaFree(h->d_recs);
  if (h->d_sched) cudaFree(h->d_sched);
  if (h->d_sched_off) cudaFree(h->d_sched_off);
  h->d_recs = nullptr;
  h->d_sched = nullptr;
  h->d_sched_off = nullptr;
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) return;
    ok = (prev == dev) || cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// ---------------------------------------------------------------- tiling
struct Tiling {
  int WM, WP, NB, TR, PR, PC, PCs, SR, SC, SCs, plane;  // PCs >= PC: patch columns per slot row
  int flat;                                              // full-row variants: slots over (image, row)
  int mos;                                               // > 0: mosaic of the batch, mos images per super-row
  double cost;
};

// Mosaic tiling (stride 1, "same" padding): the batch is laid out as ONE
// super-image, images on a grid of `mos` columns, separated by pad zero
// rows/columns (the zero ring of one image is the neighbour's), so 4x4
// patches tile 13x13 or 14x14 images with little waste.  Super-image size for
// a batch of N images:
int mosaic_rows(const escoin_csr* h, int mos, int N) { return ceil_div(N, mos) * (h->H + h->pad) - h->pad; }
int mosaic_cols(const escoin_csr* h, int mos) { return mos * (h->W + h->pad) - h->pad; }

// Max shared-memory bank-group conflict degree of the window LDS.128 pattern
// (8 lanes per quarter-warp, 16-byte accesses) for a candidate layout.
int window_conflicts(const TiledVariant& v, const Tiling& t, int CC) {
  int worst = 0;
  for (int wp = 0; wp < t.WP; ++wp) {
    for (int qtr = 0; qtr < 4; ++qtr) {
      int cnt[8] = {0};
      int addrs[8];
      int na = 0;
      for (int l = qtr * 8; l < qtr * 8 + 8; ++l) {
        const int slot = wp * 32 + l;
        const int per_img = t.TR * t.PCs;
        int img = slot / per_img, pr = (slot % per_img) / t.PCs, pc = slot % t.PCs;
        if (t.flat) { img = slot / t.PR; pr = slot % t.PR; pc = 0; }
        if (pc >= t.PC) pc = t.PC - 1;  // pad lanes read their neighbour's window (broadcast)
        if (img >= t.NB) { img = 0; pr = 0; pc = 0; }
        const int a = img * CC * t.plane + pr * v.PH * v.S * t.SCs + pc * v.PW * v.S * (v.mode == 3 ? 2 : 1);
        bool dup = false;
        for (int i = 0; i < na; ++i) dup |= (addrs[i] == a);
        if (dup) continue;
        addrs[na++] = a;
        cnt[(a / 4) & 7]++;
      }
      for (int g = 0; g < 8; ++g) worst = std::max(worst, cnt[g]);
    }
  }
  return worst;
}

// All feasible tilings of variant v at channel chunk CC, with modelled cost.
// Mode 4 (1x1 row blocks, sconv_1x1.cuh): candidates over WP at chunk CC.
// plane = TP (pixels per CTA tile, one slab row per channel).
bool choose_tiling_1x1(const TiledVariant& v, const escoin_csr* h, int CC, std::vector<Tiling>* cands) {
  if (h->K != 1 || h->stride != 1 || h->pad != 0) return false;
  const int R = v.Q, V = v.PW, HW = h->H * h->W;
  const double dens = h->nnz / (double(h->M) * h->C);
  const double u = 1.0 - std::pow(1.0 - dens, R);  // fraction of channels a warp visits
  const int G = ceil_div(h->M, R);
  bool found = false;
  for (int WP = 1; WP <= 8; WP *= 2) {
    Tiling t{};
    t.WM = 8 / WP;
    t.WP = WP;
    t.NB = 1;
    t.plane = 32 * V * WP;  // TP
    const int TP = t.plane;
    if (2.0 * 4.0 * CC * TP > 110.0 * 1024 * 0.85) continue;
    if (TP / ((HW % 4 == 0) ? 4 : 1) > 4 * kTiledThreads) continue;  // staging units per thread (kMaxQ)
    const int B = ceil_div(G, t.WM);
    const double warp_util = double(G) / (B * t.WM);
    const double ntiles = std::ceil(128.0 * HW / TP);
    const double pix_util = 128.0 * HW / (ntiles * TP);
    const double waves = ntiles * B / (148.0 * v.min_blocks);
    const double wave_eff = waves / std::ceil(waves);
    // issue slots per input channel and lane: visited records x (FFMAs + loads)
    // + staging (TP/256 16-byte copies per channel, ~8 slots each)
    // mode 4 visits u*C channels with R*V FFMAs each; mode 5 visits every
    // nonzero once (V FFMAs + V/4 LDS.128 that cost as much as the FFMAs)
    const double compute = v.mode == 5 ? dens * R * (2.0 * V + 4) : u * (R * V + 2.0 * V / 4 + 8);
    const double staging = (HW % 4 == 0 ? 8.0 / 4 : 8.0) * TP / kTiledThreads;
    t.cost = (compute + staging) / (dens * R * V * pix_util * warp_util * wave_eff);
    if (std::getenv("ESCOIN_DEBUG_TILING"))
      fprintf(stderr, "tiling %s CC=%d WP=%d TP=%d cost=%.3f\n", v.name, CC, WP, TP, t.cost);
    cands->push_back(t);
    found = true;
  }
  return found;
}

bool choose_tiling(const TiledVariant& v, const escoin_csr* h, int CC, std::vector<Tiling>* cands) {
  if (v.mode == 4 || v.mode == 5) return choose_tiling_1x1(v, h, CC, cands);
  if (v.mode == 6 && v.PW != 1) return false;
  const double slab_budget = (v.min_blocks > 1 ? 110.0 : 220.0) * 1024 * 0.85;  // leave room for records
  const int E = h->E, F = h->F;
  const int PR = ceil_div(E, v.PH), PC = ceil_div(F, v.PW);
  const int G = ceil_div(h->M, v.Q);
  const int P = v.PH * v.PW;
  const int XH = (v.PH - 1) * v.S + v.K, XW = (v.PW - 1) * v.S + v.K;
  const double dens = h->nnz / (double(h->M) * h->C * h->K * h->K);
  const int IP = v.mode == 3 ? 2 : 1;  // images per lane; slots and NB count image groups
  bool found = false;
  if (v.full_row && PC != 1) return false;  // full-row variants need the patch to span the output row
  const bool mos_ok = v.S == 1 && v.mode != 3 && !v.full_row && 2 * h->pad + 1 == h->K && E == h->H && F == h->W;
  const char* mos_env = std::getenv("ESCOIN_MOSAIC");  // experiments/tests: only mosaic width k (0 = off)
  const int mos_force = mos_env ? std::atoi(mos_env) : -1;
  for (int mos = 0; mos <= (mos_ok ? 4 : 0); ++mos)
  for (int WP = 1; WP <= 8; WP *= 2)
  for (int pcs_opt = 0; pcs_opt < 3; ++pcs_opt) {
    if (v.full_row && pcs_opt > 0) continue;
    if (mos_force >= 0 && mos != mos_force && mos_ok) continue;
    // mode 7 (row records): lanes over consecutive rows of the mosaic
    // super-image — one row segment per lane, so the patch must span it
    if (v.mode == 7 && (mos == 0 || pcs_opt > 0 || ceil_div(mosaic_cols(h, mos), v.PW) != 1)) continue;
    // mosaic: one tall super-image of the whole (benchmark-size) batch
    const int PRm = mos ? ceil_div(mosaic_rows(h, mos, 128), v.PH) : PR;
    const int PCm = mos ? ceil_div(mosaic_cols(h, mos), v.PW) : PC;
    // slot columns per patch row: PC, or padded to 4 / 8 so quarter-warps of
    // window loads hit distinct 16-byte bank groups (idle lanes in the pad)
    const int PCs = pcs_opt == 0 ? PCm : pcs_opt == 1 ? ((PCm + 3) & ~3) : ((PCm + 7) & ~7);
    if (pcs_opt > 0 && PCs == (pcs_opt == 1 ? PCm : ((PCm + 3) & ~3))) continue;  // duplicate option
    const int WM = 8 / WP;
    const int slots = 32 * WP;
    if (PCs > slots) continue;
    if (v.mode == 6 && PCs > 32) continue;  // tap records: one 32-column slab row block per CTA
    Tiling t{};
    t.WM = WM;
    t.WP = WP;
    t.PR = PRm;
    t.PC = PCm;
    t.PCs = PCs;
    t.mos = mos;
    if (v.full_row) {  // flat (image, row) slots: stage every image a 32*WP-row range can touch
      t.flat = 1;
      t.TR = PR;
      t.NB = ceil_div(slots, PR) + 1;
    } else if (mos) {
      t.NB = 1;
      t.TR = slots / PCs;
      if (t.TR * PCs < slots * 3 / 4) continue;  // too many idle lanes
    } else if (PR * PCs >= slots) {
      t.NB = 1;
      t.TR = std::min(PR, slots / PCs);
    } else {
      t.NB = slots / (PR * PCs);
      t.TR = PR;
    }
    t.SR = (t.TR * v.PH - 1) * v.S + v.K;
    t.SC = ((t.PC * v.PW - 1) * v.S + v.K) * IP;  // floats per slab row (image pairs interleaved)
    const int SC4 = (t.SC + 3) & ~3;
    if (t.SR * h->W > kMaxStagePos * kTiledThreads) continue;  // interior floats per staged plane
    // pick row/plane padding that minimises LDS.128 bank-group conflicts
    // (mode 6: fixed row stride 31*S + K, lanes read consecutive columns)
    int bestc = 1 << 30;
    if (v.mode == 6) {
      bestc = 1;
      t.SCs = 31 * v.S + v.K;
      t.plane = (t.SR * t.SCs + 3) & ~3;
    }
    for (int sp = 0; sp < 8 && v.mode != 6; ++sp) {
      const int SCs = SC4 + 4 * sp;
      for (int pp = 0; pp < 8; ++pp) {
        Tiling u = t;
        u.SCs = SCs;
        u.plane = t.SR * SCs + 4 * pp;
        const int c = window_conflicts(v, u, CC);
        if (c < bestc) {
          bestc = c;
          t.SCs = u.SCs;
          t.plane = u.plane;
        }
      }
    }
    if (2.0 * 4.0 * t.NB * CC * t.plane > slab_budget) continue;  // double-buffered slab must fit
    const double lane_util = t.flat ? 1.0 : double(t.NB * t.TR * t.PC) / slots;
    const double pix_util = mos ? 128.0 * E * F / (double(PRm * v.PH) * (PCm * v.PW))
                                : double(E) * F / (double(PR * v.PH) * (PC * v.PW));
    const int B = ceil_div(G, WM);
    const double warp_util = double(G) / (B * WM);
    // per input channel and thread: records x (FFMAs + dispatch), window loads,
    // bucket overhead; dispatch latency is ~60 issue-slot equivalents per record
    // with 2 CTAs/SM, more with 1; cases beyond ~12 KB of SASS miss the I-cache.
    const int NC = v.Q * v.K * v.K;
    const double code_kb = NC * (P + 9) * 16.0 / 1024.0;
    const double lat = (v.min_blocks > 1 ? 40.0 : 80.0) * (code_kb > 12.0 ? code_kb / 12.0 : 1.0);
    const bool vec = ((v.PW * v.S) % 4 == 0) || PC == 1;
    const double win = vec ? XH * ((XW + 3) / 4) * 4.0 * (bestc > 1 ? bestc : 1) : XH * XW;
    const double work = v.mode >= 2 ? P / 2.0 * IP + 10 : P + 9;  // issue slots per record
    // mode 6: a record per tap where any of the Q channels has a nonzero,
    // Q*P FFMAs + P loads each, no dispatch, no window
    const double u6 = 1.0 - std::pow(1.0 - dens, v.Q);
    // mode 7: a record per (c, kh) where any of K*Q weights is nonzero; per
    // record vector loads of the row + per-kw branch + Q*PW FFMAs per active kw
    const double u7 = 1.0 - std::pow(1.0 - dens, v.K * v.Q);
    const double compute = v.mode == 6 ? v.K * v.K * u6 * (v.Q * P + P + 6) + 10
                           : v.mode == 7 ? v.K * u7 * ((v.PW + v.K + 2) / 4 + 2 + (v.K * v.Q + 3) / 4 + 2 * v.K +
                                                      v.K * u6 * v.Q * P) + 10
                                         : (v.Q * dens * v.K * v.K * (work + lat) + win + 30) / IP;
    const double staging = mos ? 5.0 * t.SR * mos * h->W / kTiledThreads
                               : 5.0 * t.NB * IP * std::min(t.SR, h->H) * h->W / kTiledThreads / IP;
    // wave quantisation of the grid at the benchmark batch (128 images)
    const double nctas = t.flat ? double(ceil_div(128 * PR, slots)) * B
                         : mos  ? double(ceil_div(PRm, t.TR)) * B
                                : double(ceil_div(128, t.NB * IP)) * ceil_div(PR, t.TR) * B;
    const double waves = nctas / (148.0 * v.min_blocks);
    const double wave_eff = waves / std::ceil(waves);
    t.cost = (compute + staging) / (lane_util * pix_util * warp_util * wave_eff * v.Q * P);
    if (std::getenv("ESCOIN_DEBUG_TILING"))
      fprintf(stderr, "tiling %s CC=%d mos=%d WP=%d PCs=%d NB=%d TR=%d SCs=%d plane=%d conflicts=%d cost=%.3f\n",
              v.name, CC, mos, WP, PCs, t.NB, t.TR, t.SCs, t.plane, bestc, t.cost);
    cands->push_back(t);
    found = true;
  }
  return found;
}

// ---------------------------------------------------------------- DS-6
// Records of output-channel group g (channels g*Q .. g*Q+Q-1) bucketed by
// input channel c, grouped into m-blocks of WM groups and channel chunks of
// CC.  Each warp stream of one (m-block, chunk):
//   START{kHdrBase, c_first}  then for each c with records:
//   REC*  END{Q*K*K, c_next}          (c_first / c_next = -1: no more buckets)
// REC = {code = q*K*K + kh*K + kw, bits(value)} in ascending (q, kh, kw) —
// i.e. the CSR order of each row.  Built once on the host from the stretched
// CSR; never part of the bit-exact contract.
struct DS6 {
  std::vector<int2> recs;
  std::vector<int> sched, sched_off;
  int max_block = 0;
};

// Mode 4 streams: per (m-block, chunk, warp) a header {count} and one record
// per input channel where any of the warp's R rows has a nonzero:
// {byte offset of the channel's slab row, w[0..R-1]} (absent weights +0.0f),
// padded to 16-byte units.  Ascending c == the CSR order of every row.
void build_ds_1x1(const escoin_csr* h, const TiledVariant& v, int WM, int CC, int TP, DS6* out) {
  const int R = v.Q, M = h->M, C = h->C;
  const int G = ceil_div(M, R), B = ceil_div(G, WM), NK = ceil_div(C, CC);
  const int RS2 = 2 * ((1 + R + 3) / 4);  // int2 units per record
  const int64_t HW = int64_t(h->H) * h->W;
  std::vector<float> wd(size_t(M) * C, 0.0f);
  std::vector<unsigned char> nz(size_t(M) * C, 0);
  for (int m = 0; m < M; ++m)
    for (int64_t j = h->rowptr[m]; j < h->rowptr[m + 1]; ++j) {
      const int c = int(h->colidx[j] / HW);
      wd[size_t(m) * C + c] = h->value[j];
      nz[size_t(m) * C + c] = 1;
    }
  out->recs.clear();
  out->sched.clear();
  out->sched_off.assign(1, 0);
  out->max_block = 0;
  std::vector<int> woff(WM);
  for (int b = 0; b < B; ++b) {
    for (int k = 0; k < NK; ++k) {
      const int start = int(out->recs.size());
      int total = 0;
      for (int wm = 0; wm < WM; ++wm) {
        woff[wm] = int(out->recs.size()) - start;
        const int g = b * WM + wm;
        if (v.mode == 5) {
          // header: R counts (16-byte padded); then row by row {byte offset, w}
          const size_t hdr = out->recs.size();
          const int nh2 = 2 * ((R + 3) / 4);
          for (int i = 0; i < nh2; ++i) out->recs.push_back(make_int2(0, 0));
          for (int r = 0; r < R; ++r) {
            const int m = g * R + r;
            int cnt = 0;
            for (int cl = 0; cl < CC && g < G && m < M; ++cl) {
              const int c = k * CC + cl;
              if (c >= C) break;
              if (!nz[size_t(m) * C + c]) continue;
              int wb;
              std::memcpy(&wb, &wd[size_t(m) * C + c], 4);
              out->recs.push_back(make_int2(cl * TP * 4, wb));
              ++cnt;
            }
            reinterpret_cast<int*>(&out->recs[hdr])[r] = cnt;
            total += cnt;
          }
          if (out->recs.size() & 1) out->recs.push_back(make_int2(0, 0));
          continue;
        }
        const size_t hdr = out->recs.size();
        out->recs.push_back(make_int2(0, 0));
        out->recs.push_back(make_int2(0, 0));
        int cnt = 0;
        for (int cl = 0; cl < CC && g < G; ++cl) {
          const int c = k * CC + cl;
          if (c >= C) break;
          bool any = false;
          for (int r = 0; r < R && g * R + r < M; ++r) any |= nz[size_t(g * R + r) * C + c] != 0;
          if (!any) continue;
          std::vector<int> rec(RS2 * 2, 0);
          rec[0] = cl * TP * 4;
          for (int r = 0; r < R && g * R + r < M; ++r) std::memcpy(&rec[1 + r], &wd[size_t(g * R + r) * C + c], 4);
          for (int i = 0; i < RS2; ++i) out->recs.push_back(make_int2(rec[2 * i], rec[2 * i + 1]));
          ++cnt;
        }
        out->recs[hdr].x = cnt;
        total += cnt;
      }
      if (total == 0) {  // chunk inactive for this m-block
        out->recs.resize(start);
        continue;
      }
      const int count = int(out->recs.size()) - start;
      out->max_block = std::max(out->max_block, count);
      out->sched.push_back(k);
      out->sched.push_back(start);
      out->sched.push_back(count);
      for (int wm = 0; wm < WM; ++wm) out->sched.push_back(woff[wm]);
    }
    out->sched_off.push_back(int(out->sched.size() / (3 + WM)));
  }
}

// Mode 6 streams (tap records): per (m-block, chunk, warp) a 16-byte header
// {count} and one record per tap (c, kh, kw) — ascending, i.e. CSR order —
// where any of the warp's Q rows has a nonzero: {byte offset (c_local*plane +
// kh*SCs + kw)*4 from the lane's window origin, w[0..Q-1]} (absent: +0.0f),
// padded to 16-byte units.
void build_ds_tap(const escoin_csr* h, const TiledVariant& v, int WM, int CC, int plane, DS6* out) {
  const int Q = v.Q, M = h->M, C = h->C, K = h->K, KK = K * K;
  const int SCs = 31 * h->stride + K;  // the kernel's slab row stride (sconv_tiled.cuh, MODE 6)
  const int G = ceil_div(M, Q), B = ceil_div(G, WM), NK = ceil_div(C, CC);
  const int RS2 = 2 * ((1 + Q + 3) / 4);
  const int64_t HpWp = int64_t(h->H + 2 * h->pad) * (h->W + 2 * h->pad);
  const int Wp = h->W + 2 * h->pad;
  const size_t CKK = size_t(C) * KK;
  std::vector<float> wd(size_t(M) * CKK, 0.0f);
  std::vector<unsigned char> nz(size_t(M) * CKK, 0);
  for (int m = 0; m < M; ++m)
    for (int64_t j = h->rowptr[m]; j < h->rowptr[m + 1]; ++j) {
      const int64_t off = h->colidx[j];
      const int c = int(off / HpWp), rem = int(off - c * HpWp);
      const size_t col = size_t(c) * KK + size_t(rem / Wp) * K + rem % Wp;
      wd[size_t(m) * CKK + col] = h->value[j];
      nz[size_t(m) * CKK + col] = 1;
    }
  out->recs.clear();
  out->sched.clear();
  out->sched_off.assign(1, 0);
  out->max_block = 0;
  std::vector<int> woff(WM), rec(RS2 * 2);
  for (int b = 0; b < B; ++b) {
    for (int k = 0; k < NK; ++k) {
      const int start = int(out->recs.size());
      int total = 0;
      for (int wm = 0; wm < WM; ++wm) {
        woff[wm] = int(out->recs.size()) - start;
        const size_t hdr = out->recs.size();
        out->recs.push_back(make_int2(0, 0));
        out->recs.push_back(make_int2(0, 0));
        const int g = b * WM + wm;
        int cnt = 0;
        for (int cl = 0; cl < CC && g < G; ++cl) {
          const int c = k * CC + cl;
          if (c >= C) break;
          for (int tap = 0; tap < KK; ++tap) {
            const size_t col = size_t(c) * KK + tap;
            bool any = false;
            for (int r = 0; r < Q && g * Q + r < M; ++r) any |= nz[size_t(g * Q + r) * CKK + col] != 0;
            if (!any) continue;
            std::fill(rec.begin(), rec.end(), 0);
            rec[0] = (cl * plane + (tap / K) * SCs + tap % K) * 4;
            for (int r = 0; r < Q && g * Q + r < M; ++r) std::memcpy(&rec[1 + r], &wd[size_t(g * Q + r) * CKK + col], 4);
            for (int i = 0; i < RS2; ++i) out->recs.push_back(make_int2(rec[2 * i], rec[2 * i + 1]));
            ++cnt;
          }
        }
        out->recs[hdr].x = cnt;
        total += cnt;
      }
      if (total == 0) {
        out->recs.resize(start);
        continue;
      }
      const int count = int(out->recs.size()) - start;
      out->max_block = std::max(out->max_block, count);
      out->sched.push_back(k);
      out->sched.push_back(start);
      out->sched.push_back(count);
      for (int wm = 0; wm < WM; ++wm) out->sched.push_back(woff[wm]);
    }
    out->sched_off.push_back(int(out->sched.size() / (3 + WM)));
  }
}

// Mode 7 streams (row records): per (m-block, chunk, warp) a 16-byte header
// {count} and one record per (c, kh) — ascending — where any of the warp's Q
// rows has a nonzero: {byte offset (c_local*plane + kh*SCs)*4 from the lane's
// window origin, kw-mask (bit kw: some q has a nonzero), 0, 0} followed by the
// K*Q weights w[kw*Q + q] (absent: +0.0f), padded to 16 bytes.
void build_ds_row(const escoin_csr* h, const TiledVariant& v, int WM, int CC, int plane, int SCs, DS6* out) {
  const int Q = v.Q, M = h->M, C = h->C, K = h->K, KK = K * K;
  const int G = ceil_div(M, Q), B = ceil_div(G, WM), NK = ceil_div(C, CC);
  const int RS2 = 2 * (1 + (K * Q + 3) / 4);
  const int64_t HpWp = int64_t(h->H + 2 * h->pad) * (h->W + 2 * h->pad);
  const int Wp = h->W + 2 * h->pad;
  const size_t CKK = size_t(C) * KK;
  std::vector<float> wd(size_t(M) * CKK, 0.0f);
  std::vector<unsigned char> nz(size_t(M) * CKK, 0);
  for (int m = 0; m < M; ++m)
    for (int64_t j = h->rowptr[m]; j < h->rowptr[m + 1]; ++j) {
      const int64_t off = h->colidx[j];
      const int c = int(off / HpWp), rem = int(off - c * HpWp);
      const size_t col = size_t(c) * KK + size_t(rem / Wp) * K + rem % Wp;
      wd[size_t(m) * CKK + col] = h->value[j];
      nz[size_t(m) * CKK + col] = 1;
    }
  out->recs.clear();
  out->sched.clear();
  out->sched_off.assign(1, 0);
  out->max_block = 0;
  std::vector<int> woff(WM), rec(RS2 * 2);
  for (int b = 0; b < B; ++b) {
    for (int k = 0; k < NK; ++k) {
      const int start = int(out->recs.size());
      int total = 0;
      for (int wm = 0; wm < WM; ++wm) {
        woff[wm] = int(out->recs.size()) - start;
        const size_t hdr = out->recs.size();
        out->recs.push_back(make_int2(0, 0));
        out->recs.push_back(make_int2(0, 0));
        const int g = b * WM + wm;
        int cnt = 0;
        for (int cl = 0; cl < CC && g < G; ++cl) {
          const int c = k * CC + cl;
          if (c >= C) break;
          for (int kh = 0; kh < K; ++kh) {
            unsigned mask = 0;
            std::fill(rec.begin(), rec.end(), 0);
            for (int kw = 0; kw < K; ++kw)
              for (int r = 0; r < Q && g * Q + r < M; ++r) {
                const size_t idx = size_t(g * Q + r) * CKK + size_t(c) * KK + kh * K + kw;
                if (nz[idx]) mask |= 1u << kw;
                std::memcpy(&rec[4 + kw * Q + r], &wd[idx], 4);
              }
            if (!mask) continue;
            rec[0] = (cl * plane + kh * SCs) * 4;
            rec[1] = int(mask);
            for (int i = 0; i < RS2; ++i) out->recs.push_back(make_int2(rec[2 * i], rec[2 * i + 1]));
            ++cnt;
          }
        }
        out->recs[hdr].x = cnt;
        total += cnt;
      }
      if (total == 0) {
        out->recs.resize(start);
        continue;
      }
      const int count = int(out->recs.size()) - start;
      out->max_block = std::max(out->max_block, count);
      out->sched.push_back(k);
      out->sched.push_back(start);
      out->sched.push_back(count);
      for (int wm = 0; wm < WM; ++wm) out->sched.push_back(woff[wm]);
    }
    out->sched_off.push_back(int(out->sched.size() / (3 + WM)));
  }
}

void build_ds6(const escoin_csr* h, const TiledVariant& v, int WM, int CC, int plane, int SCs, DS6* out) {
  if (v.mode == 7) return build_ds_row(h, v, WM, CC, plane, SCs, out);
  if (v.mode == 4 || v.mode == 5) return build_ds_1x1(h, v, WM, CC, plane, out);
  if (v.mode == 6) return build_ds_tap(h, v, WM, CC, plane, out);
  const int Q = v.Q, K = h->K;
  const int G = ceil_div(h->M, Q), B = ceil_div(G, WM), NK = ceil_div(h->C, CC);
  const int64_t HpWp = int64_t(h->H + 2 * h->pad) * (h->W + 2 * h->pad);
  const int Wp = h->W + 2 * h->pad;
  const int64_t nbuckets = int64_t(B) * NK * WM * CC;
  std::vector<int64_t> cnt(nbuckets + 1, 0);
  std::vector<int64_t> key(h->nnz);
  std::vector<int> code(h->nnz);
  for (int m = 0; m < h->M; ++m) {
    const int g = m / Q, q = m % Q, b = g / WM, wm = g % WM;
    for (int64_t j = h->rowptr[m]; j < h->rowptr[m + 1]; ++j) {
      const int64_t off = h->colidx[j];
      const int c = int(off / HpWp);
      const int rem = int(off - c * HpWp);
      const int kh = rem / Wp, kw = rem % Wp;
      const int k = c / CC, cl = c % CC;
      key[j] = ((int64_t(b) * NK + k) * WM + wm) * CC + cl;
      code[j] = (q * K + kh) * K + kw;
      if (g_debug_code_mode == 1) code[j] = 0;               // experiment: one branch target
      else if (g_debug_code_mode == 2) code[j] = q * K * K;  // experiment: one target per q
      cnt[key[j] + 1]++;
    }
  }
  for (int64_t i = 0; i < nbuckets; ++i) cnt[i + 1] += cnt[i];
  std::vector<int2> sorted(h->nnz);
  {
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t j = 0; j < h->nnz; ++j) {
      int2 r;
      r.x = code[j];
      std::memcpy(&r.y, &h->value[j], 4);
      sorted[pos[key[j]]++] = r;
    }
  }
  const int END = Q * K * K;
  out->recs.clear();
  out->sched.clear();
  out->sched_off.assign(1, 0);
  out->max_block = 0;
  for (int b = 0; b < B; ++b) {
    for (int k = 0; k < NK; ++k) {
      const int64_t first = ((int64_t(b) * NK + k) * WM) * CC;
      const int64_t last = first + int64_t(WM) * CC;
      if (cnt[last] == cnt[first]) continue;  // chunk inactive for this m-block
      const int start = int(out->recs.size());
      std::vector<int> woff(WM);
      for (int wm = 0; wm < WM; ++wm) {
        std::vector<int> cls;
        for (int cl = 0; cl < CC; ++cl) {
          const int64_t bk = first + int64_t(wm) * CC + cl;
          if (cnt[bk + 1] != cnt[bk]) cls.push_back(cl);
        }
        if (v.link) {
          // Linked stream: header {idx(item0)}, then item i = {idx(item i+1)
          // relative to item i's jump list, payload(i)} (+ {abs(i+1), 0} when
          // rel_d > 0); items: NEXT{END, window offset} REC* ... DONE{END+1}.
          woff[wm] = int(out->recs.size()) - start;
          std::vector<int2> items;
          for (size_t i = 0; i < cls.size(); ++i) {
            const int64_t bk = first + int64_t(wm) * CC + cls[i];
            items.push_back(make_int2(END, cls[i] * plane * 4));
            for (int64_t r = cnt[bk]; r < cnt[bk + 1]; ++r) items.push_back(sorted[r]);
          }
          items.push_back(make_int2(END + 1, 0));
          const int D = v.rel_d;
          auto enc = [&](int pred, int abs) {  // pred < 0: START / NEXT (full list)
            if (D == 0 || pred < 0 || pred >= END) return abs;
            if (abs == END) return D;
            if (abs == END + 1) return D + 1;
            if (abs - pred - 1 >= 0 && abs - pred - 1 < D) return abs - pred - 1;
            return D + 2;  // FAR
          };
          auto put = [&](int idx, int payload, int abs) {
            out->recs.push_back(make_int2(idx, payload));
            if (D > 0) out->recs.push_back(make_int2(abs, 0));
          };
          put(items[0].x, 0, items[0].x);
          for (size_t i = 0; i < items.size(); ++i) {
            const bool last = i + 1 == items.size();
            const int nabs = last ? 0 : items[i + 1].x;
            put(last ? 0 : enc(items[i].x, nabs), items[i].y, nabs);
          }
          put(0, 0, 0);  // depth-2 loops prefetch one record past DONE
          if (out->recs.size() & 1) out->recs.push_back(make_int2(0, 0));
        } else if ((v.mode == 0 || v.mode == 2 || v.mode == 3) && v.rel_d == 0) {
          woff[wm] = int(out->recs.size()) - start;
          // One stream per warp and chunk, run by ONE inline-PTX dispatch loop:
          // per bucket NEXT{END, byte offset of channel c's window} REC*, then
          // DONE{END+1}.  NEXT reloads the input window in registers.
          for (size_t i = 0; i < cls.size(); ++i) {
            const int64_t bk = first + int64_t(wm) * CC + cls[i];
            out->recs.push_back(make_int2(END, cls[i] * plane * 4));
            for (int64_t r = cnt[bk]; r < cnt[bk + 1]; ++r) out->recs.push_back(sorted[r]);
          }
          out->recs.push_back(make_int2(END + 1, 0));
        } else if (v.rel_d > 0) {
          // Same stream, 16-byte records {idx, payload, abs, 0}: idx indexes the
          // predecessor's jump list (full list after START/NEXT; after case c
          // the D codes following c, then NEXT, DONE, FAR).
          woff[wm] = int(out->recs.size()) - start;
          const int D = v.rel_d;
          int prev = -1;  // -1: START or NEXT (full list)
          auto emit = [&](int abs, int payload) {
            int idx;
            if (prev < 0) idx = abs;
            else if (abs == END) idx = D;
            else if (abs == END + 1) idx = D + 1;
            else if (abs - prev - 1 >= 0 && abs - prev - 1 < D) idx = abs - prev - 1;
            else idx = D + 2;  // FAR
            out->recs.push_back(make_int2(idx, payload));
            out->recs.push_back(make_int2(abs, 0));
            prev = (abs >= END) ? -1 : abs;
          };
          for (size_t i = 0; i < cls.size(); ++i) {
            const int64_t bk = first + int64_t(wm) * CC + cls[i];
            emit(END, cls[i] * plane * 4);
            for (int64_t r = cnt[bk]; r < cnt[bk + 1]; ++r) emit(sorted[r].x, sorted[r].y);
          }
          emit(END + 1, 0);
        } else {
          // 16-byte units: header {c, 0, 0, 0}, then the dense Q*K*K weights of
          // the bucket in (tap, q) order, zero-padded to a multiple of 4.
          if (out->recs.size() & 1) out->recs.push_back(make_int2(0, 0));
          woff[wm] = int(out->recs.size()) - start;
          const int NS = Q * K * K, NS4 = (NS + 3) & ~3;
          std::vector<float> dense(NS4);
          for (size_t i = 0; i < cls.size(); ++i) {
            const int64_t bk = first + int64_t(wm) * CC + cls[i];
            out->recs.push_back(make_int2(cls[i], 0));
            out->recs.push_back(make_int2(0, 0));
            std::fill(dense.begin(), dense.end(), 0.0f);
            for (int64_t r = cnt[bk]; r < cnt[bk + 1]; ++r) {
              const int cd = sorted[r].x;  // (q*K + kh)*K + kw
              const int q = cd / (K * K), tap = cd % (K * K);
              std::memcpy(&dense[tap * Q + q], &sorted[r].y, 4);
            }
            for (int i2 = 0; i2 < NS4; i2 += 2) {
              int2 pr;
              std::memcpy(&pr.x, &dense[i2], 4);
              std::memcpy(&pr.y, &dense[i2 + 1], 4);
              out->recs.push_back(pr);
            }
          }
          out->recs.push_back(make_int2(kDone, 0));
          out->recs.push_back(make_int2(0, 0));
        }
      }
      if (out->recs.size() & 1) out->recs.push_back(make_int2(kDone, 0));
      const int count = int(out->recs.size()) - start;
      out->max_block = std::max(out->max_block, count);
      out->sched.push_back(k);
      out->sched.push_back(start);
      out->sched.push_back(count);
      for (int wm = 0; wm < WM; ++wm) out->sched.push_back(woff[wm]);
    }
    out->sched_off.push_back(int(out->sched.size() / (3 + WM)));
  }
}

template <typename T>
int upload(const std::vector<T>& v, T** d, cudaStream_t s) {
  const size_t bytes = std::max<size_t>(v.size() * sizeof(T), 16);
  if (cudaMalloc(reinterpret_cast<void**>(d), bytes) != cudaSuccess) return ESCOIN_ERR_ALLOC;
  if (!v.empty() && cudaMemcpyAsync(*d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return ESCOIN_ERR_CUDA;
  return ESCOIN_OK;
}

// Host-only planning of a tiled variant: tiling, channel chunk CC, derived
// format and shared-memory budget.  Returns ESCOIN_ERR_UNSUPPORTED when the
// variant cannot tile this layer.
int plan_tiled(const escoin_csr* h, const TiledVariant& v, int rank, Tiling* t, int* CCout, DS6* ds,
               size_t* smem, size_t* stage_f_out, size_t* stage_r_out, int* nstages) {
  // Candidates over every channel-chunk size, ranked by modelled cost (plus the
  // per-chunk barrier/staging latency ~1/CC); rank 0 is the model's choice,
  // escoin_csr_autotune also measures ranks 1..2.
  struct Cand {
    Tiling t;
    int CC;
    double cost;
  };
  std::vector<Cand> all;
  for (int CC = 32; CC >= 1; CC /= 2) {
    std::vector<Tiling> cs;
    choose_tiling(v, h, CC, &cs);
    for (const Tiling& tt : cs) all.push_back({tt, CC, tt.cost * (1.0 + 2.0 / CC)});
  }
  std::stable_sort(all.begin(), all.end(), [](const Cand& a, const Cand& b) { return a.cost < b.cost; });
  // Feasible plans of the best candidates, each at the deepest pipeline that
  // fits (3 stages let warps drift two chunks apart; 2 stages lock them to one
  // — modelled as +12% time); ESCOIN_STAGES forces a depth (experiments).
  struct Plan {
    size_t ci;
    int ns;
    size_t stage_f, stage_r, sm;
    double cost;
  };
  std::vector<Plan> plans;
  std::vector<DS6> dss;
  const size_t limit = size_t(v.min_blocks > 1 ? 110 : 220) * 1024;
  int force = 0;
  if (const char* e = std::getenv("ESCOIN_STAGES")) force = std::max(2, std::min(kMaxStages, std::atoi(e)));
  for (size_t ci = 0; ci < all.size() && plans.size() < size_t(rank) + 6; ++ci) {
    const Cand& c = all[ci];
    // ranks are distinct geometries (a different CC alone barely changes time)
    bool dup = false;
    for (const Plan& q : plans) {
      const Tiling& u = all[q.ci].t;
      dup |= u.mos == c.t.mos && u.WP == c.t.WP && u.PCs == c.t.PCs && u.NB == c.t.NB && u.TR == c.t.TR;
    }
    if (dup) continue;
    DS6 dd;
    build_ds6(h, v, c.t.WM, c.CC, c.t.plane, c.t.SCs, &dd);
    const size_t stage_f = (size_t(c.t.NB) * c.CC * c.t.plane + 3) & ~size_t(3);
    // slack: the dispatch loop prefetches up to two records (16 B each for
    // rel_d variants) past a warp's DONE
    const size_t stage_r = ((dd.max_block + 1) & ~1) + 4;
    int ns = force ? force : 3;
    while (ns > 2 && size_t(ns) * (stage_f * 4 + stage_r * 8) > limit) --ns;
    const size_t sm = size_t(ns) * (stage_f * 4 + stage_r * 8);
    if (sm > limit) continue;
    plans.push_back({dss.size(), ns, stage_f, stage_r, sm, c.cost * (ns == 2 ? 1.12 : 1.0)});
    dss.push_back(std::move(dd));
    plans.back().ci = ci;
  }
  std::vector<size_t> order(plans.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) { return plans[x].cost < plans[y].cost; });
  if (size_t(rank) < order.size()) {
    const size_t pi = order[rank];
    const Plan& p = plans[pi];
    *nstages = p.ns;
    *t = all[p.ci].t;
    *CCout = all[p.ci].CC;
    *ds = std::move(dss[pi]);
    *smem = p.sm;
    *stage_f_out = p.stage_f;
    *stage_r_out = p.stage_r;
    return ESCOIN_OK;
  }
  return ESCOIN_ERR_UNSUPPORTED;
}

// Build + upload the derived format of tiled variant `vi` (index into the table).
int prepare_tiled(escoin_csr* h, int vi, int rank, cudaStream_t s) {
  int nv = 0;
  const TiledVariant* tv = tiled_variants(&nv);
  const TiledVariant& v = tv[vi];
  int CC = 0;
  Tiling t{};
  DS6 ds;
  size_t smem = 0, stage_f = 0, stage_r = 0;
  int ns = 2;
  const int prc = plan_tiled(h, v, rank, &t, &CC, &ds, &smem, &stage_f, &stage_r, &ns);
  if (prc != ESCOIN_OK) return prc;
  h->targs.NS = ns;
  h->targs.stage_floats = int(stage_f);
  h->targs.stage_recs = int(stage_r);
  free_ds6(h);
  int rc;
  if ((rc = upload(ds.recs, &h->d_recs, s)) != ESCOIN_OK) return rc;
  if ((rc = upload(ds.sched, &h->d_sched, s)) != ESCOIN_OK) return rc;
  if ((rc = upload(ds.sched_off, &h->d_sched_off, s)) != ESCOIN_OK) return rc;
  if (cudaStreamSynchronize(s) != cudaSuccess) return ESCOIN_ERR_CUDA;
  TiledArgs& a = h->targs;
  a.M = h->M;
  a.C = h->C;
  a.H = h->H;
  a.W = h->W;
  a.E = h->E;
  a.F = h->F;
  a.pad = h->pad;
  a.PR = t.PR;
  a.PC = t.PC;
  a.PCs = t.PCs;
  a.WM = t.WM;
  a.WP = t.WP;
  a.NB = t.NB;
  a.IP = v.mode == 3 ? 2 : 1;
  a.flat = t.flat;
  a.mos = t.mos;
  a.TR = t.TR;
  a.SR = t.SR;
  a.SCs = t.SCs;
  a.plane = t.plane;
  a.CC = CC;
  a.tiles_r = (v.mode == 4 || v.mode == 5) ? 1 : ceil_div(t.PR, t.TR);
  a.TP = t.plane;
  a.vec16 = (h->H * h->W) % 4 == 0 ? 1 : 0;
  a.B = int(ds.sched_off.size()) - 1;
  a.smem_bytes = int(smem);
  a.recs = h->d_recs;
  a.sched = h->d_sched;
  a.sched_off = h->d_sched_off;
  a.sched_stride = 3 + t.WM;
  return ESCOIN_OK;
}

// Default variant (before/without escoin_csr_autotune): lowest modelled cost.
int auto_kernel(const escoin_csr* h) {
  int nv = 0;
  const TiledVariant* tv = tiled_variants(&nv);
  int best = 0;
  double best_cost = 0.0;
  for (int i = 0; i < nv; ++i)
    if (tv[i].K == h->K && tv[i].S == h->stride) {
      std::vector<Tiling> cs;
      if (!choose_tiling(tv[i], h, 8, &cs)) continue;
      for (const Tiling& t : cs)
        if (best == 0 || t.cost < best_cost) {
          best = i + 1;
          best_cost = t.cost;
        }
    }
  return best;
}

// Pattern-specialised kernel (jit_sconv.cpp): plan, generate, compile, load.
// tun = {Q, P, CC, NS, warps, minb, prefetch, mbarrier, units, vec, reorder, sws, perm, split, pair, hp, pw, ks} (<= 0: default;
// prefetch < 0 = off) or NULL.
int build_jit(escoin_csr* h, int n_hint, const int* tun) {
  JitPlan p;
  if (tun) {
    p.Q = tun[0]; p.P = tun[1]; p.CC = tun[2]; p.NS = tun[3]; p.warps = tun[4]; p.minb = tun[5]; p.pf = tun[6]; p.mb = tun[7];
    p.units = tun[8]; p.vec = tun[9]; p.reorder = tun[10]; p.sws = tun[11]; p.perm = tun[12]; p.split = tun[13]; p.pair = tun[14]; p.hp = tun[15]; p.pw = tun[16]; p.ks = tun[17];
  }
  if (p.P > 8 || p.Q > 256 || p.CC > 64 || p.NS > 6 || p.warps > 32 || p.minb > 8 || p.units > 32)
    return ESCOIN_ERR_UNSUPPORTED;
  const double density = double(h->nnz) / (double(h->M) * h->C * h->K * h->K);
  if (jit_plan(p, h->C, h->H, h->W, h->M, h->K, h->stride, h->pad, n_hint, density) != 0)
    return ESCOIN_ERR_UNSUPPORTED;
  if (int64_t(p.warps + p.pw) * 32 * p.minb > 2048) return ESCOIN_ERR_UNSUPPORTED;
  if (h->rowptr.size() != size_t(h->M) + 1) return ESCOIN_ERR_UNSUPPORTED;
  auto same = [&](const JitPlan& q) {
    return q.Q == p.Q && q.P == p.P && q.CC == p.CC && q.NS == p.NS && q.warps == p.warps && q.minb == p.minb &&
           q.pf == p.pf && q.mb == p.mb && q.units == p.units && q.T == p.T && q.L == p.L && q.SWs == p.SWs &&
           q.V == p.V && q.reorder == p.reorder && q.sws == p.sws && q.perm == p.perm &&
           q.split == p.split && q.f2 == p.f2 && q.Pi == p.Pi && q.co == p.co && q.pw == p.pw && q.ks == p.ks;
  };
  {
    std::lock_guard<std::mutex> lk(h->jit_mu);
    for (JitModule* jm : h->jits)  // this tuning was compiled before: select it
      if (same(jm->plan)) {
        h->jit = jm;
        h->kernel = ESCOIN_KERNEL_JIT;
        return ESCOIN_OK;
      }
  }
  JitModule* jm = new (std::nothrow) JitModule();
  if (!jm) return ESCOIN_ERR_ALLOC;
  const int rc = jit_build(*jm, p, h->rowptr.data(), h->colidx.data(), h->value.data(), nullptr);
  if (rc != 0) {
    delete jm;
    return rc == -2 ? ESCOIN_ERR_UNSUPPORTED : ESCOIN_ERR_CUDA;
  }
  std::lock_guard<std::mutex> lk(h->jit_mu);
  for (JitModule* o : h->jits)  // compiled concurrently by another thread meanwhile: keep that one
    if (same(o->plan)) {
      jit_free(*jm);
      delete jm;
      h->jit = o;
      h->kernel = ESCOIN_KERNEL_JIT;
      return ESCOIN_OK;
    }
  h->jits.push_back(jm);
  h->jit = jm;
  h->kernel = ESCOIN_KERNEL_JIT;
  return ESCOIN_OK;
}

int set_kernel(escoin_csr* h, int id, cudaStream_t s, int rank = 0) {
  int nv = 0;
  const TiledVariant* tv = tiled_variants(&nv);
  if (id == ESCOIN_KERNEL_DENSE_TC) {  // dense tcgen05 engine: the pruned weights re-densified on the device
    if (!h->d_dense) {
      if (cudaMalloc(&h->d_dense, sizeof(float) * size_t(h->M) * h->C * h->K * h->K) != cudaSuccess) {
        h->d_dense = nullptr;
        return ESCOIN_ERR_ALLOC;
      }
      if (launch_densify(h->d_rowptr, h->d_colidx, h->d_value, h->M, h->C, h->K, h->H + 2 * h->pad,
                         h->W + 2 * h->pad, h->d_dense, s) != 0 ||
          cudaStreamSynchronize(s) != cudaSuccess)
        return ESCOIN_ERR_CUDA;
    }
    free_ds6(h);
    h->kernel = id;
    return ESCOIN_OK;
  }
  if (id == ESCOIN_KERNEL_JIT) {
    if (!h->jit) {
      const int rc = build_jit(h, 128, nullptr);
      if (rc != ESCOIN_OK) return rc;
    }
    free_ds6(h);
    h->kernel = id;
    return ESCOIN_OK;
  }
  if (id == ESCOIN_KERNEL_AUTO) id = auto_kernel(h);
  if (id < 0 || id > nv) return ESCOIN_ERR_UNSUPPORTED;
  if (id > 0 && (tv[id - 1].K != h->K || tv[id - 1].S != h->stride)) return ESCOIN_ERR_UNSUPPORTED;
  if (id > 0) {
    const int rc = prepare_tiled(h, id - 1, rank, s);
    if (rc != ESCOIN_OK) return rc;
  } else {
    free_ds6(h);
  }
  h->kernel = id;
  return ESCOIN_OK;
}

int validate_shape(int M, int C, int H, int W, int K, int stride, int pad, int* E, int* F) {
  if (M < 1 || C < 1 || H < 1 || W < 1 || K < 1 || stride < 1 || pad < 0) return ESCOIN_ERR_SHAPE;
  *E = out_dim(H, K, stride, pad);
  *F = out_dim(W, K, stride, pad);
  if (*E < 1 || *F < 1) return ESCOIN_ERR_SHAPE;
  const int64_t chw = int64_t(C) * (H + 2 * pad) * (W + 2 * pad);
  if (chw > kInt32Max || int64_t(M) * C * K * K > kInt32Max) return ESCOIN_ERR_OVERFLOW;
  return ESCOIN_OK;
}

}  // namespace

// ================================================================ ABI
extern "C" {

int escoin_csr_stretch(const float* w, int M, int C, int H, int W, int K, int stride, int pad, escoin_csr** out) {
  if (!w || !out) return ESCOIN_ERR_NULL;
  *out = nullptr;
  int E, F;
  int rc = validate_shape(M, C, H, W, K, stride, pad, &E, &F);
  if (rc != ESCOIN_OK) return rc;
  escoin_csr* h = new (std::nothrow) escoin_csr();
  if (!h) return ESCOIN_ERR_ALLOC;
  h->M = M; h->C = C; h->H = H; h->W = W; h->K = K; h->stride = stride; h->pad = pad; h->E = E; h->F = F;
  const int64_t CRS = int64_t(C) * K * K;
  const int64_t Hp = H + 2 * pad, Wp = W + 2 * pad;
  try {
    h->rowptr.resize(size_t(M) + 1);
    int64_t nnz = 0;
    for (int m = 0; m < M; ++m) nnz += CRS - std::count(w + m * CRS, w + (m + 1) * CRS, 0.0f);
    if (nnz > kInt32Max) { delete h; return ESCOIN_ERR_OVERFLOW; }
    h->colidx.resize(size_t(nnz));
    h->value.resize(size_t(nnz));
    // Row m = filter m in (c, kh, kw) order; keep w != 0.0f
    // (R#6); colidx = f(c, kh, kw) over the padded input (R#4).
    int64_t j = 0;
    h->rowptr[0] = 0;
    for (int m = 0; m < M; ++m) {
      const float* wm = w + m * CRS;
      for (int c = 0; c < C; ++c)
        for (int kh = 0; kh < K; ++kh)
          for (int kw = 0; kw < K; ++kw) {
            const float v = wm[(int64_t(c) * K + kh) * K + kw];
            if (v != 0.0f) {
              h->colidx[j] = int32_t((c * Hp + kh) * Wp + kw);
              h->value[j] = v;
              ++j;
            }
          }
      h->rowptr[m + 1] = int32_t(j);
    }
    h->nnz = nnz;
  } catch (...) {
    delete h;
    return ESCOIN_ERR_ALLOC;
  }
  *out = h;
  return ESCOIN_OK;
}

int escoin_csr_stretch_device(const float* d_w, int M, int C, int H, int W, int K, int stride, int pad, int device,
                              void* cuda_stream, escoin_csr** out) {
  if (!d_w || !out) return ESCOIN_ERR_NULL;
  *out = nullptr;
  int E, F;
  int rc = validate_shape(M, C, H, W, K, stride, pad, &E, &F);
  if (rc != ESCOIN_OK) return rc;
  DeviceGuard g(device);
  if (!g.ok) return ESCOIN_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  escoin_csr* h = new (std::nothrow) escoin_csr();
  if (!h) return ESCOIN_ERR_ALLOC;
  h->M = M; h->C = C; h->H = H; h->W = W; h->K = K; h->stride = stride; h->pad = pad; h->E = E; h->F = F;
  h->device = device;
  const int64_t crs = int64_t(C) * K * K;
  int* cnt = nullptr;
  auto fail = [&](int code) {
    if (cnt) cudaFree(cnt);
    escoin_csr_free(h);
    return code;
  };
  if (cudaMalloc(&cnt, sizeof(int) * M) != cudaSuccess) return fail(ESCOIN_ERR_ALLOC);
  if (cudaMalloc(&h->d_rowptr, sizeof(int32_t) * (size_t(M) + 1)) != cudaSuccess) return fail(ESCOIN_ERR_ALLOC);
  if (launch_stretch_count(d_w, M, crs, cnt, s) != 0) return fail(ESCOIN_ERR_CUDA);
  if (launch_stretch_scan(cnt, M, h->d_rowptr, s) != 0) return fail(ESCOIN_ERR_CUDA);
  try {
    h->rowptr.resize(size_t(M) + 1);
  } catch (...) {
    return fail(ESCOIN_ERR_ALLOC);
  }
  if (cudaMemcpyAsync(h->rowptr.data(), h->d_rowptr, 4 * (size_t(M) + 1), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return fail(ESCOIN_ERR_CUDA);
  const int64_t nnz = h->rowptr[M];
  if (nnz > kInt32Max) return fail(ESCOIN_ERR_OVERFLOW);
  h->nnz = nnz;
  const size_t nb = std::max<size_t>(4 * size_t(nnz), 16);
  if (cudaMalloc(&h->d_colidx, nb) != cudaSuccess || cudaMalloc(&h->d_value, nb) != cudaSuccess)
    return fail(ESCOIN_ERR_ALLOC);
  if (launch_stretch_compact(d_w, M, crs, K, H + 2 * pad, W + 2 * pad, h->d_rowptr, h->d_colidx, h->d_value, s) != 0)
    return fail(ESCOIN_ERR_CUDA);
  try {
    h->colidx.resize(size_t(nnz));
    h->value.resize(size_t(nnz));
  } catch (...) {
    return fail(ESCOIN_ERR_ALLOC);
  }
  if (nnz > 0 && (cudaMemcpyAsync(h->colidx.data(), h->d_colidx, 4 * size_t(nnz), cudaMemcpyDeviceToHost, s) !=
                      cudaSuccess ||
                  cudaMemcpyAsync(h->value.data(), h->d_value, 4 * size_t(nnz), cudaMemcpyDeviceToHost, s) !=
                      cudaSuccess))
    return fail(ESCOIN_ERR_CUDA);
  if (cudaStreamSynchronize(s) != cudaSuccess) return fail(ESCOIN_ERR_CUDA);
  cudaFree(cnt);
  cnt = nullptr;
  if ((rc = escoin_csr_to_device(h, device, cuda_stream)) != ESCOIN_OK) return fail(rc);
  *out = h;
  return ESCOIN_OK;
}

int escoin_csr_info(const escoin_csr* h, int* M, int* C, int* H, int* W, int* K, int* stride, int* pad,
                    int64_t* nnz) {
  if (!h) return ESCOIN_ERR_NULL;
  if (M) *M = h->M;
  if (C) *C = h->C;
  if (H) *H = h->H;
  if (W) *W = h->W;
  if (K) *K = h->K;
  if (stride) *stride = h->stride;
  if (pad) *pad = h->pad;
  if (nnz) *nnz = h->nnz;
  return ESCOIN_OK;
}

int escoin_csr_host_arrays(const escoin_csr* h, const int32_t** rowptr, const int32_t** colidx,
                           const float** value) {
  if (!h) return ESCOIN_ERR_NULL;
  if (rowptr) *rowptr = h->rowptr.data();
  if (colidx) *colidx = h->colidx.data();
  if (value) *value = h->value.data();
  return ESCOIN_OK;
}

int escoin_csr_to_device(escoin_csr* h, int device, void* cuda_stream) {
  if (!h) return ESCOIN_ERR_NULL;
  if (h->on_device) return h->device == device ? ESCOIN_OK : ESCOIN_ERR_NOT_ON_DEVICE;
  DeviceGuard g(device);
  if (!g.ok) return ESCOIN_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  int rc;
  if (!h->borrowed && !h->d_rowptr) {  // (device-stretched handles already own their device CSR)
    if ((rc = upload(h->rowptr, &h->d_rowptr, s)) != ESCOIN_OK) return rc;
    if ((rc = upload(h->colidx, &h->d_colidx, s)) != ESCOIN_OK) return rc;
    if ((rc = upload(h->value, &h->d_value, s)) != ESCOIN_OK) return rc;
  }
  h->device = device;
  if ((rc = set_kernel(h, h->kernel < 0 ? ESCOIN_KERNEL_AUTO : h->kernel, s)) != ESCOIN_OK) return rc;
  if (cudaStreamSynchronize(s) != cudaSuccess) return ESCOIN_ERR_CUDA;
  h->on_device = true;
  return ESCOIN_OK;
}

int escoin_csr_wrap_device(const int32_t* d_rowptr, const int32_t* d_colidx, const float* d_value, int64_t nnz,
                           int M, int C, int H, int W, int K, int stride, int pad, int device, void* cuda_stream,
                           escoin_csr** out) {
  if (!d_rowptr || !out || (nnz > 0 && (!d_colidx || !d_value))) return ESCOIN_ERR_NULL;
  *out = nullptr;
  int E, F;
  int rc = validate_shape(M, C, H, W, K, stride, pad, &E, &F);
  if (rc != ESCOIN_OK) return rc;
  if (nnz < 0 || nnz > kInt32Max || nnz > int64_t(M) * C * K * K) return ESCOIN_ERR_CSR_MISMATCH;
  DeviceGuard g(device);
  if (!g.ok) return ESCOIN_ERR_CUDA;
  escoin_csr* h = new (std::nothrow) escoin_csr();
  if (!h) return ESCOIN_ERR_ALLOC;
  h->M = M; h->C = C; h->H = H; h->W = W; h->K = K; h->stride = stride; h->pad = pad; h->E = E; h->F = F;
  h->nnz = nnz;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  try {
    h->rowptr.resize(size_t(M) + 1);
    h->colidx.resize(size_t(nnz));
    h->value.resize(size_t(nnz));
  } catch (...) {
    delete h;
    return ESCOIN_ERR_ALLOC;
  }
  bool ok = cudaMemcpyAsync(h->rowptr.data(), d_rowptr, 4 * (size_t(M) + 1), cudaMemcpyDeviceToHost, s) == cudaSuccess;
  if (nnz > 0) {
    ok = ok && cudaMemcpyAsync(h->colidx.data(), d_colidx, 4 * size_t(nnz), cudaMemcpyDeviceToHost, s) == cudaSuccess;
    ok = ok && cudaMemcpyAsync(h->value.data(), d_value, 4 * size_t(nnz), cudaMemcpyDeviceToHost, s) == cudaSuccess;
  }
  ok = ok && cudaStreamSynchronize(s) == cudaSuccess;
  if (!ok) { delete h; return ESCOIN_ERR_CUDA; }
  // validate the borrowed CSR
  const int64_t lim = int64_t(C) * (H + 2 * pad) * (W + 2 * pad);
  bool good = h->rowptr[0] == 0 && h->rowptr[M] == nnz;
  for (int m = 0; good && m < M; ++m) good = h->rowptr[m] <= h->rowptr[m + 1];
  for (int64_t j = 0; good && j < nnz; ++j) good = h->colidx[j] >= 0 && h->colidx[j] < lim;
  if (!good) { delete h; return ESCOIN_ERR_CSR_MISMATCH; }
  h->borrowed = true;
  h->d_rowptr = const_cast<int32_t*>(d_rowptr);
  h->d_colidx = const_cast<int32_t*>(d_colidx);
  h->d_value = const_cast<float*>(d_value);
  rc = escoin_csr_to_device(h, device, cuda_stream);
  if (rc != ESCOIN_OK) { escoin_csr_free(h); return rc; }
  *out = h;
  return ESCOIN_OK;
}

void escoin_csr_free(escoin_csr* h) {
  if (!h) return;
  if (h->device >= 0) {
    DeviceGuard g(h->device);
    cudaDeviceSynchronize();
    free_ds6(h);
    if (h->d_dense) cudaFree(h->d_dense);
    for (JitModule* jm : h->jits) {
      jit_free(*jm);
      delete jm;
    }
    if (!h->borrowed) {
      if (h->d_rowptr) cudaFree(h->d_rowptr);
      if (h->d_colidx) cudaFree(h->d_colidx);
      if (h->d_value) cudaFree(h->d_value);
    }
  }
  delete h;
}

int escoin_sconv_forward(int N, int C, int H, int W, int M, int K, int stride, int pad, const escoin_csr* h,
                         const float* in, float* out, const float* bias, int relu, void* cuda_stream) {
  if (!h) return ESCOIN_ERR_NULL;
  if (N < 0) return ESCOIN_ERR_SHAPE;
  if (C != h->C || H != h->H || W != h->W || M != h->M || K != h->K || stride != h->stride || pad != h->pad)
    return ESCOIN_ERR_CSR_MISMATCH;
  if (N == 0) return ESCOIN_OK;
  if (!in || !out) return ESCOIN_ERR_NULL;
  if (!h->on_device) return ESCOIN_ERR_NOT_ON_DEVICE;
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != h->device) return ESCOIN_ERR_NOT_ON_DEVICE;
  if (int64_t(N) * C * H * W > (int64_t(1) << 40)) return ESCOIN_ERR_OVERFLOW;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  int rc;
  if (h->kernel == ESCOIN_KERNEL_JIT) {
    if (int64_t(N) * C * H * W > kInt32Max) return ESCOIN_ERR_OVERFLOW;
    JitModule& jm = *h->jit;
    if (jm.plan.ks > 1) {
      // split channels: partial sums into the handle's workspace (grown here, outside any capture, when a
      // larger batch arrives), then the fixed-order reduce + bias + ReLU
      const int64_t total = int64_t(N) * M * h->E * h->F, need = total * jm.plan.ks;
      if (need > jm.ws_elems) {
        if (jm.d_ws) cudaFree(jm.d_ws);
        jm.d_ws = nullptr;
        jm.ws_elems = 0;
        if (cudaMalloc(&jm.d_ws, size_t(need) * 4) != cudaSuccess) {
          jm.d_ws = nullptr;
          return ESCOIN_ERR_ALLOC;
        }
        jm.ws_elems = need;
      }
      rc = jit_launch(jm, in, out, bias, relu, N, s, jm.d_ws);
      if (rc == 0) rc = launch_ks_reduce(jm.d_ws, jm.plan.ks, total, M, h->E * h->F, bias, relu, out, s);
    } else {
      rc = jit_launch(jm, in, out, bias, relu, N, s);
    }
    if (rc == -2) return ESCOIN_ERR_OVERFLOW;
  } else if (h->kernel == ESCOIN_KERNEL_DENSE_TC) {
    rc = launch_dense_tc(in, h->d_dense, bias, out, N, C, H, W, M, K, stride, pad, relu ? 1 : 0, 3, s);
  } else if (h->kernel == 0) {
    rc = launch_paper(h->d_rowptr, h->d_colidx, h->d_value, in, out, bias, relu ? 1 : 0, N, C, H, W, M, K, stride,
                      pad, h->E, h->F, s);
  } else {
    int nv = 0;
    const TiledVariant* tv = tiled_variants(&nv);
    TiledArgs a = h->targs;
    a.in = in;
    a.out = out;
    a.bias = bias;
    a.relu = relu ? 1 : 0;
    a.N = N;
    if (a.mos) {  // the super-image grows with N
      a.PR = ceil_div(mosaic_rows(h, a.mos, N), tv[h->kernel - 1].PH);
      a.tiles_r = ceil_div(a.PR, a.TR);
    }
    if (tv[h->kernel - 1].mode == 4 || tv[h->kernel - 1].mode == 5)
      a.ntiles = int((int64_t(N) * H * W + a.TP - 1) / a.TP);
    else
      a.ntiles = a.mos ? a.tiles_r : a.flat ? ceil_div(N * a.PR, a.WP * 32) : ceil_div(N, a.NB * a.IP) * a.tiles_r;
    a.debug = g_debug_kernel;
    if (a.ntiles > 65535) return ESCOIN_ERR_OVERFLOW;
    rc = tv[h->kernel - 1].launch(a, s);
  }
  return rc == 0 ? ESCOIN_OK : ESCOIN_ERR_CUDA;
}

int escoin_sconv_forward_hostio(int N, int C, int H, int W, int M, int K, int stride, int pad, const escoin_csr* h,
                                const float* h_in, float* h_out, float* d_in, float* d_out, const float* bias,
                                int relu, void* cuda_stream) {
  if (!h) return ESCOIN_ERR_NULL;
  if (N > 0 && (!h_in || !h_out || !d_in || !d_out)) return ESCOIN_ERR_NULL;
  if (C != h->C || H != h->H || W != h->W || M != h->M || K != h->K || stride != h->stride || pad != h->pad)
    return ESCOIN_ERR_CSR_MISMATCH;
  if (N == 0) return ESCOIN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  const size_t in_b = size_t(N) * C * H * W * 4, out_b = size_t(N) * M * h->E * h->F * 4;
  if (cudaMemcpyAsync(d_in, h_in, in_b, cudaMemcpyHostToDevice, s) != cudaSuccess) return ESCOIN_ERR_CUDA;
  const int rc = escoin_sconv_forward(N, C, H, W, M, K, stride, pad, h, d_in, d_out, bias, relu, cuda_stream);
  if (rc != ESCOIN_OK) return rc;
  if (cudaMemcpyAsync(h_out, d_out, out_b, cudaMemcpyDeviceToHost, s) != cudaSuccess) return ESCOIN_ERR_CUDA;
  return ESCOIN_OK;
}

int escoin_kernel_count(void) {
  int nv = 0;
  tiled_variants(&nv);
  return nv + 1;
}

int escoin_kernel_info(int id, const char** name, int* K, int* stride) {
  int nv = 0;
  const TiledVariant* tv = tiled_variants(&nv);
  if (id < 0 || id > nv) return ESCOIN_ERR_UNSUPPORTED;
  if (id == 0) {
    if (name) *name = "paper_mapping";
    if (K) *K = 0;
    if (stride) *stride = 0;
  } else {
    if (name) *name = tv[id - 1].name;
    if (K) *K = tv[id - 1].K;
    if (stride) *stride = tv[id - 1].S;
  }
  return ESCOIN_OK;
}

int escoin_csr_set_kernel(escoin_csr* h, int id) {
  if (!h) return ESCOIN_ERR_NULL;
  if (!h->on_device) {
    int nv = 0;
    tiled_variants(&nv);
    if (id != ESCOIN_KERNEL_AUTO && id != ESCOIN_KERNEL_JIT && id != ESCOIN_KERNEL_DENSE_TC && (id < 0 || id > nv))
      return ESCOIN_ERR_UNSUPPORTED;
    h->kernel = id;  // resolved at escoin_csr_to_device
    return ESCOIN_OK;
  }
  DeviceGuard g(h->device);
  if (!g.ok) return ESCOIN_ERR_CUDA;
  cudaDeviceSynchronize();  // no forward may be reading the old derived format
  return set_kernel(h, id, nullptr);
}

int escoin_csr_autotune(escoin_csr* h, int N, const float* in, float* out, const float* bias, int relu, int reps,
                        void* cuda_stream, int* best_id, float* best_ms) {
  return escoin_csr_autotune_ex(h, N, in, out, bias, relu, reps, cuda_stream, nullptr, 0,
                                ESCOIN_TUNE_VARIANTS | ESCOIN_TUNE_JIT, best_id, best_ms);
}

int escoin_csr_autotune_ex(escoin_csr* h, int N, const float* in, float* out, const float* bias, int relu, int reps,
                           void* cuda_stream, void* flush_buf, int64_t flush_bytes, int flags, int* best_id,
                           float* best_ms) {
  if (!h) return ESCOIN_ERR_NULL;
  if (!h->on_device) return ESCOIN_ERR_NOT_ON_DEVICE;
  if (flush_bytes < 0 || (flush_bytes > 0 && !flush_buf)) return ESCOIN_ERR_NULL;
  if (!(flags & (ESCOIN_TUNE_VARIANTS | ESCOIN_TUNE_JIT))) return ESCOIN_ERR_UNSUPPORTED;
  if (reps < 1) reps = 1;
  DeviceGuard g(h->device);
  if (!g.ok) return ESCOIN_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return ESCOIN_ERR_CUDA;
  int rc = ESCOIN_OK;
  // one warm-up forward, then `reps` forwards each timed alone (events on s) after an optional L2
  // flush (a memset of flush_buf, outside the events) — the conditions bench.py measures under;
  // the candidate's time is the median
  auto time_it = [&](float* ms_out) -> int {
    int r = escoin_sconv_forward(N, h->C, h->H, h->W, h->M, h->K, h->stride, h->pad, h, in, out, bias, relu, s);
    if (r != ESCOIN_OK) return r;
    std::vector<float> t;
    for (int k = 0; k < reps; ++k) {
      if (flush_bytes > 0 && cudaMemsetAsync(flush_buf, k & 0xff, size_t(flush_bytes), s) != cudaSuccess)
        return ESCOIN_ERR_CUDA;
      cudaEventRecord(e0, s);
      r = escoin_sconv_forward(N, h->C, h->H, h->W, h->M, h->K, h->stride, h->pad, h, in, out, bias, relu, s);
      if (r != ESCOIN_OK) return r;
      cudaEventRecord(e1, s);
      if (cudaEventSynchronize(e1) != cudaSuccess) return ESCOIN_ERR_CUDA;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    *ms_out = t[t.size() / 2];
    return ESCOIN_OK;
  };
  int nv = 0;
  const TiledVariant* tv = tiled_variants(&nv);
  int best = -1, best_rank = 0;
  float best_t = 0.f;
  constexpr int kRanks = 4;  // tiling candidates (distinct geometries) measured per variant
  for (int idr = 0; (flags & ESCOIN_TUNE_VARIANTS) && idr <= nv * kRanks && rc == ESCOIN_OK; ++idr) {
    const int id = idr / kRanks, rank = idr % kRanks;
    if (id == 0 && rank > 0) continue;
    if (id > 0 && (tv[id - 1].K != h->K || tv[id - 1].S != h->stride)) continue;
    if (cudaStreamSynchronize(s) != cudaSuccess) { rc = ESCOIN_ERR_CUDA; break; }
    if (set_kernel(h, id, s, rank) != ESCOIN_OK) continue;  // no (further) tiling fits: skip
    float ms = 0.f;
    if ((rc = time_it(&ms)) != ESCOIN_OK) break;
    if (best < 0 || ms < best_t) { best = id; best_rank = rank; best_t = ms; }
  }
  JitModule* best_jit = h->jit;
  const int prev_kernel = h->kernel;
  for (size_t ji = 0; (flags & ESCOIN_TUNE_JIT) && ji < h->jits.size() && rc == ESCOIN_OK; ++ji) {
    h->jit = h->jits[ji];  // every compiled specialised kernel
    h->kernel = ESCOIN_KERNEL_JIT;
    float ms = 0.f;
    if ((rc = time_it(&ms)) != ESCOIN_OK) break;
    if (best < 0 || ms < best_t) { best = ESCOIN_KERNEL_JIT; best_t = ms; best_jit = h->jit; }
  }
  h->jit = best_jit;
  h->kernel = prev_kernel;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc != ESCOIN_OK) return rc;
  if (best < 0) return ESCOIN_ERR_UNSUPPORTED;
  if ((rc = set_kernel(h, best, s, best_rank)) != ESCOIN_OK) return rc;
  if (cudaStreamSynchronize(s) != cudaSuccess) return ESCOIN_ERR_CUDA;
  if (best_id) *best_id = best;
  if (best_ms) *best_ms = best_t;
  return ESCOIN_OK;
}

int escoin_csr_kernel_label(const escoin_csr* h, char* buf, int cap) {
  if (!h || !buf || cap < 1) return ESCOIN_ERR_NULL;
  std::string l;
  if (h->kernel == ESCOIN_KERNEL_JIT && h->jit) {
    l = jit_label(*h->jit);
  } else if (h->kernel == ESCOIN_KERNEL_DENSE_TC) {
    l = "dense_tcgen05_3xtf32";
  } else if (h->kernel == 0) {
    l = "paper_mapping";
  } else if (h->kernel > 0) {
    int nv = 0;
    const TiledVariant* tv = tiled_variants(&nv);
    char b[160];
    const TiledArgs& a = h->targs;
    snprintf(b, sizeof b, "%s_wm%d_wp%d_nb%d_tr%d_cc%d_ns%d_mos%d_scs%d", h->kernel <= nv ? tv[h->kernel - 1].name : "?",
             a.WM, a.WP, a.NB, a.TR, a.CC, a.NS, a.mos, a.SCs);
    l = b;
  } else {
    l = "auto";
  }
  std::snprintf(buf, size_t(cap), "%s", l.c_str());
  return int(l.size()) < cap ? ESCOIN_OK : ESCOIN_ERR_OVERFLOW;
}

double escoin_sparse_threshold(void) {
  if (const char* e = std::getenv("ESCOIN_SPARSE_THRESHOLD")) {
    char* end = nullptr;
    const double v = std::strtod(e, &end);
    if (end != e && v >= 0.0 && v <= 1.0) return v;
  }
  return ESCOIN_DEFAULT_SPARSE_THRESHOLD;
}

int escoin_select_engine(int M, int C, int K, int64_t nnz, double threshold) {
  if (M < 1 || C < 1 || K < 1 || nnz < 0) return ESCOIN_ERR_SHAPE;
  if (!(threshold >= 0.0 && threshold <= 1.0)) threshold = escoin_sparse_threshold();
  const double total = double(M) * C * K * K;
  const double sparsity = 1.0 - double(nnz) / total;
  return sparsity >= threshold ? ESCOIN_ENGINE_SPARSE : ESCOIN_ENGINE_DENSE_TC;
}

int escoin_csr_select_engine(escoin_csr* h, double threshold, int* engine) {
  if (!h) return ESCOIN_ERR_NULL;
  const int e = escoin_select_engine(h->M, h->C, h->K, h->nnz, threshold);
  if (e < 0) return e;
  if (engine) *engine = e;
  if (e == ESCOIN_ENGINE_SPARSE) {
    if (h->kernel == ESCOIN_KERNEL_DENSE_TC) return escoin_csr_set_kernel(h, ESCOIN_KERNEL_AUTO);
    return ESCOIN_OK;
  }
  return escoin_csr_set_kernel(h, ESCOIN_KERNEL_DENSE_TC);
}

int escoin_csr_jit_stats(const escoin_csr* h, int* units, int* cache_hits, double* compile_s, int64_t* ptx_bytes) {
  if (!h) return ESCOIN_ERR_NULL;
  if (!h->jit) return ESCOIN_ERR_UNSUPPORTED;
  if (units) *units = int(h->jit->units.size());
  if (cache_hits) *cache_hits = h->jit->cache_hits;
  if (compile_s) *compile_s = h->jit->compile_s;
  if (ptx_bytes) *ptx_bytes = int64_t(h->jit->ptx_bytes);
  return ESCOIN_OK;
}

int escoin_csr_jit(escoin_csr* h, int n_hint, const int* tunables, int ntunables) {
  if (!h) return ESCOIN_ERR_NULL;
  if (!h->on_device) return ESCOIN_ERR_NOT_ON_DEVICE;
  if (ntunables < 0 || ntunables > 18 || (ntunables > 0 && !tunables)) return ESCOIN_ERR_NULL;
  int tun[18] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < ntunables; ++i) tun[i] = tunables[i];
  DeviceGuard g(h->device);
  if (!g.ok) return ESCOIN_ERR_CUDA;
  return build_jit(h, n_hint > 0 ? n_hint : 128, tun);  // adds a module (selected under jit_mu), frees none
}

int escoin_csr_jit_info(const escoin_csr* h, int* tunables6, int* mos, int* regs, int64_t* code_bytes) {
  if (!h) return ESCOIN_ERR_NULL;
  if (!h->jit) return ESCOIN_ERR_UNSUPPORTED;
  const JitPlan& p = h->jit->plan;
  if (tunables6) {
    tunables6[0] = p.Q; tunables6[1] = p.P; tunables6[2] = p.CC;
    tunables6[3] = p.NS; tunables6[4] = p.warps; tunables6[5] = p.minb;
  }
  if (mos) *mos = int(h->jit->units.size());
  if (regs) *regs = h->jit->regs;
  if (code_bytes) *code_bytes = int64_t(h->jit->cubin_bytes);
  return ESCOIN_OK;
}

int escoin_csr_get_kernel(const escoin_csr* h, int* id) {
  if (!h || !id) return ESCOIN_ERR_NULL;
  *id = h->kernel;
  return ESCOIN_OK;
}

const char* escoin_status_string(int status) {
  switch (status) {
    case ESCOIN_OK: return "ok";
    case ESCOIN_ERR_NULL: return "null pointer argument";
    case ESCOIN_ERR_SHAPE: return "invalid shape";
    case ESCOIN_ERR_CSR_MISMATCH: return "shape or CSR does not match the handle";
    case ESCOIN_ERR_NOT_ON_DEVICE: return "handle not on the current device";
    case ESCOIN_ERR_OVERFLOW: return "index overflow (int32)";
    case ESCOIN_ERR_UNSUPPORTED: return "unsupported kernel variant / shape";
    case ESCOIN_ERR_ALLOC: return "allocation failed";
    case ESCOIN_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

int escoin_bench_dense_tc_forward(int N, int C, int H, int W, int M, int K, int stride, int pad, const float* w,
                                  const float* in, float* out, const float* bias, int relu, int nsplit,
                                  void* cuda_stream) {
  if (!w || !in || !out) return ESCOIN_ERR_NULL;
  if (N < 1 || C < 1 || H < 1 || W < 1 || M < 1 || K < 1 || stride < 1 || pad < 0) return ESCOIN_ERR_SHAPE;
  if (H + 2 * pad < K || W + 2 * pad < K) return ESCOIN_ERR_SHAPE;
  if (nsplit != 1 && nsplit != 3) return ESCOIN_ERR_UNSUPPORTED;
  const int rc = launch_dense_tc(in, w, bias, out, N, C, H, W, M, K, stride, pad, relu ? 1 : 0, nsplit,
                                 static_cast<cudaStream_t>(cuda_stream));
  return rc == 0 ? ESCOIN_OK : ESCOIN_ERR_CUDA;
}

const char* escoin_version(void) { return "escoin-b200 0.1 sm_100a"; }

/* Internal (not in escoin.h): host-only plan of tiled variant `id` for tests.
 * out[14] = {WM, WP, NB, TR, PR, PC, SR, SCs, plane, CC, smem_bytes, records, PCs, stages}. */
int escoin_internal_plan(const escoin_csr* h, int id, int64_t* out) {
  int nv = 0;
  const TiledVariant* tv = tiled_variants(&nv);
  if (!h || !out) return ESCOIN_ERR_NULL;
  if (id < 1 || id > nv) return ESCOIN_ERR_UNSUPPORTED;
  Tiling t{};
  DS6 ds;
  int CC = 0;
  size_t smem = 0, sf = 0, sr = 0;
  int ns = 2;
  const int rc = plan_tiled(h, tv[id - 1], 0, &t, &CC, &ds, &smem, &sf, &sr, &ns);
  if (rc != ESCOIN_OK) return rc;
  const int64_t v[14] = {t.WM, t.WP, t.NB, t.TR, t.PR, t.PC, t.SR, t.SCs, t.plane, CC, int64_t(smem),
                         int64_t(ds.recs.size()), t.PCs, ns};
  for (int i = 0; i < 14; ++i) out[i] = v[i];
  return ESCOIN_OK;
}

/* Internal (not in escoin.h): the PTX escoin_csr_jit would generate for this handle with these
 * tunables (host only, no device needed), and an in-process compile of PTX text for sm_100a.
 * Two-call pattern: *len receives the size; the text is copied when cap >= size + 1. */
int escoin_internal_jit_ptx(const escoin_csr* h, int n_hint, const int* tunables, int ntunables, char* buf,
                            int64_t cap, int64_t* len) {
  if (!h || !len || ntunables < 0 || ntunables > 18 || (ntunables > 0 && !tunables)) return ESCOIN_ERR_NULL;
  JitPlan p;
  int tun[18] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < ntunables; ++i) tun[i] = tunables[i];
  p.Q = tun[0]; p.P = tun[1]; p.CC = tun[2]; p.NS = tun[3]; p.warps = tun[4]; p.minb = tun[5]; p.pf = tun[6];
  p.mb = tun[7]; p.units = tun[8]; p.vec = tun[9]; p.reorder = tun[10]; p.sws = tun[11]; p.perm = tun[12]; p.split = tun[13]; p.pair = tun[14]; p.hp = tun[15]; p.pw = tun[16]; p.ks = tun[17];
  const double density = double(h->nnz) / (double(h->M) * h->C * h->K * h->K);
  if (jit_plan(p, h->C, h->H, h->W, h->M, h->K, h->stride, h->pad, n_hint > 0 ? n_hint : 128, density) != 0)
    return ESCOIN_ERR_UNSUPPORTED;
  const std::string ptx = jit_ptx_text(p, h->rowptr.data(), h->colidx.data(), h->value.data());
  *len = int64_t(ptx.size());
  if (buf && cap >= int64_t(ptx.size()) + 1) std::memcpy(buf, ptx.c_str(), ptx.size() + 1);
  return ESCOIN_OK;
}

/* Internal: the unit split escoin_csr_jit would use (ranges[2*u], ranges[2*u+1] = m-group range of unit u;
 * *count = units) and the PTX of m-groups [g_lo, g_hi) (two-call pattern as above). */
int escoin_internal_jit_units(const escoin_csr* h, int n_hint, const int* tunables, int ntunables, int* ranges,
                              int cap, int* count, char* buf, int64_t bufcap, int64_t* len, int g_lo, int g_hi) {
  if (!h || !count || ntunables < 0 || ntunables > 18 || (ntunables > 0 && !tunables)) return ESCOIN_ERR_NULL;
  JitPlan p;
  int tun[18] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < ntunables; ++i) tun[i] = tunables[i];
  p.Q = tun[0]; p.P = tun[1]; p.CC = tun[2]; p.NS = tun[3]; p.warps = tun[4]; p.minb = tun[5]; p.pf = tun[6];
  p.mb = tun[7]; p.units = tun[8]; p.vec = tun[9]; p.reorder = tun[10]; p.sws = tun[11]; p.perm = tun[12]; p.split = tun[13]; p.pair = tun[14]; p.hp = tun[15]; p.pw = tun[16]; p.ks = tun[17];
  const double density = double(h->nnz) / (double(h->M) * h->C * h->K * h->K);
  if (jit_plan(p, h->C, h->H, h->W, h->M, h->K, h->stride, h->pad, n_hint > 0 ? n_hint : 128, density) != 0)
    return ESCOIN_ERR_UNSUPPORTED;
  const auto r = jit_units(p, h->rowptr.data());
  *count = int(r.size());
  for (int u = 0; u < int(r.size()) && 2 * u + 1 < cap && ranges; ++u) {
    ranges[2 * u] = r[u].first;
    ranges[2 * u + 1] = r[u].second;
  }
  if (len && g_hi > g_lo) {
    if (g_lo < 0 || g_hi > p.nmg) return ESCOIN_ERR_SHAPE;
    const std::string ptx = jit_ptx_text(p, h->rowptr.data(), h->colidx.data(), h->value.data(), g_lo, g_hi);
    *len = int64_t(ptx.size());
    if (buf && bufcap >= int64_t(ptx.size()) + 1) std::memcpy(buf, ptx.c_str(), ptx.size() + 1);
  }
  return ESCOIN_OK;
}

/* Internal: host-only build of the cubin escoin_csr_jit would load (generate, compile the units,
 * link) — *units, *cubin_bytes; the compiler/linker log on failure into buf (cap bytes). */
int escoin_internal_jit_cubin(const escoin_csr* h, int n_hint, const int* tunables, int ntunables, int* units,
                              int64_t* cubin_bytes, char* buf, int64_t cap) {
  if (!h || !units || !cubin_bytes || ntunables < 0 || ntunables > 18 || (ntunables > 0 && !tunables))
    return ESCOIN_ERR_NULL;
  JitPlan p;
  int tun[18] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < ntunables; ++i) tun[i] = tunables[i];
  p.Q = tun[0]; p.P = tun[1]; p.CC = tun[2]; p.NS = tun[3]; p.warps = tun[4]; p.minb = tun[5]; p.pf = tun[6];
  p.mb = tun[7]; p.units = tun[8]; p.vec = tun[9]; p.reorder = tun[10]; p.sws = tun[11]; p.perm = tun[12]; p.split = tun[13]; p.pair = tun[14]; p.hp = tun[15]; p.pw = tun[16]; p.ks = tun[17];
  const double density = double(h->nnz) / (double(h->M) * h->C * h->K * h->K);
  if (jit_plan(p, h->C, h->H, h->W, h->M, h->K, h->stride, h->pad, n_hint > 0 ? n_hint : 128, density) != 0)
    return ESCOIN_ERR_UNSUPPORTED;
  JitModule jm;
  std::vector<char> cubin;
  std::string log;
  const int rc = jit_cubin(jm, p, h->rowptr.data(), h->colidx.data(), h->value.data(), &cubin, &log);
  if (rc != 0) {
    if (buf && cap > 0) std::snprintf(buf, size_t(cap), "%s", log.c_str());
    return ESCOIN_ERR_UNSUPPORTED;
  }
  *units = int(jm.units.size());
  *cubin_bytes = int64_t(cubin.size());
  return ESCOIN_OK;
}

/* Internal: label of the plan escoin_csr_jit would compile (host only, nothing compiled). */
int escoin_internal_jit_label(const escoin_csr* h, int n_hint, const int* tunables, int ntunables, char* buf,
                              int cap) {
  if (!h || !buf || cap < 1 || ntunables < 0 || ntunables > 18 || (ntunables > 0 && !tunables)) return ESCOIN_ERR_NULL;
  JitPlan p;
  int tun[18] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < ntunables; ++i) tun[i] = tunables[i];
  p.Q = tun[0]; p.P = tun[1]; p.CC = tun[2]; p.NS = tun[3]; p.warps = tun[4]; p.minb = tun[5]; p.pf = tun[6];
  p.mb = tun[7]; p.units = tun[8]; p.vec = tun[9]; p.reorder = tun[10]; p.sws = tun[11]; p.perm = tun[12]; p.split = tun[13]; p.pair = tun[14]; p.hp = tun[15]; p.pw = tun[16]; p.ks = tun[17];
  const double density = double(h->nnz) / (double(h->M) * h->C * h->K * h->K);
  if (jit_plan(p, h->C, h->H, h->W, h->M, h->K, h->stride, h->pad, n_hint > 0 ? n_hint : 128, density) != 0)
    return ESCOIN_ERR_UNSUPPORTED;
  JitModule jm;
  jm.plan = p;
  jm.units.resize(jit_units(p, h->rowptr.data()).size());
  std::snprintf(buf, size_t(cap), "%s", jit_label(jm).c_str());
  return ESCOIN_OK;
}

int escoin_internal_ptx_compile(const char* ptx, int64_t* cubin_bytes) {
  if (!ptx || !cubin_bytes) return ESCOIN_ERR_NULL;
  size_t n = 0;
  if (jit_compile_only(ptx, &n) != 0) return ESCOIN_ERR_UNSUPPORTED;
  *cubin_bytes = int64_t(n);
  return ESCOIN_OK;
}

}  // extern "C"
