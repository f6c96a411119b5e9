// escoin_internal.h — shared between the host library and the kernels.
// Not part of the public ABI (include/escoin.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace escoin {

constexpr int kTiledThreads = 256;   // 8 warps = WM x WP
constexpr int kMaxStages = 4;       // smem pipeline depth limit (mbarrier pairs per CTA)
constexpr int kMaxStagePos = 8;      // staged plane positions per thread (SR*SCs <= 2048)
constexpr int kHdrBase = 1 << 20;    // bucket header record: code = kHdrBase + c_local
constexpr int kDone = -1;            // end of a warp's record stream for one chunk

// Launch parameters of the register-tiled kernel (see sconv_tiled.cuh).
struct TiledArgs {
  const float* in;
  float* out;
  const float* bias;
  int relu;
  int N, C, H, W, M, E, F, pad;
  int PR, PC;           // patch grid of one image: ceil(E/PH) x ceil(F/PW)
  int PCs;              // slot columns per patch row (>= PC; lanes with pc >= PC idle)
  int WM, WP, NB, TR;   // warps along m / along pixels; image groups and patch rows per CTA
  int IP;               // images per lane (image group size): 2 for mode-3 variants, else 1
  int flat;             // 1: full-row patches (PC == 1) over a flat (image, patch-row) index, so one
                        // warp's 32 rows may span images (no idle lanes for PR not dividing 32)
  int mos;              // > 0: mosaic tiling — the batch is one super-image with `mos` images per
                        // super-row, periods H+pad / W+pad (shared zero separators); NB = 1
  int SR, SCs, plane;   // staged slab rows, row stride (words), plane stride (words)
  int TP, vec16;        // mode 4 (1x1): pixels per CTA tile (flat over the batch); HW % 4 == 0
  int CC;               // input channels per chunk
  int tiles_r;          // ceil(PR / TR)
  int B, ntiles;        // grid: m-blocks x pixel tiles
  int NS;               // shared-memory stages (2..kMaxStages), mbarrier-pipelined
  int stage_floats;     // floats per slab stage (multiple of 4)
  int stage_recs;       // records per record stage (even)
  int smem_bytes;
  const int2* recs;     // derived format (DS-6) records
  const int* sched;     // per active chunk: [k, rec_start, rec_count, woff[WM]]
  const int* sched_off; // [B+1] first entry of each m-block
  int sched_stride;     // 3 + WM
  int debug;            // timing experiments only (ESCOIN_DEBUG_KERNEL): 1 skip input staging, 4 skip stores
};

typedef int (*TiledLaunchFn)(const TiledArgs&, cudaStream_t);

struct TiledVariant {
  const char* name;
  int K, S, PH, PW, Q;
  int min_blocks;  // CTAs per SM the kernel is compiled for (__launch_bounds__)
  int mode;        // 0: per-record brx dispatch; 1: dense-bucket mask sweep; 2/3: FFMA2; 4: 1x1 row blocks
  int full_row;    // patch spans the whole output row (PC must be 1): vector window loads, flat tiling
  int rel_d;       // > 0: 16-byte records with predecessor-relative dispatch indices (chunk_loop_rel)
  int link;        // 1: linked records {idx(next), payload(self)} behind a header (chunk_loop_link)
  TiledLaunchFn launch;
};

// Paper-mapping kernel (variant 0), sconv_paper.cu.
int launch_paper(const int* rowptr, const int* colidx, const float* value, const float* in, float* out,
                 const float* bias, int relu, int N, int C, int H, int W, int M, int K, int S, int pad, int E,
                 int F, cudaStream_t s);

const TiledVariant* tiled_variants(int* count);

// Dense tcgen05 implicit-GEMM comparison point (dense_tc.cu); nsplit 1 = TF32, 3 = 3xTF32.
int launch_dense_tc(const float* in, const float* w, const float* bias, float* out, int N, int C, int H, int W,
                    int M, int K, int S, int pad, int relu, int nsplit, cudaStream_t s);

// Device weight stretching (stretch_device.cu).
int launch_stretch_count(const float* w, int M, int64_t crs, int* cnt, cudaStream_t s);
int launch_stretch_scan(const int* cnt, int M, int32_t* rowptr, cudaStream_t s);
// split-channel partial sums [ks][total] -> out (z order, + bias[(i / EF) % M], ReLU)
int launch_ks_reduce(const float* ws, int ks, int64_t total, int M, int EF, const float* bias, int relu, float* out,
                     cudaStream_t s);
int launch_densify(const int32_t* rowptr, const int32_t* colidx, const float* value, int M, int C, int K, int Hp,
                   int Wp, float* w, cudaStream_t s);
int launch_stretch_compact(const float* w, int M, int64_t crs, int K, int Hp, int Wp, const int32_t* rowptr,
                           int32_t* colidx, float* value, cudaStream_t s);

}  // namespace escoin
