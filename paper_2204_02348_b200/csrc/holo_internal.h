// Internal plan / kernel parameter structures shared by the CUDA kernels and
// the C-ABI implementation.  Not part of the public boundary.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "holo_fft.cuh"

namespace holo {

constexpr int kMaxPol = 2;
constexpr int kMaxWl = 16;
constexpr int kThreads = 256;

// Device-resident constant tables of one plan (all pointers into one cudaMalloc).
struct DevTables {
  const float2* tw_nx;    // [nx]   W_nx^i
  const float2* tw_ny;    // [ny]
  const float2* tw_gw;    // [gw]
  const float2* tw_gh;    // [gh]
  const float2* win_tab;  // [P][L][wh*ww] mask * recentring phase (/ sinc envelope)
  const float2* rem_x;    // [P][L][gw] removal phase along x  (incl. ifftshift sign)
  const float2* rem_y;    // [P][L][gh] removal phase along y  (incl. constant, sign, 1/(nx ny))
  const float* hx;        // [P][G][gw] dequantised basis profiles (float32)
  const float* hy;        // [P][G][gh]
  const float* xa;        // [gw] field axis (float32)
  const float* ya;        // [gh]
  const double* xad;      // [gw] the same axes widened to fp64 (analysis.py:78-79)
  const double* yad;      // [gh]
  const int16_t* mode_m;  // [M]
  const int16_t* mode_n;  // [M]
};

// Tables of the specialised 128-window kernels (holo_fast.cu, holo_fast_tc.cu).
struct FastTables {
  const float2* px;        // [P][L][WW] recentring phase along x
  const float2* py;        // [P][L][WH] recentring phase along y
  const int16_t* crange;   // [WW][2] first/last row inside the circular mask, per column
  const uint32_t* a_tc;    // [P][2][128][64] f16x2: row-DFT matrix (hi, lo) for wavelength 0
  const uint32_t* a_tcp;   // the same matrix with the rows packed: Re of column c at row 2c, Im at row 2c + 1 (holo_tc2.cu)
  const uint32_t* a2_tc;   // [P][2][128][64] f16x2: column-DFT matrix [Cr; Ci] (hi, lo) for wavelength 0
  const uint4* c2_tc;      // [P][hi | lo][24 KB]: the same [Cr; Ci] as a K-major shared-memory B operand
  const uint4* tco_img;    // [P][hx hi, hx lo, hy hi, hy lo][GP16 x 48 halves]: exact fp16 split of the int16 basis
  const float* tco_inv;    // [P][2][GP16] 1 / per-order basis scale (x, y)
  int tco_gp;              // GP16 (0: tensor-core overlap unavailable)
  const float* half_tab;   // [P][x | y][22][16]: transposed half profiles (axis index 0, then n/2..n-1) of the
                           // register-resident tail (holo_tailr.cu); null unless G <= 16 on 42-point axes
  int hsym;                // bit 2q: pol q's x profiles satisfy h_m(c - d) = (-1)^m h_m(c + d) exactly on the
                           // quantised basis (c = gw / 2, the axis origin); bit 2q + 1: the y profiles
};

struct Geometry {
  int W, H, P;
  int nx, ny, wh, ww, gh, gw;
  int mode;               // resolution mode
  int L, G, M;
  int col0[kMaxPol], row0[kMaxPol];
  int k0[kMaxPol][kMaxWl][2];
  float dxdy[kMaxPol];    // float32(complex64(dx*dy)) per pol
  double dx, dy;          // field-axis pitch (fp64 from the float32 axes)
  int radix_nx[8], nst_nx, radix_ny[8], nst_ny, radix_gw[8], nst_gw, radix_gh[8], nst_gh;
};

// Placement of the per-CTA working buffers: offset in shared memory (bytes) or,
// when the region does not fit, offset inside the CTA's global workspace slab.
struct Region {
  int64_t off;
  int in_smem;
};

struct Layout {
  Region R, S0, S1, Wt, Gd, Acc;
  int CH;                 // row pairs per row-pass chunk
  int CC;                 // columns per column-pass chunk
  int smem_bytes;         // dynamic shared memory per CTA
  int64_t slab_bytes;     // global workspace per CTA (0 if all in smem)
  int grid;               // persistent CTAs
  int64_t agg_off;        // workspace offset of per-CTA fp64 aggregate images (summary)
  int64_t agg_per_cta;    // bytes of one CTA's aggregate images
};

// Raise `func`'s dynamic shared-memory limit to at least `bytes` on the CURRENT device.
// cudaFuncSetAttribute is per device, so the configured size is tracked per
// (device, kernel) under a mutex: a process driving several GPUs (or several host
// threads) opts every kernel in on every device it launches on (holo_capi.cu).
cudaError_t ensure_smem_optin(const void* func, size_t bytes);

struct RunParams {
  Geometry g;
  DevTables t;
  Layout lay;
  const void* frames;
  int fmt, transpose;
  int B, A;
  const int32_t* members;
  const int32_t* wl;
  const float2* bcal;
  int cal_pols, cal_batch;
  int row_offset;          // global index of row 0: batch calibration is indexed by the global row (engine.py:247-249)
  const float2* rcal;
  int rcal_count;
  int16_t* fr;
  int16_t* fi;
  float* scale;
  float2* coefs;
  float2* raw;
  float2* windows;
  float* params;
  int param_slots;
  char* work;
  unsigned flags;
};

}  // namespace holo
