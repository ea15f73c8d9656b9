// Device helpers shared by the specialised 128-window kernels
// (holo_fast.cu: SIMT row pass; holo_fast_tc.cu: tcgen05 row DFT).
#pragma once
#include "holo_internal.h"

namespace holo {

// zs row (one row pair) layout, 2*WW+2 float2:
//   [0,32)        Z[-kx_c], c < 32        (read by column round 0)
//   [32,64)       Z[+kx_c], c < 32        (read by column round 0)
//   [64,64+R2)    Z[+kx_c], c >= 32       (read by column round 1, R2 = WW-32)
//   [64+R2,64+2R2) Z[-kx_c], c >= 32
// After round 0 the first 64 slots of every row are free and hold W.
template <int WW> HOLO_DEV int zs_pos(int c) { return c < 32 ? 32 + c : 64 + (c - 32); }
template <int WW> HOLO_DEV int zs_neg(int c) { return c < 32 ? c : 64 + (WW - 32) + (c - 32); }
template <int ZS> HOLO_DEV int w_addr(int i) { return (i >> 6) * ZS + (i & 63); }

// Compile-time Stockham stage over COUNT sequences of length N (index algebra
// in holo_fft.cuh); element e of sequence q at q*SS + e*ES.  MAPPED: the source
// is W inside zs (w_addr).
template <int P, int N, int L, int COUNT, int SS, int ES, bool INV, int MAPPED_ZS = 0>
HOLO_DEV void ct_stage(const float2* __restrict__ src, float2* __restrict__ dst, const float2* tw, int tid0 = -1,
                       int nthr = -1) {
  constexpr int m_in = N / L, mp = m_in / P, per = N / P, total = COUNT * per;
  if (tid0 < 0) { tid0 = threadIdx.x; nthr = blockDim.x; }
  for (int task = tid0; task < total; task += nthr) {
    int q, r;
    if (SS == 1) { q = task % COUNT; r = task / COUNT; }
    else { q = task / per; r = task - q * per; }
    const int k = r / mp, qp = r - k * mp;
    float2 v[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int i = q * SS + (k * m_in + qp + mp * j) * ES;
      v[j] = src[MAPPED_ZS ? w_addr<MAPPED_ZS>(i) : i];
    }
    if (L > 1) {
      // j*k*mp < N whenever (P-1)(L-1)mp < N (every stage of the 42 = 6 x 7 plans): no modulo
      constexpr bool kWrap = (P - 1) * (L - 1) * mp >= N;
#pragma unroll
      for (int j = 1; j < P; ++j) v[j] = cmul(v[j], twid<INV>(tw[kWrap ? (j * k * mp) % N : j * k * mp]));
    }
    dft_fixed<P, INV>(v);
#pragma unroll
    for (int t = 0; t < P; ++t) dst[q * SS + ((k + L * t) * mp + qp) * ES] = v[t];
  }
}

// Last stage of the inverse transform (along x, for every row y) with the
// epilogue fused in: reads T[c][y] (column-major), writes F[y][x] row-major,
// applies the removal phase (separable ey[y] * ex[x], incl. ifftshift sign and
// 1/(nx ny)), the optional batch calibration, and keeps the running max
// |Re|,|Im| for the int16 scale.
template <int P, int N, int L, int COUNT>
HOLO_DEV float ct_stage_final_rows(const float2* __restrict__ src, float2* __restrict__ dst, const float2* tw,
                                   const float2* ey, const float2* ex, bool use_bc, float2 bc, float osc = 1.f,
                                   int tid0 = -1, int nthr = -1, const float2* __restrict__ rc = nullptr) {
  constexpr int m_in = N / L, mp = m_in / P, per = N / P, total = COUNT * per;
  static_assert(mp == 1, "final stage");
  float lmax = 0.f;
  if (tid0 < 0) { tid0 = threadIdx.x; nthr = blockDim.x; }
  for (int task = tid0; task < total; task += nthr) {
    const int y = task % COUNT, k = task / COUNT;
    float2 v[P];
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = src[y + (k * m_in + j) * COUNT];
    constexpr bool kWrap = (P - 1) * (L - 1) >= N;
#pragma unroll
    for (int j = 1; j < P; ++j) v[j] = cmul(v[j], twid<true>(tw[kWrap ? (j * k) % N : j * k]));
    dft_fixed<P, true>(v);
    const float2 eyq = cscale(ey[y], osc);
    if (!use_bc && !rc) {   // the common case, without the predicated-off calibration multiplies
#pragma unroll
      for (int t = 0; t < P; ++t) {
        const int x = k + L * t;
        const float2 o = cmul(cmul(v[t], eyq), ex[x]);
        lmax = fmaxf(lmax, fmaxf(fabsf(o.x), fabsf(o.y)));
        dst[y * N + x] = o;
      }
      continue;
    }
#pragma unroll
    for (int t = 0; t < P; ++t) {
      const int x = k + L * t;
      float2 o = cmul(cmul(v[t], eyq), ex[x]);
      if (use_bc) o = cmul(o, bc);
      if (rc) o = cmul(o, __ldg(&rc[y * N + x]));   // reference calibration (engine.py:250-255)
      lmax = fmaxf(lmax, fmaxf(fabsf(o.x), fabsf(o.y)));
      dst[y * N + x] = o;
    }
  }
  return lmax;
}

// First half of a 128-point FFT with 16 points per thread (8 threads per
// transform): on entry z holds x[t + 8 j]; on exit z[k1] = W128^(t k1) DFT16(z)[k1].
HOLO_DEV void fft128_stage1(float2* z, int t, const float2* twt) {
  dft16<false>(z);
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) z[k1] = cmul(z[k1], twt[k1 * 8 + t]);   // W128^(t k1), conflict-free
}
// Second half for k1 = t + 8h: 8x8 transpose through the group's tile, DFT-8;
// v[k2] = X[t + 8h + 16 k2].
HOLO_DEV void fft128_stage2(const float2* z, int h, float2* xg, int t, float2* v) {
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) xg[kk * 9 + t] = z[8 * h + kk];
  __syncwarp();
#pragma unroll
  for (int tp = 0; tp < 8; ++tp) v[tp] = xg[t * 9 + tp];
  __syncwarp();
  dft8<false>(v);
}

}  // namespace holo
