// Tensor-core variant of the specialised 128-window kernel (tcgen05, sm_100a).
//
// The row pass -- a pruned 128-point R2C DFT of every window row, the largest
// block of floating-point work on the path -- is one GEMM on the 5th-generation
// tensor cores per window:
//
//   D[n][y] = sum_x A[n][x] * f[y][x]        M = 128 (n), N = 128 (y), K = 128 (x)
//   A[n][x] = Re / Im of exp(-2 pi i kx_c x / 128) * px[c]   (n = c / 64 + c)
//
// so D holds Re and Im of R[y][c] * px[c] for the WW bins the Fourier window
// keeps, with the recentring phase already applied (holopipe/pipeline.py:79-127).
// Precision is fp32-class through an fp16 split of both operands,
// A*f ~= Ah*fh + Al*fh + Ah*fl (products exact, fp32 accumulation; the frame is
// scaled by an exact power of two so fh+fl keep 22 bits).
//
//   A  (constant per pol)   TMEM columns [0,128): hi | lo, loaded once per CTA
//   f  (window, per item)   shared memory, canonical K-major layout, two K chunks
//   D  (accumulator)        TMEM columns [128,256), drained to shared memory
//
// Warp-specialised (one 512-thread CTA per SM, all 512 TMEM columns): warps 0-3
// stage windows and issue the 24 tcgen05.mma per window into one of two TMEM
// accumulators; warps 4-15 drain them and run everything after the row pass --
// column FFTs, 42x42 IFFT, removal phase, int16 packing, HG overlap -- with the
// SIMT code of holo_fast.cu (shared helpers in holo_fast_common.cuh).  Opt-in
// (HPG_FLAG_TC): the SIMT tail on 12 warps is slower than fast128_kernel.
#include <cuda_fp16.h>

#include <algorithm>

#include "holo_fast_common.cuh"
#include "holo_tc_common.cuh"
#include "holo_internal.h"

namespace holo {

namespace {

constexpr int kTcGroups = 48;   // consumer 8-thread groups
constexpr int kZP = 136;  // T plane row pitch (floats)

}  // namespace

template <int WH, int WW>
struct TcLayout {
  static constexpr int XG = 72;        // 8x8 exchange tile per 8-thread group (float2)
  static constexpr int GMAX = 48;
  static constexpr size_t stage = 0;                                                // f hi | lo, 8 K-steps
  static constexpr size_t stage_bytes = 2 * 8 * 4096;
  static constexpr size_t r0 = stage + stage_bytes;                                 // T planes / W / F / basis
  static constexpr size_t planes_bytes = 2 * (size_t)WW * kZP * sizeof(float);
  static constexpr size_t xbuf = (r0 + planes_bytes + 255) & ~size_t(255);          // [48][XG]
  static constexpr size_t twt = xbuf + kTcGroups * XG * sizeof(float2);             // [128]
  static constexpr size_t twh = twt + 128 * sizeof(float2);
  static constexpr size_t tww = twh + WH * sizeof(float2);
  static constexpr size_t ph = tww + WW * sizeof(float2);                           // py[WH] ex[WW] ey[WH]
  static constexpr size_t invs = (ph + (2 * WH + WW) * sizeof(float2) + 15) & ~size_t(15);   // [2][128]
  static constexpr size_t basis = invs + 2 * 128 * sizeof(float);
  static constexpr size_t basis_stage_off = ((WH * WW * sizeof(float2)) + 255) & ~size_t(255);  // in r0
  static_assert(WH * WW * sizeof(float2) <= planes_bytes, "W / F must fit r0");
  static_assert(basis_stage_off + (WH + WW) * GMAX * sizeof(float) <= planes_bytes, "basis staging must fit r0");
  static_assert(WH * WW * sizeof(float2) <= kTcGroups * XG * sizeof(float2), "IFFT ping-pong must fit xbuf");
  static_assert(WH * GMAX * sizeof(float2) <= kTcGroups * XG * sizeof(float2), "overlap U must fit xbuf");
  static_assert(WW <= 64 && WW <= kTcGroups, "one column round");
};

constexpr int kTcPersistentGP = 48;
constexpr int kProd = 128;           // producer threads (warps 0-3)
constexpr int kCons = 384;           // consumer threads (warps 4-15)
constexpr int kBarCons = 1, kBarProd = 2;


// Warp-specialised, software-pipelined over the CTA's windows k = 0, 1, ...:
//   producer (warps 0-3): window k -> registers (per-row power-of-two scale) ->
//     fp16 hi/lo in the canonical K-major layout -> 24 tcgen05.mma into
//     accumulator D[k & 1] -> commit (mbarrier fullD[k & 1])
//   consumer (warps 4-15): drain D[k & 1] (x 1/scale per row) -> release
//     (emptyD[k & 1]) -> column FFTs, IFFT, removal, int16, overlap
// so the tensor core, the HBM reads and the SIMT tail of consecutive windows overlap.
template <int WH, int WW>
__global__ void __launch_bounds__(kProd + kCons, 1) fast128tc_kernel(const __grid_constant__ RunParams p,
                                                                    const __grid_constant__ FastTables ft) {
  using LY = TcLayout<WH, WW>;
  extern __shared__ __align__(1024) char smem[];
  __shared__ float redf[16];
  __shared__ __align__(8) uint64_t fullD[2], emptyD[2], invsB[2];
  __shared__ uint32_t tbase;
  char* stage = smem + LY::stage;
  char* r0 = smem + LY::r0;
  float* planeRe = reinterpret_cast<float*>(r0);
  float* planeIm = planeRe + WW * kZP;
  float2* xbuf = reinterpret_cast<float2*>(smem + LY::xbuf);
  float2* twt = reinterpret_cast<float2*>(smem + LY::twt);
  float2* twh = reinterpret_cast<float2*>(smem + LY::twh);
  float2* tww = reinterpret_cast<float2*>(smem + LY::tww);
  float2* s_py = reinterpret_cast<float2*>(smem + LY::ph);
  float2* s_ex = s_py + WH;
  float2* s_ey = s_ex + WW;
  float* invs = reinterpret_cast<float*>(smem + LY::invs);
  const Geometry& g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = g.G, GP = (G + 3) & ~3;
  const bool keep_basis = p.coefs && G > 0 && GP <= kTcPersistentGP;
  float* hxP = reinterpret_cast<float*>(smem + LY::basis);   // [P][WW][GP] when kept

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fullD[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&emptyD[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&invsB[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = tid; i < 128; i += blockDim.x) twt[i] = p.t.tw_nx[((i >> 3) * (i & 7)) & 127];
  for (int i = tid; i < WH; i += blockDim.x) twh[i] = p.t.tw_gh[i];
  for (int i = tid; i < WW; i += blockDim.x) tww[i] = p.t.tw_gw[i];
  if (keep_basis) {   // every pol's basis, transposed [x][m] / [y][n], for the CTA's lifetime
    for (int i = tid; i < g.P * (GP / 4) * WW; i += blockDim.x) {
      const int q = i / ((GP / 4) * WW), r = i - q * (GP / 4) * WW, x = r % WW, m4 = 4 * (r / WW);
      const float* hx = p.t.hx + (size_t)q * G * WW;
      float4 hv;
      hv.x = m4 + 0 < G ? __ldg(&hx[(m4 + 0) * WW + x]) : 0.f;
      hv.y = m4 + 1 < G ? __ldg(&hx[(m4 + 1) * WW + x]) : 0.f;
      hv.z = m4 + 2 < G ? __ldg(&hx[(m4 + 2) * WW + x]) : 0.f;
      hv.w = m4 + 3 < G ? __ldg(&hx[(m4 + 3) * WW + x]) : 0.f;
      *reinterpret_cast<float4*>(&hxP[(q * (WW + WH) + x) * GP + m4]) = hv;
    }
    for (int i = tid; i < g.P * (GP / 4) * WH; i += blockDim.x) {
      const int q = i / ((GP / 4) * WH), r = i - q * (GP / 4) * WH, y = r % WH, n4 = 4 * (r / WH);
      const float* hy = p.t.hy + (size_t)q * G * WH;
      float4 hv;
      hv.x = n4 + 0 < G ? __ldg(&hy[(n4 + 0) * WH + y]) : 0.f;
      hv.y = n4 + 1 < G ? __ldg(&hy[(n4 + 1) * WH + y]) : 0.f;
      hv.z = n4 + 2 < G ? __ldg(&hy[(n4 + 2) * WH + y]) : 0.f;
      hv.w = n4 + 3 < G ? __ldg(&hy[(n4 + 3) * WH + y]) : 0.f;
      *reinterpret_cast<float4*>(&hxP[(q * (WW + WH) + WW + y) * GP + n4]) = hv;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;   // A hi [0,64) lo [64,128); D0 [128,256); D1 [256,384)
  const int items = p.B * g.P;
  const int W = g.W, H = g.H;

  if (warp < 4) {
    // ================================= producer =================================
    const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const int seg = tid & 3, rs = tid >> 2;   // 4 threads per row, 32 x each
    int loaded_q = -1;
    int k = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++k) {
      const int s = k & 1;
      const int b = item / g.P, q = item - b * g.P;
      const int row0 = g.row0[q], col0 = g.col0[q];
      {   // warm L2 with the next window of this CTA
        const int nitem = item + gridDim.x;
        if (nitem < items) {
          const int nb = nitem / g.P, nq = nitem - nb * g.P;
          const int es = p.fmt == 0 ? 4 : 2;
          const char* base = reinterpret_cast<const char*>(p.frames) +
                             ((int64_t)nb * W * H + (int64_t)g.row0[nq] * W + g.col0[nq]) * es;
          for (int i = tid; i < 128 * 5; i += kProd) {
            const int row = i / 5, part = i - row * 5;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (int64_t)row * W * es + min(part * 128, 128 * es - 1)));
          }
        }
      }
      if (k >= 1) {   // previous window's MMAs finished: stage buffer and A are free
        mbar_wait(&fullD[(k - 1) & 1], ((k - 1) >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      if (k >= 2) {   // the consumer drained D[s] (and read invs[s]) two windows ago
        mbar_wait(&emptyD[s], ((k >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      if (q != loaded_q) {
        const uint32_t* src = ft.a_tc + (size_t)q * 2 * 64 * 128 + warp * 32 + lane;   // column-major table
        uint32_t r[32];
#pragma unroll
        for (int part = 0; part < 2; ++part) {
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const uint32_t* s2 = src + ((size_t)part * 64 + half * 32) * 128;
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __ldg(s2 + j * 128);
            tmem_st32(tm + ((uint32_t)(warp * 32) << 16) + part * 64 + half * 32, r);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
        loaded_q = q;
      }
#pragma unroll 1
      for (int rp = 0; rp < 2; ++rp) {   // two rows per thread per pass, loads in flight together
        float v[2][32];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int y = rs + 32 * (2 * rp + rr);
          const int64_t base = (int64_t)b * W * H + (int64_t)(row0 + y) * W + col0 + 32 * seg;
          if (p.fmt == 0) {
            const float* src = reinterpret_cast<const float*>(p.frames) + base;
            if ((col0 & 3) == 0) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 a = __ldg(reinterpret_cast<const float4*>(src) + j);
                v[rr][4 * j] = a.x; v[rr][4 * j + 1] = a.y; v[rr][4 * j + 2] = a.z; v[rr][4 * j + 3] = a.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[rr][j] = __ldg(src + j);
            }
          } else {
            const unsigned short* src = reinterpret_cast<const unsigned short*>(p.frames) + base;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[rr][j] = (float)__ldg(src + j);
          }
        }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int y = rs + 32 * (2 * rp + rr);
          float m = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) m = fmaxf(m, fabsf(v[rr][j]));
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
          // exact power-of-two row scale: |f| * s < 2^14, fh + fl keep 22 bits
          int e2 = 0;
          frexpf(m, &e2);
          const float sc = m > 0.f ? ldexpf(1.f, 14 - e2) : 1.f;
          if (seg == 0) invs[s * 128 + y] = m > 0.f ? ldexpf(1.f, e2 - 14) : 1.f;
#pragma unroll
          for (int j = 0; j < 4; ++j) {          // octet j: x = 32 seg + 8 j
            const int gk = 2 * seg + (j >> 1), kh = j & 1;
            const uint32_t off = (uint32_t)gk * 4096 + ((uint32_t)((y >> 3) * 2 + kh) * 8 + (y & 7)) * 16;
            uint32_t hi2[4], lo2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a = v[rr][8 * j + 2 * e] * sc, c = v[rr][8 * j + 2 * e + 1] * sc;
              hi2[e] = pack_h2(a, c);
              const float2 back = __half22float2(*reinterpret_cast<const __half2*>(&hi2[e]));
              lo2[e] = pack_h2(a - back.x, c - back.y);
            }
            *reinterpret_cast<uint4*>(stage + off) = make_uint4(hi2[0], hi2[1], hi2[2], hi2[3]);
            *reinterpret_cast<uint4*>(stage + 32768 + off) = make_uint4(lo2[0], lo2[1], lo2[2], lo2[3]);
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      nbar(kBarProd, kProd);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (warp == 0 && elect_one()) {   // elect.sync: direct UTCHMMA issue (holo_tc_common.cuh)
        const uint32_t d = tm + 128 + 128 * s;
        const uint32_t sb = smem_u32(stage);
#pragma unroll
        for (int gk = 0; gk < 8; ++gk) {
          const uint64_t bh = umma_desc(sb + gk * 4096, 128, 256);
          const uint64_t bl = umma_desc(sb + 32768 + gk * 4096, 128, 256);
          mma_f16_ts(d, tm + gk * 8, bh, idesc, gk != 0);
          mma_f16_ts(d, tm + 64 + gk * 8, bh, idesc, 1);
          mma_f16_ts(d, tm + gk * 8, bl, idesc, 1);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&fullD[s])));
        mbar_arrive(&invsB[s]);
      }
    }
  } else {

  // ================================= consumer =================================
  const int ct = tid - kProd, t = ct & 7, grp = ct >> 3, cw = ct >> 5;
  float2* xg = xbuf + grp * LY::XG;
  int staged_q = -1;
  int k = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x, ++k) {
    const int s = k & 1;
    const int b = item / g.P, q = item - b * g.P;
    const int kys = (g.k0[q][0][1] - WH / 2) & 127;
    for (int i = ct; i < WH; i += kCons) {
      s_py[i] = ft.py[q * WH + i];
      s_ey[i] = p.t.rem_y[q * WH + i];
    }
    for (int i = ct; i < WW; i += kCons) s_ex[i] = p.t.rem_x[q * WW + i];
    mbar_wait(&fullD[s], (k >> 1) & 1);
    mbar_wait(&invsB[s], (k >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    nbar(kBarCons, kCons);

    // ------------------------------------------------ drain D -> T planes [c][y]
    {
      const int quarter = warp & 3, part = (warp - 4) >> 2;
      const int n = quarter * 32 + lane, c = n & 63;
      float* plane = (n < 64 ? planeRe : planeIm) + c * kZP;
      const float* iv = invs + s * 128;
      const int y_begin = part * 48, y_end = part == 2 ? 128 : y_begin + 48;
      const uint32_t d = tm + 128 + 128 * s;
#pragma unroll 1
      for (int y0 = y_begin; y0 < y_end; y0 += 16) {
        uint32_t r[16];
        tmem_ld16(d + ((uint32_t)(quarter * 32) << 16) + y0, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (c < WW) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const float4 sc = *reinterpret_cast<const float4*>(iv + y0 + j);
            *reinterpret_cast<float4*>(plane + y0 + j) =
                make_float4(__uint_as_float(r[j]) * sc.x, __uint_as_float(r[j + 1]) * sc.y,
                            __uint_as_float(r[j + 2]) * sc.z, __uint_as_float(r[j + 3]) * sc.w);
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    nbar(kBarCons, kCons);
    if (ct == 0) mbar_arrive(&emptyD[s]);

    // --------------------------------------------------------- column pass
    float2 o0[8], o1[8];
    const int c = grp;
    const bool active = c < WW;
    if ((cw * 4) < WW) {
      float2 z[16];
      if (active) {
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = make_float2(planeRe[c * kZP + t + 8 * j], planeIm[c * kZP + t + 8 * j]);
        fft128_stage1(z, t, twt);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = make_float2(0.f, 0.f);
      }
      fft128_stage2(z, 0, xg, t, o0);
      fft128_stage2(z, 1, xg, t, o1);
    }
    nbar(kBarCons, kCons);   // every T plane read: r0 now hosts W (column-major)
    float2* Wt = reinterpret_cast<float2*>(r0);
    if (active) {
      const int rlo = ft.crange[2 * c], rhi = ft.crange[2 * c + 1];
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = (t + 8 * h + 16 * k2 - kys) & 127;
          if (r < WH) {
            float2 val = make_float2(0.f, 0.f);
            if (r >= rlo && r <= rhi) val = cmul(h ? o1[k2] : o0[k2], s_py[r]);
            Wt[c * WH + r] = val;
          }
        }
      }
    }
    nbar(kBarCons, kCons);

    // ------------------------------------------------ IFFT (along y, then along x)
    float2* T = xbuf;
    float2* F = reinterpret_cast<float2*>(r0);
    ct_stage<6, WH, 1, WW, WH, 1, true>(Wt, T, twh, ct, kCons);
    nbar(kBarCons, kCons);
    ct_stage<7, WH, 6, WW, WH, 1, true>(T, F, twh, ct, kCons);
    nbar(kBarCons, kCons);
    ct_stage<6, WW, 1, WH, 1, WH, true>(F, T, tww, ct, kCons);
    nbar(kBarCons, kCons);
    // ------------------------------------------- removal phase, peak, int16
    float2 bc = make_float2(1.f, 0.f);
    if (p.bcal) bc = p.bcal[(size_t)min(q, p.cal_pols - 1) * p.cal_batch + ((p.row_offset + b) % p.cal_batch)];
    float lmax = ct_stage_final_rows<7, WW, 6, WH>(T, F, tww, s_ey, s_ex, p.bcal != nullptr, bc, 1.f, ct, kCons);
#pragma unroll
    for (int o = 16; o; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    if (lane == 0) redf[cw] = lmax;
    nbar(kBarCons, kCons);
    lmax = redf[0];
#pragma unroll
    for (int j = 1; j < kCons / 32; ++j) lmax = fmaxf(lmax, redf[j]);
    if (p.raw)
      for (int i = ct; i < WH * WW; i += kCons) p.raw[(size_t)item * WH * WW + i] = F[i];
    const float scale = lmax > 0.f ? (float)(32767.0 / (double)lmax) : 1.0f;
    int16_t* fro = p.fr + (size_t)item * WH * WW;
    int16_t* fio = p.fi + (size_t)item * WH * WW;
    for (int i = ct; i < WH * WW / 2; i += kCons) {
      const float4 vv = reinterpret_cast<const float4*>(F)[i];
      const int ra = __float2int_rn(__fmul_rn(vv.x, scale)), ia = __float2int_rn(__fmul_rn(vv.y, scale));
      const int rb = __float2int_rn(__fmul_rn(vv.z, scale)), ib = __float2int_rn(__fmul_rn(vv.w, scale));
      reinterpret_cast<int*>(fro)[i] = (ra & 0xffff) | (rb << 16);
      reinterpret_cast<int*>(fio)[i] = (ia & 0xffff) | (ib << 16);
      reinterpret_cast<float4*>(F)[i] = make_float4((float)ra, (float)ia, (float)rb, (float)ib);
    }
    if (ct == 0) p.scale[item] = scale;

    // ---------------------------------------------------------- HG overlap
    if (p.coefs && G > 0) {
      float* hxT;
      float* hyT;
      if (keep_basis) {
        hxT = hxP + (size_t)q * (WW + WH) * GP;
        hyT = hxT + WW * GP;
      } else {
        hxT = reinterpret_cast<float*>(r0 + LY::basis_stage_off);
        hyT = hxT + WW * GP;
        if (q != staged_q) {
          const float* hx = p.t.hx + (size_t)q * G * WW;
          const float* hy = p.t.hy + (size_t)q * G * WH;
          for (int i = ct; i < (GP / 4) * WW; i += kCons) {
            const int x = i % WW, m4 = 4 * (i / WW);
            float4 hv;
            hv.x = m4 + 0 < G ? __ldg(&hx[(m4 + 0) * WW + x]) : 0.f;
            hv.y = m4 + 1 < G ? __ldg(&hx[(m4 + 1) * WW + x]) : 0.f;
            hv.z = m4 + 2 < G ? __ldg(&hx[(m4 + 2) * WW + x]) : 0.f;
            hv.w = m4 + 3 < G ? __ldg(&hx[(m4 + 3) * WW + x]) : 0.f;
            *reinterpret_cast<float4*>(&hxT[x * GP + m4]) = hv;
          }
          for (int i = ct; i < (GP / 4) * WH; i += kCons) {
            const int y = i % WH, n4 = 4 * (i / WH);
            float4 hv;
            hv.x = n4 + 0 < G ? __ldg(&hy[(n4 + 0) * WH + y]) : 0.f;
            hv.y = n4 + 1 < G ? __ldg(&hy[(n4 + 1) * WH + y]) : 0.f;
            hv.z = n4 + 2 < G ? __ldg(&hy[(n4 + 2) * WH + y]) : 0.f;
            hv.w = n4 + 3 < G ? __ldg(&hy[(n4 + 3) * WH + y]) : 0.f;
            *reinterpret_cast<float4*>(&hyT[y * GP + n4]) = hv;
          }
        }
      }
      nbar(kBarCons, kCons);
      float2* U = xbuf;
      const int GQ = GP >> 2;
      for (int idx = ct; idx < WH * GQ; idx += kCons) {
        const int y = idx / GQ, mq = idx - y * GQ;
        const float2* row = F + y * WW;
        float4 ar = make_float4(0.f, 0.f, 0.f, 0.f), ai = ar;
#pragma unroll 6
        for (int x = 0; x < WW; ++x) {
          const float2 vx = row[x];
          const float4 hv = *reinterpret_cast<const float4*>(&hxT[x * GP + 4 * mq]);
          ar.x = fmaf(vx.x, hv.x, ar.x); ai.x = fmaf(vx.y, hv.x, ai.x);
          ar.y = fmaf(vx.x, hv.y, ar.y); ai.y = fmaf(vx.y, hv.y, ai.y);
          ar.z = fmaf(vx.x, hv.z, ar.z); ai.z = fmaf(vx.y, hv.z, ai.z);
          ar.w = fmaf(vx.x, hv.w, ar.w); ai.w = fmaf(vx.y, hv.w, ai.w);
        }
        float2* u = U + y * GP + 4 * mq;
        u[0] = make_float2(ar.x, ai.x);
        u[1] = make_float2(ar.y, ai.y);
        u[2] = make_float2(ar.z, ai.z);
        u[3] = make_float2(ar.w, ai.w);
      }
      nbar(kBarCons, kCons);
      const float dd = __fdiv_rn(g.dxdy[q], scale);
      float2* out = p.coefs + (size_t)item * g.M;
      for (int i = ct; i < g.M; i += kCons) {
        const int m = p.t.mode_m[i], n = p.t.mode_n[i];
        float ax = 0.f, ay = 0.f;
#pragma unroll 6
        for (int y = 0; y < WH; ++y) {
          const float2 uv = U[y * GP + m];
          const float hv = hyT[y * GP + n];
          ax = fmaf(uv.x, hv, ax);
          ay = fmaf(uv.y, hv, ay);
        }
        out[i] = make_float2(ax * dd, ay * dd);
      }
      staged_q = keep_basis ? -1 : q;
    }
    nbar(kBarCons, kCons);   // window done: r0, xbuf and the per-window tables may be reused
  }
  }
  // every accumulator was drained by the consumer: the allocating warp frees TMEM
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

bool tc_supported(const Geometry& g, int A, int fmt, int transpose, int fill, const void* rcal, unsigned flags,
                  const void* windows) {
  return g.nx == 128 && g.ny == 128 && g.wh == 42 && g.ww == 42 && g.gh == 42 && g.gw == 42 && A == 1 && g.L == 1 &&
         g.G <= TcLayout<42, 42>::GMAX && !(fmt == 1 && transpose) && !fill && rcal == nullptr &&
         (flags & 1u) == 0 && windows == nullptr;
}

cudaError_t launch_fast_tc(const RunParams& p, const FastTables& ft, int num_sms, cudaStream_t s) {
  using LY = TcLayout<42, 42>;
  const int GP = (p.g.G + 3) & ~3;
  size_t bytes = LY::basis + ((p.coefs && p.g.G > 0 && GP <= kTcPersistentGP)
                                  ? (size_t)p.g.P * (42 + 42) * GP * sizeof(float) : 0) + 64;
  // one CTA per SM: it owns all 512 TMEM columns
  bytes = std::max(bytes, (size_t)120 * 1024);
  cudaError_t e = ensure_smem_optin((const void*)fast128tc_kernel<42, 42>, bytes);
  if (e != cudaSuccess) return e;
  const int items = p.B * p.g.P;
  const int grid = std::max(1, std::min(items, num_sms));
  fast128tc_kernel<42, 42><<<grid, kProd + kCons, bytes, s>>>(p, ft);
  return cudaGetLastError();
}

}  // namespace holo
