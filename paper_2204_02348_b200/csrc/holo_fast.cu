// Fused kernel for the hot geometry class: 128 x 128 FFT window, a WH x WW
// (42 x 42 for BASELINE) Fourier window, IFFT resolution mode 1, no
// averaging (fill-factor envelope and reference calibration are folded in).
// Same algorithm and numerical conventions as the generic kernel
// (holo_pipeline.cu) with every size a compile-time constant.  One (frame, pol)
// item per 256-thread CTA at a time, three CTAs per SM (64 KB shared memory,
// <= 85 registers); TCO = true moves the HG overlap onto tcgen05 (G > 16):
//
//   row pass    8 threads per (row y, row y+64) pair, 16 points per thread:
//               DFT-16 in registers -> twiddle W128^(t k1) -> two 8x8
//               transposes through a padded shared tile -> DFT-8 -> keep only
//               the bins the window needs, Z[kx_c] and Z[-kx_c] (the two halves
//               of the Hermitian split, holopipe/pipeline.py:89-98), in zs
//   column pass 8 threads per kept column: Hermitian split on load, same
//               128-point FFT, keep the WH needed rows, circular mask (row
//               range per column) * separable recentring phase (pipeline.py:72-127).
//               The window W is written into the zs slots the first column
//               round has already consumed (zs row layout below).
//   IFFT        compile-time Stockham (42 = 6 x 7) along rows then columns
//               (pipeline.py:130-149); removal phase (pipeline.py:163-185) and
//               the peak search fused into the last stage
//   epilogue    int16 packing (pipeline.py:188-199) and the separable HG
//               overlap (hgbasis.py:101-116) on the integer-valued field with
//               the 1/scale of the dequantisation folded into the coefficients
//
// Frames are read straight from HBM into registers (each warp load touches
// four full 32-byte sectors): HBM traffic is the window read and the int16 /
// scale / coefficient writes.
#include <algorithm>

#include "holo_internal.h"
#include "holo_fast_common.cuh"
#include "holo_tc_common.cuh"

namespace holo {

template <int WH, int WW, int NT = 256>
struct FastLayout {
  static constexpr int ZS = 2 * WW + 2;            // zs row pitch (float2)
  static constexpr int XG = 72;                    // 8x8 exchange tile per 8-thread group (float2)
  static constexpr int NG = NT / 8;                // 8-thread FFT groups per CTA
  static constexpr int GMAX = 48;                  // max basis orders on this path
  static constexpr size_t zs = 0;                                          // [64][ZS]
  static constexpr size_t xbuf = zs + 64 * ZS * sizeof(float2);            // [NG][XG]
  static constexpr size_t tw128 = xbuf + NG * XG * sizeof(float2);         // [128]
  static constexpr size_t twh = tw128 + 128 * sizeof(float2);              // [WH]
  static constexpr size_t tww = twh + WH * sizeof(float2);                 // [WW]
  static constexpr size_t ph = tww + WW * sizeof(float2);                  // px[WW] py[WH] ex[WW] ey[WH]
  static constexpr size_t bytes = ph + 2 * (WH + WW) * sizeof(float2) + 64;
  // after the IFFT, zs holds F (linear, [WH][WW]) then the staged basis
  static constexpr size_t basis_off = ((WH * WW * sizeof(float2)) + 255) & ~size_t(255);
  static_assert(WW > 32 && WW <= 64 && WH <= 64, "zs row layout assumes two column rounds");
  static_assert((WH * WW + 63) / 64 <= 64, "W must fit the freed zs slots");
  static_assert(WH * WW * sizeof(float2) <= 32 * XG * sizeof(float2), "IFFT ping-pong must fit xbuf");
  static_assert(WH * GMAX * sizeof(float2) <= 32 * XG * sizeof(float2), "overlap U must fit xbuf");
  static_assert(basis_off + (WH + WW) * GMAX * sizeof(float) <= 64 * ZS * sizeof(float2), "basis must fit zs");
};

// the transposed basis of one pol stays resident when it fits next to the 64 KB layout
// without dropping below 3 CTAs per SM
constexpr int kPersistentBasisGP = 36;
HOLO_DEV bool persistent_basis(int GP) { return GP <= kPersistentBasisGP; }

// Tensor-core HG overlap (TCO): operands in shared memory, UMMA K-major layout
// [row/8][kstep 3][khalf][row%8][8 halves] (SBO 768 B, kstep 256 B, LBO 128 B).
//   GEMM 1: U[(Re y | Im 48+y)][m] = sum_x F16[y][x] qx[m][x]   M=128 N=GP16 K=48
//   GEMM 2: C[(Re m | Im 48+m)][n] = sum_y U[y][m] qy[n][y]      (U scaled by 2^-22, fp16 hi/lo)
// F16 (the int16 field) and q (the int16 basis) split exactly as 32 (v >> 5) + (v & 31).
constexpr unsigned kFlagNoTco = 32u;          // HPG_FLAG_SIMT_OVERLAP
constexpr uint32_t kTcoA = 16384;              // A operand (F16 split, then U split) at zs + 16 KB
constexpr uint32_t kTcoPart = 12 * 768;        // one part: 96 rows x 48 K halves
HOLO_DEV uint32_t tco_off(int row, int k) {    // byte offset of (row, k) in one operand part
  return (uint32_t)(row >> 3) * 768 + (uint32_t)(k >> 4) * 256 + (uint32_t)((k >> 3) & 1) * 128 +
         (uint32_t)(row & 7) * 16 + (uint32_t)(k & 7) * 2;
}
HOLO_DEV void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// The overlap of one item on the tensor cores.  On entry the A operand (the int16 field split)
// is complete in shared memory except the padding rows; B operands are staged into `bsm`.
template <int WH, int WW>
HOLO_DEV void tco_overlap(const RunParams& p, const FastTables& ft, int item, int q, float scale, char* A, char* bsm,
                          uint32_t tm, uint64_t* bar, uint32_t& phase) {
  const Geometry& g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = g.G, GP = ft.tco_gp;
  const uint32_t part = (uint32_t)GP * 96;   // bytes of one B part (GP rows x 48 halves)
  {   // padding rows 42..47 and 90..95 of A (all K, both parts): 12 rows x 6 chunks x 2
    for (int i = tid; i < 12 * 6 * 2; i += blockDim.x) {
      const int pr = i / 12, rr = i - pr * 12, row = rr < 6 ? WH + rr : 48 + WH + (rr - 6);
      const int kc = pr % 6, pt = pr / 6;
      *reinterpret_cast<uint4*>(A + pt * kTcoPart + tco_off(row, 8 * kc)) = make_uint4(0u, 0u, 0u, 0u);
    }
    // B images of this pol (hx hi | hx lo | hy hi | hy lo)
    const uint4* src = ft.tco_img + (size_t)q * 4 * part / 16;
    for (int i = tid; i < (int)(4 * part / 16); i += blockDim.x) reinterpret_cast<uint4*>(bsm)[i] = __ldg(src + i);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t idesc = idesc_f16(128, GP);
  const uint32_t sa = smem_u32(A), sb = smem_u32(bsm);
  // issued under elect.sync by the converged warp 0 (holo_tc_common.cuh: 112 -> ~40 cycles per issued MMA)
  if (warp == 0 && elect_one()) {   // GEMM 1: D1[row][m] = sum_x A[row][x] qx[m][x]
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) {
      const uint64_t ah = umma_desc(sa + ks * 256, 128, 768), al = umma_desc(sa + kTcoPart + ks * 256, 128, 768);
      const uint64_t bh = umma_desc(sb + ks * 256, 128, 768), bl = umma_desc(sb + part + ks * 256, 128, 768);
      mma_f16_ss(tm, ah, bh, idesc, ks != 0);
      mma_f16_ss(tm, ah, bl, idesc, 1);
      mma_f16_ss(tm, al, bh, idesc, 1);
      mma_f16_ss(tm, al, bl, idesc, 1);   // all four integer products: GEMM 1 is exact
    }
    tc_commit(bar);
  }
  mbar_wait(bar, phase & 1);
  ++phase;
  tc_fence_after();
  {   // drain D1 -> A (now the GEMM-2 operand U^T: rows Re m | Im 48+m, K = y), scaled by 2^-22
    const int quarter = warp & 3, hcol = warp >> 2;
    const int row = quarter * 32 + lane;   // D1 row: Re y (< 48) or Im y (48..95)
    const int yy = row < 48 ? row : row - 48, im = row >= 48;
    const int half = GP / 2;
    for (int c0 = hcol * half; c0 < (hcol + 1) * half; c0 += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tm + ((uint32_t)(quarter * 32) << 16) + c0));
      tmem_wait_ld();
      if (row < 96) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float u = __uint_as_float(r[e]) * 2.384185791015625e-07f;   // 2^-22
          const __half h = __float2half_rn(u);
          const __half l = __float2half_rn(u - __half2float(h));
          const int m = c0 + e;
          const uint32_t o = tco_off(im * 48 + m, yy);
          *reinterpret_cast<__half*>(A + o) = h;
          *reinterpret_cast<__half*>(A + kTcoPart + o) = l;
        }
      }
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && elect_one()) {   // GEMM 2: D2[row2][n] = sum_y A[row2][y] qy[n][y]
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) {
      const uint64_t ah = umma_desc(sa + ks * 256, 128, 768), al = umma_desc(sa + kTcoPart + ks * 256, 128, 768);
      const uint64_t bh = umma_desc(sb + 2 * part + ks * 256, 128, 768),
                     bl = umma_desc(sb + 3 * part + ks * 256, 128, 768);
      mma_f16_ss(tm + 64, ah, bh, idesc, ks != 0);
      mma_f16_ss(tm + 64, al, bh, idesc, 1);
      mma_f16_ss(tm + 64, ah, bl, idesc, 1);
    }
    tc_commit(bar);
  }
  mbar_wait(bar, phase & 1);
  ++phase;
  tc_fence_after();
  {   // drain D2 -> coefficients (group-major index of (m, n), engine.py / hgbasis.py:17-27)
    const int quarter = warp & 3, hcol = warp >> 2;
    const int row = quarter * 32 + lane;
    const int m = row < 48 ? row : row - 48, im = row >= 48;
    const float d = __fdiv_rn(g.dxdy[q], scale) * 4194304.f;   // 2^22 undoes the U scaling
    const float* invx = ft.tco_inv + (size_t)q * 2 * GP;
    const float* invy = invx + GP;
    float* out = reinterpret_cast<float*>(p.coefs + (size_t)item * g.M) + im;
    const float fm = (row < 96 && m < G) ? d * __ldg(&invx[m]) : 0.f;
    const int half = GP / 2;
    for (int c0 = hcol * half; c0 < (hcol + 1) * half; c0 += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tm + 64 + ((uint32_t)(quarter * 32) << 16) + c0));
      tmem_wait_ld();
      if (row < 96 && m < G) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int n = c0 + e, gg = m + n;
          if (gg < G) out[2 * (gg * (gg + 1) / 2 + n)] = __uint_as_float(r[e]) * fm * __ldg(&invy[n]);
        }
      }
    }
  }
  tc_fence_before();
}

// NT = 256: the throughput configuration (3 CTAs/SM).  NT = 512: one window per SM with every phase in a
// single round, for batches smaller than the SM count (latency-bound, e.g. PR1's 16 windows).
template <int WH, int WW, bool TCO, int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 3 : 1) fast128_kernel(const __grid_constant__ RunParams p,
                                                                       const __grid_constant__ FastTables ft) {
  using LY = FastLayout<WH, WW, NT>;
  constexpr int ZS = LY::ZS, NG = LY::NG, NW = NT / 32;
  static_assert(!TCO || NT == 256, "the TMEM drain assumes 8 warps");
  extern __shared__ __align__(16) char smem[];
  __shared__ float redf[NW];
  __shared__ int slot[128];
  __shared__ int slot_both;
  int slot_kxs = -1;
  float2* zs = reinterpret_cast<float2*>(smem + LY::zs);
  float2* xbuf = reinterpret_cast<float2*>(smem + LY::xbuf);
  float2* tw128 = reinterpret_cast<float2*>(smem + LY::tw128);
  float2* twh = reinterpret_cast<float2*>(smem + LY::twh);
  float2* tww = reinterpret_cast<float2*>(smem + LY::tww);
  float2* s_px = reinterpret_cast<float2*>(smem + LY::ph);
  float2* s_py = s_px + WW;
  float2* s_ex = s_py + WH;
  float2* s_ey = s_ex + WW;
  const Geometry& g = p.g;
  const int tid = threadIdx.x, t = tid & 7, grp = tid >> 3;
  float2* xg = xbuf + grp * LY::XG;

  for (int i = tid; i < 128; i += blockDim.x) tw128[i] = p.t.tw_nx[((i >> 3) * (i & 7)) & 127];
  for (int i = tid; i < WH; i += blockDim.x) twh[i] = p.t.tw_gh[i];
  for (int i = tid; i < WW; i += blockDim.x) tww[i] = p.t.tw_gw[i];
  __shared__ __align__(8) uint64_t tco_bar;
  __shared__ uint32_t tco_tbase;
  uint32_t tco_phase = 0;
  if (TCO) {
    if ((tid >> 5) == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tco_tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
      mbar_init(&tco_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  const int items = p.B * g.P;
  int staged_q = -1;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int b = g.P == 1 ? item : (g.P == 2 ? item >> 1 : item / g.P), q = item - b * g.P;
    const int w = p.wl ? p.wl[b] : 0;
    const int pl = q * g.L + w;
    const int kxs = (g.k0[q][w][0] - WW / 2) & 127, kys = (g.k0[q][w][1] - WH / 2) & 127;
    __syncthreads();  // previous item done with every buffer
    for (int i = tid; i < WW; i += blockDim.x) {
      s_px[i] = ft.px[pl * WW + i];
      s_ex[i] = p.t.rem_x[pl * WW + i];
    }
    for (int i = tid; i < WH; i += blockDim.x) {
      s_py[i] = ft.py[pl * WH + i];
      s_ey[i] = p.t.rem_y[pl * WH + i];
    }
    if (kxs != slot_kxs) {   // FFT bin -> zs slots: primary | secondary << 16 (-1 = none)
      if (tid == 0) slot_both = 0;
      __syncthreads();
      for (int kk = tid; kk < 128; kk += blockDim.x) {
        const int cp = (kk - kxs) & 127, cm = (128 - kk - kxs) & 127;
        const int sp = cp < WW ? zs_pos<WW>(cp) : -1, sn = cm < WW ? zs_neg<WW>(cm) : -1;
        // a bin is normally in the +kx window or the mirrored -kx one; both only when the window
        // reaches kx = 0 or nx/2 -- then the secondary slot is used (flag checked per item)
        const int pri = sp >= 0 ? sp : sn, sec = sp >= 0 ? sn : -1;
        slot[kk] = (pri & 0xffff) | (sec << 16);
        if (sec >= 0) slot_both = 1;
      }
      slot_kxs = kxs;
      __syncthreads();
    }
    const bool both = slot_both != 0;

    // ------------------------------------------------------------ row pass
    const int W = g.W, H = g.H;
#pragma unroll 1
    for (int pr = grp; pr < 64; pr += NG) {   // warp-uniform trip count
      float2 z[16];
      if (p.fmt == 0) {
        const float* fa = reinterpret_cast<const float*>(p.frames) + (int64_t)b * W * H +
                          (int64_t)(g.row0[q] + pr) * W + g.col0[q] + t;
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = make_float2(__ldg(fa + 8 * j), __ldg(fa + 64 * W + 8 * j));
      } else {
        const unsigned short* fa = reinterpret_cast<const unsigned short*>(p.frames) + (int64_t)b * W * H +
                                   (int64_t)(g.row0[q] + pr) * W + g.col0[q] + t;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          z[j] = make_float2((float)__ldg(fa + 8 * j), (float)__ldg(fa + 64 * W + 8 * j));
      }
      fft128_stage1(z, t, tw128);
      float2* zrow = zs + pr * ZS;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float2 v[8];
        fft128_stage2(z, h, xg, t, v);
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) {
          const int sl = slot[t + 8 * h + 16 * k2];   // zs slot(s) of bin kk: +kx_c and/or -kx_c
          const int sp = (short)(sl & 0xffff);
          if (sp >= 0) zrow[sp] = v[k2];
          if (both) {
            const int sn = sl >> 16;
            if (sn >= 0) zrow[sn] = v[k2];
          }
        }
      }
    }
    __syncthreads();
    {
      // warm L2 with the window this CTA processes next (its HBM latency then
      // hides behind this item's column pass, IFFT and overlap)
      const int nitem = item + gridDim.x;
      if (nitem < items) {
        const int nb = nitem / g.P, nq = nitem - nb * g.P;
        const int es = p.fmt == 0 ? 4 : 2;
        const char* base = reinterpret_cast<const char*>(p.frames) +
                           ((int64_t)nb * W * H + (int64_t)g.row0[nq] * W + g.col0[nq]) * es;
        if (tid < 128) {   // one bulk prefetch per window row: the 16-byte aligned span inside the row
          const uintptr_t a = reinterpret_cast<uintptr_t>(base + (int64_t)tid * W * es);
          const uintptr_t a0 = (a + 15) & ~uintptr_t(15), a1 = (a + 128 * es) & ~uintptr_t(15);
          if (a1 > a0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
        }
      }
    }

    // --------------------------------------------------------- column pass
#pragma unroll 1
    for (int rnd = 0; rnd < (WW + NG - 1) / NG; ++rnd) {
      const int c = rnd * NG + grp;
      const bool active = c < WW;
      // warps whose four groups are all past the last column skip the round (the exchange is warp-local)
      if (rnd > 0 && rnd * NG + ((tid >> 5) << 2) >= WW) continue;
      float2 z[16];
      if (active) {
        const int sp = zs_pos<WW>(c), sn = zs_neg<WW>(c);
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const float2 zk = zs[(t + 8 * jj) * ZS + sp], zm = zs[(t + 8 * jj) * ZS + sn];
          z[jj] = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
          z[jj + 8] = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
        }
        fft128_stage1(z, t, tw128);
      } else {
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) z[jj] = make_float2(0.f, 0.f);
      }
      float2 o0[8], o1[8];
      fft128_stage2(z, 0, xg, t, o0);   // all lanes take part in the warp exchange
      fft128_stage2(z, 1, xg, t, o1);
      if (rnd == 0) __syncthreads();    // round 0 consumed zs slots [0,64) of every row
      if (active) {
        const float2 pxc = s_px[c];
        const int rlo = ft.crange[2 * c], rhi = ft.crange[2 * c + 1];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = (t + 8 * h + 16 * k2 - kys) & 127;
            if (r < WH) {
              float2 val = make_float2(0.f, 0.f);
              if (r >= rlo && r <= rhi) val = cmul(h ? o1[k2] : o0[k2], cmul(s_py[r], pxc));
              zs[w_addr<ZS>(c * WH + r)] = val;
            }
          }
        }
      }
    }
    __syncthreads();

    // ------------------------------------------------ IFFT (rows, then columns)
    float2* T = xbuf;
    float2* F = zs;   // linear [WH][WW] once the mapped W has been consumed
    // W is column-major (WT[c][r]): transform along r (y) first, then along c (x)
    ct_stage<6, WH, 1, WW, WH, 1, true, ZS>(zs, T, twh);
    __syncthreads();
    ct_stage<7, WH, 6, WW, WH, 1, true>(T, F, twh);
    __syncthreads();
    ct_stage<6, WW, 1, WH, 1, WH, true>(F, T, tww);
    __syncthreads();
    // ------------------------------------------- removal phase, peak, int16
    float2 bc = make_float2(1.f, 0.f);
    if (p.bcal) bc = p.bcal[(size_t)min(q, p.cal_pols - 1) * p.cal_batch + ((p.row_offset + b) % p.cal_batch)];
    const float2* rc = p.rcal ? p.rcal + ((size_t)(w % p.rcal_count) * g.P + q) * WH * WW : nullptr;
    float lmax = ct_stage_final_rows<7, WW, 6, WH>(T, F, tww, s_ey, s_ex, p.bcal != nullptr, bc, 1.f, -1, -1, rc);
#pragma unroll
    for (int o = 16; o; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    if ((tid & 31) == 0) redf[tid >> 5] = lmax;
    __syncthreads();
    lmax = redf[0];
#pragma unroll
    for (int j = 1; j < NW; ++j) lmax = fmaxf(lmax, redf[j]);
    if (p.raw)
      for (int i = tid; i < WH * WW; i += blockDim.x) p.raw[(size_t)item * WH * WW + i] = F[i];
    const float scale = lmax > 0.f ? (float)(32767.0 / (double)lmax) : 1.0f;
    int16_t* fro = p.fr + (size_t)item * WH * WW;
    int16_t* fio = p.fi + (size_t)item * WH * WW;
    for (int i = tid; i < WH * WW / 2; i += blockDim.x) {
      const float4 v = reinterpret_cast<const float4*>(F)[i];
      const int r0 = __float2int_rn(__fmul_rn(v.x, scale)), i0 = __float2int_rn(__fmul_rn(v.y, scale));
      const int r1 = __float2int_rn(__fmul_rn(v.z, scale)), i1 = __float2int_rn(__fmul_rn(v.w, scale));
      reinterpret_cast<int*>(fro)[i] = (r0 & 0xffff) | (r1 << 16);
      reinterpret_cast<int*>(fio)[i] = (i0 & 0xffff) | (i1 << 16);
      if (TCO) {   // exact fp16 split of the int16 field into the GEMM-1 A operand (rows Re y | Im 48+y)
        const int y = (2 * i) / WW, x = 2 * i - y * WW;
        char* A = reinterpret_cast<char*>(zs) + kTcoA;
        const uint32_t hr = pack_h2((float)(32 * (r0 >> 5)), (float)(32 * (r1 >> 5)));
        const uint32_t lr = pack_h2((float)(r0 & 31), (float)(r1 & 31));
        const uint32_t hi_ = pack_h2((float)(32 * (i0 >> 5)), (float)(32 * (i1 >> 5)));
        const uint32_t li = pack_h2((float)(i0 & 31), (float)(i1 & 31));
        if (x == WW - 2) {   // last pair of the row: also clear the K padding x = WW .. 47 (16-byte chunk)
          *reinterpret_cast<uint4*>(A + tco_off(y, x)) = make_uint4(hr, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(A + kTcoPart + tco_off(y, x)) = make_uint4(lr, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(A + tco_off(48 + y, x)) = make_uint4(hi_, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(A + kTcoPart + tco_off(48 + y, x)) = make_uint4(li, 0u, 0u, 0u);
        } else {
          *reinterpret_cast<uint32_t*>(A + tco_off(y, x)) = hr;
          *reinterpret_cast<uint32_t*>(A + kTcoPart + tco_off(y, x)) = lr;
          *reinterpret_cast<uint32_t*>(A + tco_off(48 + y, x)) = hi_;
          *reinterpret_cast<uint32_t*>(A + kTcoPart + tco_off(48 + y, x)) = li;
        }
      } else {
        // integer-valued copy for the overlap; the 1/scale of the dequantisation
        // (holopipe/engine.py:367-369) is applied once to each coefficient
        reinterpret_cast<float4*>(F)[i] = make_float4((float)r0, (float)i0, (float)r1, (float)i1);
      }
    }
    if (tid == 0) p.scale[item] = scale;

    // ---------------------------------------------------------- HG overlap
    if (TCO && p.coefs && g.G > 0) {
      tco_overlap<WH, WW>(p, ft, item, q, scale, reinterpret_cast<char*>(zs) + kTcoA,
                          reinterpret_cast<char*>(xbuf), tco_tbase, &tco_bar, tco_phase);
    } else if (p.coefs && g.G > 0) {
      const int G = g.G, GP = (G + 3) & ~3;
      // basis, transposed to [x][m] so one 16-byte load gives 4 orders: kept for
      // the CTA's lifetime when it fits (items of one CTA share a pol whenever
      // gridDim is a multiple of P), else staged per item into the free zs
      const bool keep = persistent_basis(GP);
      float* hxT = keep ? reinterpret_cast<float*>(smem + LY::bytes)
                        : reinterpret_cast<float*>(smem + LY::zs + LY::basis_off);   // [WW][GP]
      float* hyT = hxT + WW * GP;                                                   // [WH][GP]
      float2* U = xbuf;                                                             // [WH][GP]
      if (!keep || q != staged_q) {
        const float* hx = p.t.hx + (size_t)q * G * WW;
        const float* hy = p.t.hy + (size_t)q * G * WH;
        for (int i = tid; i < (GP / 4) * WW; i += blockDim.x) {   // thread -> (x, 4 orders)
          const int x = i % WW, m4 = 4 * (i / WW);
          float4 h;
          h.x = m4 + 0 < G ? __ldg(&hx[(m4 + 0) * WW + x]) : 0.f;
          h.y = m4 + 1 < G ? __ldg(&hx[(m4 + 1) * WW + x]) : 0.f;
          h.z = m4 + 2 < G ? __ldg(&hx[(m4 + 2) * WW + x]) : 0.f;
          h.w = m4 + 3 < G ? __ldg(&hx[(m4 + 3) * WW + x]) : 0.f;
          *reinterpret_cast<float4*>(&hxT[x * GP + m4]) = h;
        }
        for (int i = tid; i < (GP / 4) * WH; i += blockDim.x) {
          const int y = i % WH, n4 = 4 * (i / WH);
          float4 h;
          h.x = n4 + 0 < G ? __ldg(&hy[(n4 + 0) * WH + y]) : 0.f;
          h.y = n4 + 1 < G ? __ldg(&hy[(n4 + 1) * WH + y]) : 0.f;
          h.z = n4 + 2 < G ? __ldg(&hy[(n4 + 2) * WH + y]) : 0.f;
          h.w = n4 + 3 < G ? __ldg(&hy[(n4 + 3) * WH + y]) : 0.f;
          *reinterpret_cast<float4*>(&hyT[y * GP + n4]) = h;
        }
        staged_q = keep ? q : -1;
      }
      __syncthreads();
      const int GQ = GP >> 2;
      // HG parity (ft.hsym, checked on the quantised profiles at plan time): h_m(c - d) = (-1)^m h_m(c + d)
      // around the axis origin c = W / 2, so each +-d pair of samples enters as F(c + d) +- F(c - d)
      constexpr int CX = WW / 2, NPX = WW - 1 - CX, CY = WH / 2, NPY = WH - 1 - CY;
      const bool xsym = (ft.hsym >> (2 * q)) & 1, ysym = (ft.hsym >> (2 * q + 1)) & 1;
      for (int idx = tid; idx < WH * GQ; idx += blockDim.x) {
        const int y = idx / GQ, mq = idx - y * GQ;
        const float2* row = F + y * WW;
        float4 ar = make_float4(0.f, 0.f, 0.f, 0.f), ai = ar;
        if (xsym) {   // 4 mq is even: orders 4mq, 4mq + 2 take the sums, 4mq + 1, 4mq + 3 the differences
#pragma unroll 5
          for (int dd = 1; dd <= NPX; ++dd) {
            const float2 vp = row[CX + dd], vm = row[CX - dd];
            const float2 sv = make_float2(vp.x + vm.x, vp.y + vm.y), dv = make_float2(vp.x - vm.x, vp.y - vm.y);
            const float4 h = *reinterpret_cast<const float4*>(&hxT[(CX + dd) * GP + 4 * mq]);
            ar.x = fmaf(sv.x, h.x, ar.x); ai.x = fmaf(sv.y, h.x, ai.x);
            ar.y = fmaf(dv.x, h.y, ar.y); ai.y = fmaf(dv.y, h.y, ai.y);
            ar.z = fmaf(sv.x, h.z, ar.z); ai.z = fmaf(sv.y, h.z, ai.z);
            ar.w = fmaf(dv.x, h.w, ar.w); ai.w = fmaf(dv.y, h.w, ai.w);
          }
#pragma unroll
          for (int k = 0; k < 1 + (CX - NPX); ++k) {   // the origin, and x = 0 when W is even
            const int x = k == 0 ? CX : 0;
            const float2 v = row[x];
            const float4 h = *reinterpret_cast<const float4*>(&hxT[x * GP + 4 * mq]);
            ar.x = fmaf(v.x, h.x, ar.x); ai.x = fmaf(v.y, h.x, ai.x);
            ar.y = fmaf(v.x, h.y, ar.y); ai.y = fmaf(v.y, h.y, ai.y);
            ar.z = fmaf(v.x, h.z, ar.z); ai.z = fmaf(v.y, h.z, ai.z);
            ar.w = fmaf(v.x, h.w, ar.w); ai.w = fmaf(v.y, h.w, ai.w);
          }
        } else {
#pragma unroll 6
          for (int x = 0; x < WW; ++x) {
            const float2 v = row[x];
            const float4 h = *reinterpret_cast<const float4*>(&hxT[x * GP + 4 * mq]);
            ar.x = fmaf(v.x, h.x, ar.x); ai.x = fmaf(v.y, h.x, ai.x);
            ar.y = fmaf(v.x, h.y, ar.y); ai.y = fmaf(v.y, h.y, ai.y);
            ar.z = fmaf(v.x, h.z, ar.z); ai.z = fmaf(v.y, h.z, ai.z);
            ar.w = fmaf(v.x, h.w, ar.w); ai.w = fmaf(v.y, h.w, ai.w);
          }
        }
        float2* u = U + y * GP + 4 * mq;
        u[0] = make_float2(ar.x, ai.x);
        u[1] = make_float2(ar.y, ai.y);
        u[2] = make_float2(ar.z, ai.z);
        u[3] = make_float2(ar.w, ai.w);
      }
      __syncthreads();
      const float d = __fdiv_rn(g.dxdy[q], scale);
      float2* out = p.coefs + (size_t)item * g.M;
      // two lanes per coefficient (adjacent lanes split the y pairs), combined with one shuffle
      for (int t0 = 0; t0 < 2 * g.M; t0 += blockDim.x) {
        const int tt = t0 + tid, i = tt >> 1, half = tt & 1;
        float ax = 0.f, ay = 0.f;
        if (i < g.M) {
          const int m = p.t.mode_m[i], n = p.t.mode_n[i];
          if (ysym) {
            const float sg = (n & 1) ? -1.f : 1.f;
#pragma unroll 5
            for (int dd = 1 + half; dd <= NPY; dd += 2) {
              const float2 vp = U[(CY + dd) * GP + m], vm = U[(CY - dd) * GP + m];
              const float hv = hyT[(CY + dd) * GP + n];
              ax = fmaf(fmaf(sg, vm.x, vp.x), hv, ax);
              ay = fmaf(fmaf(sg, vm.y, vp.y), hv, ay);
            }
            if (half == 0 || CY > NPY) {   // the origin (lane 0) and y = 0 when H is even (lane 1)
              const int y = half == 0 ? CY : 0;
              const float2 v = U[y * GP + m];
              const float hv = hyT[y * GP + n];
              ax = fmaf(v.x, hv, ax);
              ay = fmaf(v.y, hv, ay);
            }
          } else {
#pragma unroll 7
            for (int y = half; y < WH; y += 2) {
              const float2 v = U[y * GP + m];
              const float hv = hyT[y * GP + n];
              ax = fmaf(v.x, hv, ax);
              ay = fmaf(v.y, hv, ay);
            }
          }
        }
        ax += __shfl_xor_sync(0xffffffffu, ax, 1);
        ay += __shfl_xor_sync(0xffffffffu, ay, 1);
        if (i < g.M && half == 0) out[i] = make_float2(ax * d, ay * d);
      }
    }
  }
  if (TCO) {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if ((tid >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tco_tbase));
  }
}

bool fast_supported(const Geometry& g, int A, int fmt, int transpose, int fill, const void* rcal,
                    unsigned flags, const void* windows) {
  (void)fill;   // the fill-factor envelope is folded into the separable recentring tables
  (void)rcal;   // the reference calibration is applied in the final IFFT stage
  return g.nx == 128 && g.ny == 128 && g.wh == 42 && g.ww == 42 && g.gh == 42 && g.gw == 42 && A == 1 &&
         g.G <= FastLayout<42, 42>::GMAX && !(fmt == 1 && transpose) &&
         (flags & 1u) == 0 && windows == nullptr;
}

template <int NT>
static cudaError_t launch_fast_nt(const RunParams& p, const FastTables& ft, int num_sms, cudaStream_t s) {
  using LY = FastLayout<42, 42, NT>;
  const int GP = (p.g.G + 3) & ~3;
  const size_t bytes = LY::bytes + ((p.coefs && p.g.G > 0 && GP <= kPersistentBasisGP)
                                        ? (size_t)(42 + 42) * GP * sizeof(float) : 0);
  // tensor-core overlap pays for large bases (G > 16: config 5 G = 45 +32 %); below that its two MMA
  // round trips per item cost more than the SIMT overlap they replace (dual-pol G = 14: -10 %)
  const bool tco = NT == 256 && ft.tco_gp >= 32 && p.coefs && p.g.G > 0 && !(p.flags & kFlagNoTco);
  auto kt = fast128_kernel<42, 42, true, 256>;
  auto kf = fast128_kernel<42, 42, false, NT>;
  cudaError_t e = ensure_smem_optin((const void*)kt, bytes);
  if (e != cudaSuccess) return e;
  e = ensure_smem_optin((const void*)kf, bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  // same registers / shared memory for both variants; the occupancy API reports 1 CTA/SM for kernels that
  // allocate tensor memory, but 3 x 128 TMEM columns fit the SM's 512
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, NT, bytes);
  if (tco) per_sm = std::min(per_sm, 4);
  const int items = p.B * p.g.P;
  const int grid = std::max(1, std::min(items, num_sms * std::max(per_sm, 1)));
  if (tco)
    kt<<<grid, 256, bytes, s>>>(p, ft);
  else
    kf<<<grid, NT, bytes, s>>>(p, ft);
  return cudaGetLastError();
}

cudaError_t launch_fast(const RunParams& p, const FastTables& ft, int num_sms, cudaStream_t s) {
  // fewer windows than SMs: nothing to overlap across CTAs, so give each window the whole SM
  const char* env = getenv("HOLO_FAST_NT");   // diagnostic override, read per launch
  const int forced_nt = env ? atoi(env) : 0;
  const int items = p.B * p.g.P;
  const bool wide = forced_nt ? forced_nt == 512 : items <= num_sms;
  return wide ? launch_fast_nt<512>(p, ft, num_sms, s) : launch_fast_nt<256>(p, ft, num_sms, s);
}

}  // namespace holo
