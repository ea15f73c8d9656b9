// Two-kernel tensor-core path for the 128-window / 42x42 geometry (sm_100a).
//
// K1  fourier128_tc2_kernel   frames -> the four column-DFT product planes of the Fourier window
//     Both DFTs of the crop are GEMMs on the 5th-generation tensor cores:
//       row DFT     D1[c'][y] = sum_x A1[c'][x] f[y][x]       M=128 N=128 K=128   A1 const (TMEM), f (SMEM)
//                   A1 = [Re; Im] exp(-2 pi i kx_c (x - xi_x + nx/2)/nx)   (recentring folded in)
//       column DFT  D2[c'][n] = sum_y D1[c'][y] C2[n][y]      M=128 N=96  K=128   D1 (TMEM, converted to fp16
//                   hi/lo in place), C2 = [Cr; Ci] const (SMEM), C[r][y] = exp(-2 pi i ky_r (y - xi_y + ny/2)/ny)
//       lanes c' = c carry Re R, lanes 64 + c carry Im R; columns r carry Cr, 48 + r carry Ci, so D2 holds
//       Cr Rr, Ci Rr, Cr Ri, Ci Ri; the tail forms W = (Cr Rr - Ci Ri) + i (Cr Ri + Ci Rr) and masks it
//       (holopipe/pipeline.py:72-127).
//     fp32-class precision from fp16 hi/lo operand splits (3 products, fp32 accumulation) with exact
//     power-of-two scalings (per row for the row-DFT operand, per window for the column-DFT operand).
//     TMEM (512 columns): A1 hi|lo [0,128)  D1 x2 [128,384) (double-buffered)  D2 [384,480).
//     Warp roles (one CTA per SM, persistent, every CTA owns one pol):
//       warps 0-7   producers: landed window -> registers -> per-row 2^k scale -> fp16 hi/lo row-DFT operand,
//                   written one K half at a time (the row GEMM of K half 0 overlaps the conversion of half 1)
//       warp  8     MMA issuer: S1(0) | S1(k+1) S2(k) ... (the row GEMM runs one window ahead)
//       warp  9     TMA issuer: half windows into a 3-slot landing ring (two halves ahead)
//       warps 10-17 consumers: D1(k) -> fp16 hi/lo in TMEM (the column GEMM's A operand, no shared-memory
//                   round trip); D2(k) -> the product planes, coalesced stores (lanes = window columns)
// K2  tail (holo_tail.cu, or field128_kernel below): W -> 42x42 IFFT, removal phase, calibrations,
//     int16 packing, HG overlap.  W lives in the workspace between the two launches; batches are
//     processed in chunks small enough for W to stay resident in L2.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <utility>

#include "holo_fast_common.cuh"
#include "holo_internal.h"
#include "holo_tc_common.cuh"

namespace holo {

namespace {

// Warp roles.  A warp reaches the TMEM lane quarter warp % 4, and the DFT rows are packed into lanes 0..83
// (Re R of column c at lane 2c, Im R at lane 2c + 1), so the six consumer warps are the ones with
// warp % 4 < 3 among warps 0-7; warps 3 and 7 issue the MMAs and the TMA loads; warps 8-15 are the producers.
constexpr int kMmaWarp = 3;                 // tcgen05.mma issuer
constexpr int kTmaWarp = 7;                 // TMA issuer
constexpr int kProdWarp0 = 8;               // producers: warps 8-15
constexpr int kProd2 = 256;                 // producer threads
constexpr int kCons2 = 192;                 // consumer threads (warps 0-2, 4-6)
constexpr int kK1Threads = 512;
constexpr int kBarCons2 = 2, kBarSub0 = 3;   // kBarSub0 + sub: the 3 warps of one K half
constexpr int kN2 = 48;                     // column-DFT N per real part (42 rows, padded)
constexpr int kWinW = 42, kWinH = 42;
constexpr int kSlots = 3;                   // landing ring: half windows

// dynamic shared memory (bytes)
constexpr uint32_t kBox = 4096;                    // TMA box: 32 rows x 128 B (32 f32 / 64 u16), 128B swizzle
constexpr uint32_t kSlot = 8 * kBox;               // one half window: [chunk 2][box 4]
constexpr uint32_t kLand = 0;                      // [slot 3][half window]
constexpr uint32_t kStage = kSlots * kSlot;        // row-DFT operand, N = 128 rows: [hi 32 KB | lo 32 KB]
constexpr uint32_t kStageHalf = 32768;
constexpr uint32_t kC2 = kStage + 2 * kStageHalf;  // column-DFT constant [Cr; Ci]: hi | lo
constexpr uint32_t kC2Part = 8 * 3072;             // [8 ksteps][12 ngroups][2][8][16 B]
constexpr uint32_t kFac = kC2 + 2 * kC2Part;       // facrow[2][128] f32: 2^e_y of every window row
constexpr uint32_t kK1Bytes = kFac + 2 * 128 * 4;
static_assert(kK1Bytes <= 227 * 1024 - 1024, "K1 shared memory");

// canonical K-major, no-swizzle operand layout: [kstep][row/8][khalf][row%8][8 halves]
HOLO_DEV uint32_t kmaj_off(int row, int k, int ngroups) {
  return (uint32_t)(k >> 4) * (ngroups * 256) + ((uint32_t)(row >> 3) * 2 + ((k >> 3) & 1)) * 128 +
         (uint32_t)(row & 7) * 16;
}

HOLO_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// frexp exponent of a finite positive float (m = f 2^e, f in [0.5, 1)); -1000 for 0 / subnormal
HOLO_DEV int exp_of(float m) {
  const int b = (__float_as_int(m) >> 23) & 0xff;
  return b == 0 ? -1000 : b - 126;
}
HOLO_DEV float pow2f(int e) { return __int_as_float((e + 127) << 23); }   // 2^e, -126 <= e <= 127

// {a, b} -> f16x2 (a in the low half), one F2FP
HOLO_DEV uint32_t f16x2(float a, float b) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(b), "f"(a));
  return d;
}
// exact split of two floats into fp16 hi + lo: hi keeps the top 11 significant bits (exact in fp16 for
// |v| in the fp16 normal range, which the power-of-two scalings guarantee for every significant value),
// lo = v - hi is exact in fp32 and rounded once to fp16 (22 significant bits in hi + lo)
HOLO_DEV void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const float ha = __uint_as_float(__float_as_uint(a) & 0xffffe000u);
  const float hb = __uint_as_float(__float_as_uint(b) & 0xffffe000u);
  hi = f16x2(ha, hb);
  lo = f16x2(a - ha, b - hb);
}
// The same split of (a, b) * (sa, sb) with the packed fp32 instructions of sm_100 (FMUL2 / FADD2: two lanes per
// issued instruction, same results): 6 instructions per pair instead of 8.  The kernel is issue-bound on
// exactly these splits.
HOLO_DEV void split2_scaled(float a, float b, float sa, float sb, uint32_t& hi, uint32_t& lo) {
  unsigned long long v, sc, vs, h, l;
  asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(a), "f"(b));
  asm("mov.b64 %0, {%1, %2};" : "=l"(sc) : "f"(sa), "f"(sb));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(vs) : "l"(v), "l"(sc));
  h = vs & 0xffffe000ffffe000ull;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(l) : "l"(vs), "l"(h));
  float ha, hb, la, lb;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(ha), "=f"(hb) : "l"(h));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(la), "=f"(lb) : "l"(l));
  hi = f16x2(ha, hb);
  lo = f16x2(la, lb);
}

}  // namespace

// Phase timestamps of CTA 0 (clock64), for tools/tc2_trace.py (hpg_debug_trace).
__device__ long long g_tc2_trace[4][64][8];
__device__ long long g_tc2_span[160][4];   // per CTA: globaltimer start / end (ns), clock64 start / end
HOLO_DEV long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TC2_MARK(role, kk, ev)                                                   \
  do {                                                                           \
    if (blockIdx.x == 0 && (kk) < 64) g_tc2_trace[role][kk][ev] = clock64();     \
  } while (0)

// TMA (tensor map over the frame buffer [F][H][W]) of half h of an item's window into landing slot
// `slot`: two 32-row chunks x 4 boxes of 128 bytes per row, issued by one thread.
template <int FMT>
HOLO_DEV void issue_half(const RunParams& p, const CUtensorMap* tmap, int item, int h, char* smem, int slot,
                         uint64_t* bar) {
  const Geometry& g = p.g;
  const int b = item / g.P, q = item - b * g.P;
  constexpr int bw = FMT == 0 ? 32 : 64;   // box width in elements (128 bytes)
  const int nbox = 128 / bw;
  mbar_expect_tx(bar, 2u * nbox * kBox);
#pragma unroll 1
  for (int jj = 0; jj < 2; ++jj) {
    const int j = 2 * h + jj;
    for (int qx = 0; qx < nbox; ++qx) {
      const uint32_t dst = smem_u32(smem + kLand + slot * kSlot + (jj * 4 + qx) * kBox);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(tmap)), "r"(g.col0[q] + qx * bw), "r"(g.row0[q] + 32 * j), "r"(b),
          "r"(smem_u32(bar))
          : "memory");
    }
  }
}

// wout: [items][2][42 r][42 c] float, relative to item i0: Re W and Im W of the masked Fourier window
template <int FMT>
__global__ void __launch_bounds__(kK1Threads, 1)
    fourier128_tc2_kernel(const __grid_constant__ RunParams p, const __grid_constant__ FastTables ft,
                          const __grid_constant__ CUtensorMap tmap, int i0, int i1, float* __restrict__ wout) {
  extern __shared__ __align__(1024) char smem[];
  // landfull/landfree[slot]: TMA ring; staged[h]: K half h of the stage written; stfree[h]: row GEMM done with
  // K half h of the stage; meta[s]: row scales of slot s published; facfree[s]: slot s consumed; d1full[b]: row GEMM into D1 buffer b done;
  // a2ready[b][h]: K half h of the converted D1 buffer b ready; d1free[b]: column GEMM done with D1 buffer b;
  // d2full: column GEMM done; d2free: D2 drained
  __shared__ __align__(8) uint64_t landfull[kSlots], landfree[kSlots], staged[2], stfree[2], meta[2], facfree[2],
      d1full[2], a2ready[2][2], d1free[2], d2full, d2free, c2full, a1ready;
  __shared__ uint32_t tbase;
  __shared__ int emaxw[2][8];   // per window slot: largest row exponent seen by each producer warp
  float* facrow = reinterpret_cast<float*>(smem + kFac);
  const Geometry& g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int first = i0 + blockIdx.x;
  const int nk = first < i1 ? (i1 - first + gridDim.x - 1) / gridDim.x : 0;   // windows of this CTA
  const int q = first % g.P;   // gridDim.x and i0 are multiples of P: one pol per CTA

  if (tid == 0 && blockIdx.x < 160) {
    g_tc2_span[blockIdx.x][0] = gtimer();
    g_tc2_span[blockIdx.x][2] = clock64();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&landfull[i], 1);
      mbar_init(&landfree[i], kProd2 / 32);   // one arrival per producer warp
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&staged[i], kProd2 / 32);     // K half i written: one arrival per producer warp
      mbar_init(&stfree[i], 1);
      mbar_init(&meta[i], kProd2 / 32);       // row scales published: one arrival per producer warp
      mbar_init(&facfree[i], 1);
      mbar_init(&d1full[i], 1);
      mbar_init(&a2ready[i][0], 1);
      mbar_init(&a2ready[i][1], 1);
      mbar_init(&d1free[i], 1);
    }
    mbar_init(&d2full, 1);
    mbar_init(&c2full, 1);
    mbar_init(&a1ready, 12);   // one arrival per warp that loads a chunk of the row-DFT constant
    mbar_init(&d2free, kCons2 / 32);   // D2 copied to registers: one arrival per consumer warp
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  tc_fence_before();
  __syncthreads();   // barriers initialised, TMEM base published
  tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t tA1 = tm, tD2 = tm + 384;
  auto tD1 = [&](int k) { return tm + 128 + 128 * (uint32_t)(k & 1); };
  const int pre = min(kSlots, 2 * nk);   // the first frame loads fly while the constant tables are set up
  if (warp == kTmaWarp && nk > 0 && elect_one()) {
    for (int jh = 0; jh < pre; ++jh)
      issue_half<FMT>(p, &tmap, first + (jh >> 1) * gridDim.x, jh & 1, smem, jh, &landfull[jh]);
    // the column-DFT constant of this CTA's pol: one 48 KB bulk copy into shared memory
    mbar_expect_tx(&c2full, 2 * kC2Part);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem + kC2)),
                 "l"(ft.c2_tc + (size_t)q * (2 * kC2Part / 16)), "r"(2 * kC2Part), "r"(smem_u32(&c2full))
                 : "memory");
  }
  if ((warp & 3) != 3 && nk > 0) {
    // row-DFT constant of this CTA's pol into TMEM lanes 0..95 (column-major table: coalesced): 12 warps,
    // one 32-column chunk each (lanes 96..127 carry no DFT row and are never read back)
    const int quarter = warp & 3, chunk = warp >> 2;
    const int part = chunk >> 1, hh = chunk & 1;
    const uint32_t* s2 = ft.a_tcp + (size_t)q * 2 * 64 * 128 + quarter * 32 + lane + ((size_t)part * 64 + hh * 32) * 128;
    uint32_t r[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = __ldg(s2 + j * 128);
    tmem_st32(tA1 + ((uint32_t)(quarter * 32) << 16) + part * 64 + hh * 32, r);
    tmem_wait_st();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&a1ready);   // no CTA-wide barrier: the producers start on the first window at once
  }
  asm volatile("griddepcontrol.launch_dependents;");   // the tail's CTAs may take over SMs as this grid's CTAs exit

  if (warp >= kProdWarp0) {
    // ================================= producers =================================
    // Phase A: both halves of the window into registers (row max -> exact power-of-two row scale), landing
    // slots released at once.  Phase B: the row-DFT operand is written one K half (64 samples of every row)
    // at a time, so the row GEMM of K half 0 runs while K half 1 is converted and the stage halves are
    // refilled for the next window while the other half's MMAs run.
    const int r8 = lane & 7, gq = lane >> 3;   // row within the warp's 8, octet group
    const int pw = warp - kProdWarp0;
    const bool mark = tid == kProdWarp0 * 32;
    for (int k = 0; k < nk; ++k) {
      const int s = k & 1;
      int emax_t = -1000;
      float v[2][32];   // rows y = 64 h + 8 pw + r8; octets o = gq + 4 i, i = 0..3
      float sc[2];
      if (mark) TC2_MARK(0, k, 0);
      if (k >= 2) mbar_wait_warp(&facfree[s], ((k >> 1) - 1) & 1);   // conversion of window k-2 done with slot s
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jh = 2 * k + h, slot = jh % kSlots;
        mbar_wait_warp(&landfull[slot], (jh / kSlots) & 1);
        if (mark) TC2_MARK(0, k, 1 + h);
        const int yl = 8 * pw + r8, y = 64 * h + yl;
        const int jj = yl >> 5, rb = y & 31;   // chunk within the half, row in box
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int o = gq + 4 * i;
          if (FMT == 0) {   // f32: box qx = o / 4, 16-byte chunks 2(o%4), 2(o%4)+1, swizzled by row
            const char* box = smem + kLand + slot * kSlot + (jj * 4 + (o >> 2)) * kBox + rb * 128;
            const int c0 = (2 * (o & 3)) ^ (rb & 7), c1 = (2 * (o & 3) + 1) ^ (rb & 7);
            const float4 a = *reinterpret_cast<const float4*>(box + c0 * 16);
            const float4 c = *reinterpret_cast<const float4*>(box + c1 * 16);
            v[h][8 * i + 0] = a.x; v[h][8 * i + 1] = a.y; v[h][8 * i + 2] = a.z; v[h][8 * i + 3] = a.w;
            v[h][8 * i + 4] = c.x; v[h][8 * i + 5] = c.y; v[h][8 * i + 6] = c.z; v[h][8 * i + 7] = c.w;
          } else {            // u16: box qx = o / 8, one 16-byte chunk o%8
            const char* box = smem + kLand + slot * kSlot + (jj * 4 + (o >> 3)) * kBox + rb * 128;
            const uint4 a = *reinterpret_cast<const uint4*>(box + (((o & 7) ^ (rb & 7)) * 16));
            const uint32_t w4[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[h][8 * i + 2 * e] = (float)(w4[e] & 0xffffu);
              v[h][8 * i + 2 * e + 1] = (float)(w4[e] >> 16);
            }
          }
        }
        float m = 0.f;
#pragma unroll
        for (int e = 0; e < 32; ++e) m = fmaxf(m, fabsf(v[h][e]));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
        if (lane == 0) mbar_arrive(&landfree[slot]);   // this warp's rows are in registers (8 arrivals free the slot)
        // exact power-of-two row scale: |f| * sc < 2^14, fh + fl keep 22 bits
        const int ey = exp_of(m);
        sc[h] = ey > -1000 ? pow2f(14 - ey) : 1.f;
        if (gq == 0) facrow[s * 128 + y] = ey > -1000 ? pow2f(ey) : 0.f;   // undone after the row GEMM
        emax_t = max(emax_t, ey);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) emax_t = max(emax_t, __shfl_xor_sync(0xffffffffu, emax_t, o));
      __syncwarp();   // the warp's row scales are written
      if (lane == 0) {
        emaxw[s][pw] = emax_t;
        mbar_arrive(&meta[s]);
      }
      char* st = smem + kStage;   // one K-major N = 128 operand: hi [0, 32 KB), lo [32 KB, 64 KB)
#pragma unroll
      for (int kh = 0; kh < 2; ++kh) {   // K half kh = samples 64 kh .. 64 kh + 63 = octets 8 kh .. 8 kh + 7
        if (k >= 1) mbar_wait_warp(&stfree[kh], (k - 1) & 1);   // row GEMM of k-1 done with this K half
        if (mark) TC2_MARK(0, k, 3 + 2 * kh);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int y = 64 * h + 8 * pw + r8;
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            const int i = 2 * kh + ii;
            const uint32_t off = kmaj_off(y, 8 * (gq + 4 * i), 16);
            uint32_t hi2[4], lo2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              split2_scaled(v[h][8 * i + 2 * e], v[h][8 * i + 2 * e + 1], sc[h], sc[h], hi2[e], lo2[e]);
            *reinterpret_cast<uint4*>(st + off) = make_uint4(hi2[0], hi2[1], hi2[2], hi2[3]);
            *reinterpret_cast<uint4*>(st + 32768 + off) = make_uint4(lo2[0], lo2[1], lo2[2], lo2[3]);
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&staged[kh]);   // 8 arrivals: K half written by every producer warp
        if (mark) TC2_MARK(0, k, 4 + 2 * kh);
      }
    }
  } else if (warp == kTmaWarp) {
    // ================================ TMA issuer ================================
    for (int jh = pre; jh < 2 * nk; ++jh) {   // the whole warp walks the ring (converged), lane 0 issues
      const int slot = jh % kSlots;
      mbar_wait_warp(&landfree[slot], ((jh / kSlots) - 1) & 1);
      if (elect_one()) issue_half<FMT>(p, &tmap, first + (jh >> 1) * gridDim.x, jh & 1, smem, slot, &landfull[slot]);
      __syncwarp();
    }
  } else if (warp == kMmaWarp) {
    // ================================ MMA issuer ================================
    const uint32_t idesc2 = idesc_f16(128, 2 * kN2);
    const uint32_t idesc1 = idesc_f16(128, 128);
    auto row_gemm = [&](int k) {   // D1(k) = A1 * stage, N = 128: 12 MMAs per K half as the halves are staged
      // D1 buffer k & 1 was last read by the column GEMM of window k-2: tcgen05.mma instructions of one thread
      // execute in issue order, so the overwrite needs no barrier
#pragma unroll 1
      for (int kh = 0; kh < 2; ++kh) {
        mbar_wait_warp(&staged[kh], k & 1);
        if (lane == 0 && kh == 0) TC2_MARK(2, k, 0);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sb = smem_u32(smem + kStage), d = tD1(k);
#pragma unroll
          for (int gk = 4 * kh; gk < 4 * kh + 4; ++gk) {
            const uint64_t bh = umma_desc(sb + gk * 4096, 128, 256);
            const uint64_t bl = umma_desc(sb + 32768 + gk * 4096, 128, 256);
            mma_f16_ts(d, tA1 + gk * 8, bh, idesc1, gk != 0);
            mma_f16_ts(d, tA1 + 64 + gk * 8, bh, idesc1, 1);
            mma_f16_ts(d, tA1 + gk * 8, bl, idesc1, 1);
          }
          tc_commit(&stfree[kh]);   // the producers may refill this K half while the other half's MMAs run
          if (kh == 1) {
            tc_commit(&d1full[k & 1]);
            TC2_MARK(2, k, 1);
          }
        }
        __syncwarp();
      }
    };
    auto col_gemm = [&](int k, int h) {   // D2 (+)= D1(k)[:, K half h] (fp16 hi/lo in TMEM) * C2, N = 96
      // per D1 buffer: the consumer may convert window k + 1 before this wait, never window k + 2
      mbar_wait_warp(&a2ready[k & 1][h], (k >> 1) & 1);
      if (h == 0 && k >= 1) mbar_wait_warp(&d2free, (k - 1) & 1);
      if (lane == 0) TC2_MARK(2, k, 4 + 2 * h);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sb = smem_u32(smem + kC2), a = tD1(k);
#pragma unroll
        for (int ks = 4 * h; ks < 4 * h + 4; ++ks) {   // K-step ks: hi at column 32 (ks/2) + 8 (ks%2), lo +16
          const uint32_t ah = a + 32 * (ks >> 1) + 8 * (ks & 1), al = ah + 16;
          const uint64_t bh = umma_desc(sb + ks * 3072, 128, 256), bl = umma_desc(sb + kC2Part + ks * 3072, 128, 256);
          mma_f16_ts(tD2, ah, bh, idesc2, ks != 0);
          mma_f16_ts(tD2, al, bh, idesc2, 1);
          mma_f16_ts(tD2, ah, bl, idesc2, 1);
        }
        if (h == 1) {
          tc_commit(&d2full);
          tc_commit(&d1free[k & 1]);
        }
        TC2_MARK(2, k, 5 + 2 * h);
      }
      __syncwarp();
    };
    if (nk > 0) {
      mbar_wait_warp(&a1ready, 0);   // the row-DFT constant is in TMEM
      tc_fence_after();
      row_gemm(0);
    }
    if (nk > 0) mbar_wait_warp(&c2full, 0);   // the column-DFT constant has landed
    for (int k = 0; k < nk; ++k) {
      if (k + 1 < nk) row_gemm(k + 1);
      col_gemm(k, 0);
      col_gemm(k, 1);
    }
  } else {
    // ================================= consumers =================================
    const int ct = tid, quarter = warp & 3, sub = warp >> 2;   // warps 0-2 (sub 0), 4-6 (sub 1)
    const int ci = sub * 96 + quarter * 32 + lane;             // consumer thread index 0..191
    const uint32_t lanebase = (uint32_t)(quarter * 32) << 16;
    const int n = quarter * 32 + lane;   // D1 / D2 lane: Re R (even n) / Im R (odd n) of column n / 2, n < 84
    const bool im = n & 1, used = n < 2 * kWinW;
    const int c = n >> 1;
    float gsv[2] = {1.f, 1.f};   // output scale of the windows in flight, read while the slot's scales are ours
    auto convert = [&](int k) {
      // ---- D1(k) -> fp16 hi/lo in place (this warp: K half `sub`, two 32-column chunks)
      mbar_wait_warp(&meta[k & 1], (k >> 1) & 1);
      int em = emaxw[k & 1][0];
#pragma unroll
      for (int j = 1; j < 8; ++j) em = max(em, emaxw[k & 1][j]);
      // column-operand scale per row: D1 * 2^(e_y - e_max - 6) = R * 2^(8 - e_max) < 2^15
      const float gdn = pow2f(max(-126, min(127, -em - 6)));
      gsv[k & 1] = pow2f(max(-126, min(127, em - 8)));
      if (ci < 128) facrow[(k & 1) * 128 + ci] *= gdn;   // one multiply per row instead of one per element
      nbar(kBarCons2, kCons2);
      mbar_wait_warp(&d1full[k & 1], (k >> 1) & 1);
      tc_fence_after();
      if (ct == 0) TC2_MARK(1, k, 0);
      const float* fs = facrow + (k & 1) * 128;
#pragma unroll 1
      for (int j = 0; j < 2; ++j) {
        const int y0 = 64 * sub + 32 * j;
        const uint32_t col = tD1(k) + lanebase + y0;
        uint32_t r[32];
        tmem_ld32(col, r);
        tmem_wait_ld();
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float4 f4 = *reinterpret_cast<const float4*>(fs + y0 + 4 * e);
          split2_scaled(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]), f4.x, f4.y, hi[2 * e], lo[2 * e]);
          split2_scaled(__uint_as_float(r[4 * e + 2]), __uint_as_float(r[4 * e + 3]), f4.z, f4.w, hi[2 * e + 1],
                        lo[2 * e + 1]);
        }
        tmem_st16(col, hi);
        tmem_st16(col + 16, lo);
      }
      tmem_wait_st();
      tc_fence_before();
      nbar(kBarSub0 + sub, 96);
      if (ct == 0) TC2_MARK(1, k, 1);
      if (quarter == 0 && lane == 0) mbar_arrive(&a2ready[k & 1][sub]);   // one arrival per K half
      nbar(kBarCons2, kCons2);   // both halves converted: the slot's scales were read by every consumer
      if (ct == 0) mbar_arrive(&facfree[k & 1]);
    };
    const int mlo = used ? ft.crange[2 * c] : 1, mhi = used ? ft.crange[2 * c + 1] : 0;
    auto drain = [&](int k) {
      // ---- D2(k) -> W = (Cr Rr - Ci Ri) + i (Cr Ri + Ci Rr).  D2 columns r hold Cr R, columns 48 + r hold
      // Ci R of the lane's R part; the Re / Im lanes of a column are neighbours, so the cross term comes by one
      // shuffle.  This warp handles the 24 rows r = 24 sub .. 24 sub + 23; masked (pipeline.py:72-76) stores.
      const float gs = gsv[k & 1];
      mbar_wait_warp(&d2full, k & 1);
      tc_fence_after();
      if (ct == 0) TC2_MARK(1, k, 5);
      uint32_t a[24], b[24];
      tmem_ld16(tD2 + lanebase + 24 * sub, a);
      tmem_ld8(tD2 + lanebase + 24 * sub + 16, a + 16);
      tmem_ld16(tD2 + lanebase + kN2 + 24 * sub, b);
      tmem_ld8(tD2 + lanebase + kN2 + 24 * sub + 16, b + 16);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&d2free);   // D2 is in registers (6 arrivals): the next column GEMM may start
      const float sg = im ? gs : -gs;        // Im: + Ci Rr (from the Re lane); Re: - Ci Ri (from the Im lane)
      float* wo = wout + ((size_t)(first + k * gridDim.x - i0) * 2 + (im ? 1 : 0)) * (kWinH * kWinW) + c;
#pragma unroll
      for (int j = 0; j < 24; ++j) {
        const int rr = 24 * sub + j;
        const float other = __uint_as_float(__shfl_xor_sync(0xffffffffu, b[j], 1));
        const float val = fmaf(other, sg, __uint_as_float(a[j]) * gs);
        if (used && rr < kWinH) wo[rr * kWinW] = (rr >= mlo && rr <= mhi) ? val : 0.f;
      }
      if (ct == 0) TC2_MARK(1, k, 6);
    };
    // D1 is double-buffered: convert window k + 1 while the column GEMM of window k runs, then drain D2(k)
    if (nk > 0) convert(0);
    for (int k = 0; k < nk; ++k) {
      if (k + 1 < nk) convert(k + 1);
      drain(k);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  if (tid == 0 && blockIdx.x < 160) {
    g_tc2_span[blockIdx.x][1] = gtimer();
    g_tc2_span[blockIdx.x][3] = clock64();
  }
}

// ---------------------------------------------------------------------------
// K2: window -> field -> int16 -> coefficients (SIMT, 3+ CTAs per SM)
template <int WH, int WW>
struct FieldLayout {
  static constexpr size_t T = 0;                                            // IFFT ping
  static constexpr size_t F = T + WH * WW * sizeof(float2);                  // IFFT pong / field
  static constexpr size_t U = F + WH * WW * sizeof(float2);                  // overlap partials [WH][GP]
  static constexpr int GMAX = 48;
  static constexpr size_t twh = U + WH * GMAX * sizeof(float2);
  static constexpr size_t tww = twh + WH * sizeof(float2);
  static constexpr size_t ph = tww + WW * sizeof(float2);                    // ex[WW] ey[WH]
  static constexpr size_t basis = (ph + (WH + WW) * sizeof(float2) + 15) & ~size_t(15);
};

template <int WH, int WW>
__global__ void __launch_bounds__(256, 3)
    field128_kernel(const __grid_constant__ RunParams p, int i0, int i1, const float* __restrict__ win,
                    const int16_t* __restrict__ crange) {
  using LY = FieldLayout<WH, WW>;
  extern __shared__ __align__(1024) char smem[];
  __shared__ float redf[8];
  float2* T = reinterpret_cast<float2*>(smem + LY::T);
  float2* F = reinterpret_cast<float2*>(smem + LY::F);
  float2* U = reinterpret_cast<float2*>(smem + LY::U);
  float2* twh = reinterpret_cast<float2*>(smem + LY::twh);
  float2* tww = reinterpret_cast<float2*>(smem + LY::tww);
  float2* s_ex = reinterpret_cast<float2*>(smem + LY::ph);
  float2* s_ey = s_ex + WW;
  float* hxP = reinterpret_cast<float*>(smem + LY::basis);
  const Geometry& g = p.g;
  const int tid = threadIdx.x;
  const int G = g.G, GP = (G + 3) & ~3;
  for (int i = tid; i < WH; i += blockDim.x) twh[i] = p.t.tw_gh[i];
  for (int i = tid; i < WW; i += blockDim.x) tww[i] = p.t.tw_gw[i];
  int staged_q = -1;
  for (int item = i0 + blockIdx.x; item < i1; item += gridDim.x) {
    const int b = item / g.P, q = item - b * g.P;
    __syncthreads();   // previous item done with every buffer
    for (int i = tid; i < WW; i += blockDim.x) s_ex[i] = p.t.rem_x[q * g.L * WW + i];
    for (int i = tid; i < WH; i += blockDim.x) s_ey[i] = p.t.rem_y[q * g.L * WH + i];
    if (p.coefs && G > 0 && q != staged_q) {   // basis of this pol, transposed [x][m] / [y][n]
      const float* hx = p.t.hx + (size_t)q * G * WW;
      const float* hy = p.t.hy + (size_t)q * G * WH;
      for (int i = tid; i < (GP / 4) * WW; i += blockDim.x) {
        const int x = i % WW, m4 = 4 * (i / WW);
        float4 h;
        h.x = m4 + 0 < G ? __ldg(&hx[(m4 + 0) * WW + x]) : 0.f;
        h.y = m4 + 1 < G ? __ldg(&hx[(m4 + 1) * WW + x]) : 0.f;
        h.z = m4 + 2 < G ? __ldg(&hx[(m4 + 2) * WW + x]) : 0.f;
        h.w = m4 + 3 < G ? __ldg(&hx[(m4 + 3) * WW + x]) : 0.f;
        *reinterpret_cast<float4*>(&hxP[x * GP + m4]) = h;
      }
      for (int i = tid; i < (GP / 4) * WH; i += blockDim.x) {
        const int y = i % WH, n4 = 4 * (i / WH);
        float4 h;
        h.x = n4 + 0 < G ? __ldg(&hy[(n4 + 0) * WH + y]) : 0.f;
        h.y = n4 + 1 < G ? __ldg(&hy[(n4 + 1) * WH + y]) : 0.f;
        h.z = n4 + 2 < G ? __ldg(&hy[(n4 + 2) * WH + y]) : 0.f;
        h.w = n4 + 3 < G ? __ldg(&hy[(n4 + 3) * WH + y]) : 0.f;
        *reinterpret_cast<float4*>(&hxP[(WW + y) * GP + n4]) = h;
      }
      staged_q = q;
    }
    __syncthreads();
    const float* Wp = win + (size_t)(item - i0) * 2 * WH * WW;   // masked window planes [Re | Im][r][c]
    for (int i = tid; i < WH * WW; i += blockDim.x) {            // -> F, column-major [c][r]
      const int r = i / WW, c = i - r * WW;
      F[c * WH + r] = make_float2(__ldg(Wp + i), __ldg(Wp + WH * WW + i));
    }
    __syncthreads();
    // IFFT along r (y) first, then along c (x)
    ct_stage<6, WH, 1, WW, WH, 1, true>(F, T, twh);
    __syncthreads();
    ct_stage<7, WH, 6, WW, WH, 1, true>(T, F, twh);
    __syncthreads();
    ct_stage<6, WW, 1, WH, 1, WH, true>(F, T, tww);
    __syncthreads();
    float2 bc = make_float2(1.f, 0.f);
    if (p.bcal) bc = p.bcal[(size_t)min(q, p.cal_pols - 1) * p.cal_batch + ((p.row_offset + b) % p.cal_batch)];
    float lmax = ct_stage_final_rows<7, WW, 6, WH>(T, F, tww, s_ey, s_ex, p.bcal != nullptr, bc);
#pragma unroll
    for (int o = 16; o; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    if ((tid & 31) == 0) redf[tid >> 5] = lmax;
    __syncthreads();
    lmax = redf[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) lmax = fmaxf(lmax, redf[j]);
    if (p.raw)
      for (int i = tid; i < WH * WW; i += blockDim.x) p.raw[(size_t)item * WH * WW + i] = F[i];
    const float scale = lmax > 0.f ? (float)(32767.0 / (double)lmax) : 1.0f;
    int16_t* fro = p.fr + (size_t)item * WH * WW;
    int16_t* fio = p.fi + (size_t)item * WH * WW;
    for (int i = tid; i < WH * WW / 2; i += blockDim.x) {
      const float4 v = reinterpret_cast<const float4*>(F)[i];
      const int r0 = __float2int_rn(__fmul_rn(v.x, scale)), im0 = __float2int_rn(__fmul_rn(v.y, scale));
      const int r1 = __float2int_rn(__fmul_rn(v.z, scale)), im1 = __float2int_rn(__fmul_rn(v.w, scale));
      reinterpret_cast<int*>(fro)[i] = (r0 & 0xffff) | (r1 << 16);
      reinterpret_cast<int*>(fio)[i] = (im0 & 0xffff) | (im1 << 16);
      reinterpret_cast<float4*>(F)[i] = make_float4((float)r0, (float)im0, (float)r1, (float)im1);
    }
    if (tid == 0) p.scale[item] = scale;
    if (p.coefs && G > 0) {
      const float* hxT = hxP;
      const float* hyT = hxP + WW * GP;
      __syncthreads();
      const int GQ = GP >> 2;
      for (int idx = tid; idx < WH * GQ; idx += blockDim.x) {
        const int y = idx / GQ, mq = idx - y * GQ;
        const float2* row = F + y * WW;
        float4 ar = make_float4(0.f, 0.f, 0.f, 0.f), ai = ar;
#pragma unroll 6
        for (int x = 0; x < WW; ++x) {
          const float2 v = row[x];
          const float4 h = *reinterpret_cast<const float4*>(&hxT[x * GP + 4 * mq]);
          ar.x = fmaf(v.x, h.x, ar.x); ai.x = fmaf(v.y, h.x, ai.x);
          ar.y = fmaf(v.x, h.y, ar.y); ai.y = fmaf(v.y, h.y, ai.y);
          ar.z = fmaf(v.x, h.z, ar.z); ai.z = fmaf(v.y, h.z, ai.z);
          ar.w = fmaf(v.x, h.w, ar.w); ai.w = fmaf(v.y, h.w, ai.w);
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
      for (int i = tid; i < g.M; i += blockDim.x) {
        const int m = p.t.mode_m[i], n = p.t.mode_n[i];
        float ax = 0.f, ay = 0.f;
#pragma unroll 6
        for (int y = 0; y < WH; ++y) {
          const float2 v = U[y * GP + m];
          const float hv = hyT[y * GP + n];
          ax = fmaf(v.x, hv, ax);
          ay = fmaf(v.y, hv, ay);
        }
        out[i] = make_float2(ax * d, ay * d);
      }
    }
  }
}

extern "C" int hpg_debug_span(long long* out) {   // copies g_tc2_span (160*4 int64) to host
  return cudaMemcpyFromSymbol(out, g_tc2_span, sizeof(g_tc2_span)) == cudaSuccess ? 0 : 1;
}

extern "C" int hpg_debug_trace(long long* out) {   // copies g_tc2_trace (2*64*8 int64) to host
  return cudaMemcpyFromSymbol(out, g_tc2_trace, sizeof(g_tc2_trace)) == cudaSuccess ? 0 : 1;
}

bool tail_supported(const Geometry& g);
cudaError_t launch_tail(const RunParams& p, const FastTables& ft, int num_sms, cudaStream_t s, int i0, int i1,
                        const float* win);
bool tailr_supported(const Geometry& g, const void* rcal);
cudaError_t launch_tailr(const RunParams& p, const FastTables& ft, cudaStream_t s, int i0, int i1, const float* win);

constexpr int kTc2Chunk = 2048;   // items per K1/K2 pair: the product planes (28 KB each) stay in L2

bool tc2_supported(const Geometry& g, int A, int fmt, int transpose, int fill, const void* rcal, unsigned flags,
                   const void* windows) {
  (void)fill;   // the fill-factor envelope is folded into the DFT matrices (ensure_tc_tables)
  (void)rcal;   // the reference calibration (one wavelength here) is applied by the tail with the removal phase
  const int es = fmt == 1 ? 2 : 4;
  const bool aligned = (g.W * es) % 16 == 0;   // TMA tensor map: 16-byte row stride
  return g.nx == 128 && g.ny == 128 && g.wh == 42 && g.ww == 42 && g.gh == 42 && g.gw == 42 && A == 1 &&
         g.L == 1 && g.G <= FieldLayout<42, 42>::GMAX && !(fmt == 1 && transpose) &&
         (flags & 1u) == 0 && windows == nullptr && aligned;
}

int64_t tc2_chunk() { return kTc2Chunk; }

size_t tc2_workspace(int64_t items) {
  return (size_t)std::min<int64_t>(items, kTc2Chunk) * 2 * 42 * 42 * sizeof(float);   // Re W, Im W
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Tensor map over the frame buffer [B][H][W] (f32 or u16), 32-row x 128-byte boxes, 128B swizzle.
static cudaError_t frame_tensor_map(const RunParams& p, CUtensorMap* map) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const cuuint64_t es = p.fmt == 0 ? 4 : 2;
  const cuuint64_t dims[3] = {(cuuint64_t)p.g.W, (cuuint64_t)p.g.H, (cuuint64_t)std::max(p.B, 1)};
  const cuuint64_t strides[2] = {(cuuint64_t)p.g.W * es, (cuuint64_t)p.g.W * p.g.H * es};
  const cuuint32_t box[3] = {(cuuint32_t)(128 / es), 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const char* env = getenv("HOLO_TMA_PROMO");   // diagnostic: 0 none, 1 64 B, 2 128 B (default: measured best), 3 256 B
  const CUtensorMapL2promotion promo = !env ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                       : env[0] == '0' ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                       : env[0] == '1' ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                       : env[0] == '2' ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                       : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = encode(map, p.fmt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3,
                      const_cast<void*>(p.frames), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, promo,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_tc2(const RunParams& p, const FastTables& ft, int num_sms, cudaStream_t s) {
  using LY = FieldLayout<42, 42>;
  const int GP = (p.g.G + 3) & ~3;
  const size_t k2_bytes = LY::basis + (size_t)(42 + 42) * std::max(GP, 4) * sizeof(float);
  int k2_per_sm = 1;
  for (const auto& kb : {std::make_pair((const void*)fourier128_tc2_kernel<0>, (size_t)kK1Bytes),
                         std::make_pair((const void*)fourier128_tc2_kernel<1>, (size_t)kK1Bytes),
                         std::make_pair((const void*)field128_kernel<42, 42>, LY::basis + 84 * 48 * sizeof(float))}) {
    const cudaError_t e = ensure_smem_optin(kb.first, kb.second);
    if (e != cudaSuccess) return e;
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k2_per_sm, field128_kernel<42, 42>, 256, k2_bytes);
  float* wbuf = reinterpret_cast<float*>(p.work);
  CUtensorMap tmap;
  cudaError_t te = frame_tensor_map(p, &tmap);
  if (te != cudaSuccess) return te;
  const int items = p.B * p.g.P;
  for (int i0 = 0; i0 < items; i0 += kTc2Chunk) {
    const int i1 = std::min(items, i0 + kTc2Chunk);
    const int n = i1 - i0;
    // one pol per CTA: the grid (and every chunk start) is a multiple of P
    const int g1 = std::max(1, std::min(n, num_sms) / p.g.P * p.g.P);
    if (p.fmt == 0)
      fourier128_tc2_kernel<0><<<g1, kK1Threads, kK1Bytes, s>>>(p, ft, tmap, i0, i1, wbuf);
    else
      fourier128_tc2_kernel<1><<<g1, kK1Threads, kK1Bytes, s>>>(p, ft, tmap, i0, i1, wbuf);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // diagnostic: HOLO_TAIL=0 runs the round-1 CTA-wide tail, HOLO_TAIL=2 the warp-pair tail
    const char* env = getenv("HOLO_TAIL");
    if (tailr_supported(p.g, p.rcal) && !(env && (env[0] == '0' || env[0] == '2'))) {
      e = launch_tailr(p, ft, s, i0, i1, wbuf);
    } else if (tail_supported(p.g) && !(env && env[0] == '0')) {
      e = launch_tail(p, ft, num_sms, s, i0, i1, wbuf);
    } else {
      field128_kernel<42, 42><<<std::max(1, std::min(n, num_sms * std::max(k2_per_sm, 1))), 256, k2_bytes, s>>>(
          p, i0, i1, wbuf, ft.crange);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace holo
