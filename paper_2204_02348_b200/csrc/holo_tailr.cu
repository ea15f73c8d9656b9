// Register-resident field tail of the 128-window / 42 x 42 geometry (two-kernel tensor-core path):
// product planes -> masked W -> 42 x 42 inverse DFT -> removal phase, batch calibration -> int16 packing
// -> HG overlap (holopipe/pipeline.py:72-76,130-199, engine.py:234-272, hgbasis.py:101-116).
//
// One THREAD per 42-point sequence: a thread holds a whole column (then a whole row) of the window in
// registers and runs the prime-factor 42 = 6 x 7 inverse DFT on it with every index a compile-time
// constant -- no twiddles, no index arithmetic and no shared-memory traffic inside a transform.  Three
// windows of one pol share a 128-thread CTA (3 x 42 = 126 lanes busy), four CTAs per SM:
//
//   phase 1  the three windows (Re / Im planes, 14 KB each) land in shared memory by cp.async.bulk; thread
//            (window, column c) reads its column (lanes = consecutive c), IDFT-42 along y, transposed store
//            T[y][c] over the landing area (pitch 43: conflict-free both ways)
//   phase 2  thread (window, row y): loads T[y][:], IDFT-42 along x, removal phase and calibration, peak
//            (warp reduction + one shared atomic per warp segment), int16 rounding; the row of integers
//            stays in registers for the first overlap contraction U[m][y] = sum_x F[y][x] hx[m][x]
//            (HG parity folds x = 21 +- d), written to shared memory
//   phase 3  CTA-wide: coalesced int16 plane stores from the staged words; second contraction
//            c[m, n] = sum_y U[m][y] hy[n][y], one (window, mode) per thread.
#include <algorithm>
#include <cstdlib>

#include "holo_internal.h"
#include "holo_tc_common.cuh"

namespace holo {

namespace {

constexpr int kN = 42;        // field side (wh = ww = gh = gw = 42)
constexpr int kP = 43;        // shared-memory pitch (elements) of a 42-sequence
constexpr int kWin = 3;       // windows per CTA
constexpr int kThr = 128;     // threads per CTA (126 active in phases 1-2)

// Good-Thomas map of 42 = 6 x 7: input n = (7 n1 + 6 n2) mod 42; the DFT-6 over n1 and the DFT-7 over n2
// run in place, and natural output index k ends at position (7 (k mod 6) + 6 (k mod 7)) mod 42.
__host__ __device__ constexpr int pos_of(int k) { return (7 * (k % 6) + 6 * (k % 7)) % kN; }

// in-place inverse/forward DFT-6 as 2 x 3 prime-factor (no twiddles): n1 = (3a + 2b) mod 6, k1 = (3c + 4d) mod 6
template <bool INV> HOLO_DEV void dft6p(float2* x) {
  float2 s0 = cadd(x[0], x[3]), d0 = csub(x[0], x[3]);
  float2 s1 = cadd(x[2], x[5]), d1 = csub(x[2], x[5]);
  float2 s2 = cadd(x[4], x[1]), d2 = csub(x[4], x[1]);
  dft3<INV>(s0, s1, s2);
  dft3<INV>(d0, d1, d2);
  x[0] = s0; x[4] = s1; x[2] = s2;
  x[3] = d0; x[1] = d1; x[5] = d2;
}

template <bool INV> HOLO_DEV void dft42(float2 (&v)[kN]) {
#pragma unroll
  for (int n2 = 0; n2 < 7; ++n2) {
    float2 t[6];
#pragma unroll
    for (int n1 = 0; n1 < 6; ++n1) t[n1] = v[(7 * n1 + 6 * n2) % kN];
    dft6p<INV>(t);
#pragma unroll
    for (int k1 = 0; k1 < 6; ++k1) v[(7 * k1 + 6 * n2) % kN] = t[k1];
  }
#pragma unroll
  for (int k1 = 0; k1 < 6; ++k1) {
    float2 t[7];
#pragma unroll
    for (int n2 = 0; n2 < 7; ++n2) t[n2] = v[(7 * k1 + 6 * n2) % kN];
    dft7<INV>(t);
#pragma unroll
    for (int k2 = 0; k2 < 7; ++k2) v[(7 * k1 + 6 * k2) % kN] = t[k2];
  }
}

}  // namespace

// per-CTA shared memory: [window 3][T (42 x 43 float2) | later Fq (42 x 43 words) + U (GP x 43 float2)]
// | ex[42] ey[42] | hxT[42][GP] hyT[42][GP]
struct TailRLayout {
  int win_bytes, ph_off, basis_off, total;
};

inline TailRLayout tailr_layout(int G) {
  TailRLayout L;
  const int GP = std::max(4, (G + 3) & ~3);
  L.win_bytes = (std::max(kN * kP * 8, kN * kP * 4 + (G > 0 ? GP * kP * 8 : 0)) + 15) & ~15;
  L.ph_off = kWin * L.win_bytes;
  L.basis_off = L.ph_off + 2 * kN * 8;
  L.total = L.basis_off + (G > 0 ? 2 * kN * GP * 4 : 0);
  return L;
}

// Small symmetric bases (G <= 16, HG parity on both axes: every batch the two-kernel path is chosen for): only
// x = 0 and x >= 21 of the transposed profiles are needed, 22 rows x 16 orders = 1.4 KB per axis -- small enough
// for the spare 1.7 KB behind Fq + U in a window's region.  With no basis region of its own the CTA needs
// 44 KB of shared memory and five fit an SM: the whole 2,000-window batch is resident in a single wave.
// (Round 2 first passed these tables as a kernel parameter so that the FMAs took them as constant operands;
// the constant loads of 20 warps walking a 5.4 KB table thrashed the constant cache -- the first contraction
// took 17 K of the CTA's 53 K cycles, tools/tail_trace.py.)
constexpr int kPG = 16;                        // padded order count of the half tables
constexpr int kHalfRows = kN / 2 + 1;          // row 0: x = 0; row 1 + d: x = 21 + d, d = 0..20
constexpr int kHalfOff = (kN * kP * 4 + kPG * kP * 8 + 15) & ~15;   // behind Fq + U
static_assert(kHalfOff + kHalfRows * kPG * 4 <= kN * kP * 8, "the half table must fit the window region");

namespace {

// U[m][y = s] = sum_x F[y][x] hx[m][x] for an x-symmetric basis; v holds the folded row (v[pos(21 + d)] =
// F(21 + d) + F(21 - d), v[pos(21 - d)] = the difference, d = 1..20; x = 21 and x = 0 plain); hxh: half table.
// Two orders (one even, one odd) per pass: four accumulators and one 8-byte basis load live next to the row.
HOLO_DEV void overlap_x_half(const float* __restrict__ hxh, const float2 (&v)[kN], float2* U, int s, int G) {
  constexpr int CX = kN / 2;
#pragma unroll 1
  for (int mp = 0; 2 * mp < G; ++mp) {   // the zero-padded orders beyond G are never read back
    const float* hq = hxh + 2 * mp;
    const float2 h1 = *reinterpret_cast<const float2*>(hq), h0 = *reinterpret_cast<const float2*>(hq + kPG);
    float2 ae = make_float2(fmaf(v[pos_of(0)].x, h1.x, v[pos_of(CX)].x * h0.x),
                            fmaf(v[pos_of(0)].y, h1.x, v[pos_of(CX)].y * h0.x));
    float2 ao = make_float2(fmaf(v[pos_of(0)].x, h1.y, v[pos_of(CX)].x * h0.y),
                            fmaf(v[pos_of(0)].y, h1.y, v[pos_of(CX)].y * h0.y));
#pragma unroll
    for (int d = 1; d < CX; ++d) {
      const float2 h = *reinterpret_cast<const float2*>(hq + (1 + d) * kPG);
      const float2 sv = v[pos_of(CX + d)], dv = v[pos_of(CX - d)];   // even order: sums, odd order: differences
      ae.x = fmaf(sv.x, h.x, ae.x);
      ae.y = fmaf(sv.y, h.x, ae.y);
      ao.x = fmaf(dv.x, h.y, ao.x);
      ao.y = fmaf(dv.y, h.y, ao.y);
    }
    U[(2 * mp) * kP + s] = ae;
    U[(2 * mp + 1) * kP + s] = ao;
  }
}

// c[m, n] = sum_y U[m][y] hy[n][y] for every n of one (window, m), y-symmetric basis; hyh: half table
HOLO_DEV void overlap_y_half(const float* __restrict__ hyh, const float2* Um, int m, int G, float d, float2* out) {
  constexpr int CY = kN / 2;
  float ax[kPG], ay[kPG];
  {
    const float2 u0 = Um[CY], u1 = Um[0];
#pragma unroll
    for (int n4 = 0; n4 < kPG / 4; ++n4) {
      const float4 a1 = *reinterpret_cast<const float4*>(hyh + 4 * n4);
      const float4 a0 = *reinterpret_cast<const float4*>(hyh + kPG + 4 * n4);
      const float h1v[4] = {a1.x, a1.y, a1.z, a1.w}, h0v[4] = {a0.x, a0.y, a0.z, a0.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        ax[4 * n4 + j] = fmaf(u1.x, h1v[j], u0.x * h0v[j]);
        ay[4 * n4 + j] = fmaf(u1.y, h1v[j], u0.y * h0v[j]);
      }
    }
  }
#pragma unroll 4
  for (int dd = 1; dd < CY; ++dd) {
    const float2 vp = Um[CY + dd], vm = Um[CY - dd];
    const float2 se = cadd(vp, vm), so = csub(vp, vm);
#pragma unroll
    for (int n4 = 0; n4 < kPG / 4; ++n4) {
      const float4 h4 = *reinterpret_cast<const float4*>(hyh + (1 + dd) * kPG + 4 * n4);
      const float hv[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = 4 * n4 + j;
        ax[n] = fmaf((n & 1) ? so.x : se.x, hv[j], ax[n]);
        ay[n] = fmaf((n & 1) ? so.y : se.y, hv[j], ay[n]);
      }
    }
  }
#pragma unroll
  for (int n = 0; n < kPG; ++n) {
    const int gg = m + n;   // group-major mode index (hgbasis.py:17-27)
    if (gg < G) out[gg * (gg + 1) / 2 + n] = make_float2(ax[n] * d, ay[n] * d);
  }
}

}  // namespace

// win: [items][2][42 r][42 c] float, relative to item i0: Re / Im of K1's masked Fourier window
// (holopipe/pipeline.py:72-127).  CTA (pol q, task): the three windows
// i0 + q + P (3 task + {0, 1, 2}) (i0 is a multiple of P).
// Phase timestamps of two CTAs (clock64) for tools/tail_trace.py; compiled in with -DHOLO_TAIL_TRACE only.
#ifdef HOLO_TAIL_TRACE
__device__ long long g_tail_trace[2][16];
#define TAIL_MARK(i) do { if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2)) g_tail_trace[blockIdx.x ? 1 : 0][i] = clock64(); } while (0)
#else
#define TAIL_MARK(i) do { } while (0)
#endif

template <bool PB>
HOLO_DEV void tail_body(const RunParams& p, const FastTables& ft, int i0, int i1, const float* __restrict__ win,
                        const TailRLayout& L) {
  TAIL_MARK(0);
  extern __shared__ __align__(16) char smem[];
  __shared__ int s_max[kWin];
  __shared__ float s_scale[kWin];
  const Geometry& g = p.g;
  const int P = g.P;
  const int q = blockIdx.x % P, task = blockIdx.x / P;
  const int tid = threadIdx.x;
  const bool lane_on = tid < kWin * kN;
  const int w3 = lane_on ? tid / kN : kWin - 1, s = lane_on ? tid - w3 * kN : 0;
  const int item = i0 + q + P * (task * kWin + w3);
  const bool valid = lane_on && item < i1;
  if (i0 + q + P * (task * kWin) >= i1) return;   // no window for this CTA (uniform)

  const int G = (p.coefs && g.G > 0) ? g.G : 0;
  const int GP = max(4, (g.G + 3) & ~3);
  float2* sex = reinterpret_cast<float2*>(smem + L.ph_off);
  float2* sey = sex + kN;
  float* hxT = reinterpret_cast<float*>(smem + L.basis_off);   // [x][GP]
  float* hyT = hxT + kN * GP;                                  // [y][GP]
  for (int i = tid; i < kN; i += kThr) {   // removal phase of this pol (one wavelength on this path)
    sex[i] = p.t.rem_x[q * g.L * kN + i];
    sey[i] = p.t.rem_y[q * g.L * kN + i];
  }
  if (!PB && G > 0) {   // basis of this pol, transposed [x][m] / [y][n] (hgbasis.py:95-99 profiles)
    const float* hx = p.t.hx + (size_t)q * g.G * kN;
    const float* hy = p.t.hy + (size_t)q * g.G * kN;
    for (int i = tid; i < kN * GP; i += kThr) {
      const int x = i / GP, m = i - x * GP;
      hxT[i] = m < G ? __ldg(&hx[m * kN + x]) : 0.f;
      hyT[i] = m < G ? __ldg(&hy[m * kN + x]) : 0.f;
    }
  }
  if (tid < kWin) s_max[tid] = 0;

  // ------------------------------------------------------------------ phase 1: column c = s
  // the window planes [Re | Im][42 r][42 c] (14,112 contiguous bytes per window) arrive by bulk copy
  __shared__ __align__(8) uint64_t landed;
  if (tid == 0) {
    mbar_init(&landed, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  constexpr uint32_t kWinBytes = 2 * kN * kN * 4;
  if (tid == 0) {
    // programmatic dependent launch: everything above overlapped the end of the Fourier kernel; its window
    // buffer is complete (and visible) once the whole primary grid has finished
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int nv = 0;
    for (int w = 0; w < kWin; ++w) nv += (i0 + q + P * (task * kWin + w)) < i1;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&landed)), "r"(nv * kWinBytes)
                 : "memory");
    for (int w = 0; w < nv; ++w) {
      const float* src = win + (size_t)(i0 + q + P * (task * kWin + w) - i0) * 2 * kN * kN;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem + w * L.win_bytes)),
          "l"(src), "r"(kWinBytes), "r"(smem_u32(&landed))
          : "memory");
    }
  }
  float2 v[kN];
  TAIL_MARK(1);
  mbar_wait(&landed, 0);
  TAIL_MARK(2);
  {
    const float* wp = reinterpret_cast<const float*>(smem + w3 * L.win_bytes) + s;
#pragma unroll
    for (int r = 0; r < kN; ++r)
      v[r] = valid ? make_float2(wp[r * kN], wp[kN * kN + r * kN]) : make_float2(0.f, 0.f);
  }
  __syncthreads();   // every column is in registers: the landing area becomes T
  TAIL_MARK(3);
  dft42<true>(v);   // along y (holopipe/pipeline.py:130-149)
  TAIL_MARK(4);
  float2* T = reinterpret_cast<float2*>(smem + w3 * L.win_bytes);   // [y][kP]
  if (lane_on) {
#pragma unroll
    for (int k = 0; k < kN; ++k) T[k * kP + s] = v[pos_of(k)];
  }
  __syncthreads();

  // ------------------------------------------------------------------ phase 2: row y = s
  if (lane_on) {
#pragma unroll
    for (int c = 0; c < kN; ++c) v[c] = T[s * kP + c];
  }
  TAIL_MARK(6);
  dft42<true>(v);   // along x; F[y][x] is v[pos_of(x)]
  TAIL_MARK(7);
  const int b = valid ? item / P : 0;
  float2 bc = make_float2(1.f, 0.f);
  if (p.bcal) bc = p.bcal[(size_t)min(q, p.cal_pols - 1) * p.cal_batch + ((p.row_offset + b) % p.cal_batch)];
  const float2* rc = p.rcal ? p.rcal + (size_t)q * kN * kN : nullptr;
  float lmax = 0.f;
  {
    const float2 eyq = sey[s];
    if (!p.bcal && !rc) {   // the common case without its 8 predicated-off multiplies and a load per sample
#pragma unroll
      for (int x = 0; x < kN; ++x) {
        const float2 o = cmul(cmul(v[pos_of(x)], eyq), sex[x]);   // same operation order as ct_stage_final_rows
        lmax = fmaxf(lmax, fmaxf(fabsf(o.x), fabsf(o.y)));
        v[pos_of(x)] = o;
      }
    } else {
#pragma unroll
      for (int x = 0; x < kN; ++x) {
        float2 o = cmul(cmul(v[pos_of(x)], eyq), sex[x]);
        if (p.bcal) o = cmul(o, bc);
        if (rc) o = cmul(o, __ldg(&rc[s * kN + x]));   // reference calibration (engine.py:250-255)
        lmax = fmaxf(lmax, fmaxf(fabsf(o.x), fabsf(o.y)));
        v[pos_of(x)] = o;
      }
    }
  }
  {   // peak of each window: lanes of one warp belong to at most two windows
    const unsigned seg = __match_any_sync(0xffffffffu, lane_on ? w3 : kWin);
    const int mx = __reduce_max_sync(seg, __float_as_int(lmax));   // lmax >= 0: integer order = float order
    if (lane_on && (tid & 31) == __ffs(seg) - 1) atomicMax(&s_max[w3], mx);
  }
  TAIL_MARK(8);
  __syncthreads();   // every T row has been read: the window's region is free for Fq / U
  TAIL_MARK(9);
  float* hxh = reinterpret_cast<float*>(smem + kHalfOff);                 // spare space of window 0's region
  float* hyh = reinterpret_cast<float*>(smem + L.win_bytes + kHalfOff);   // ... of window 1's region
  if (PB && G > 0 && tid == 0) {   // the two half tables of this pol by bulk copy behind the int16 rounding
    constexpr uint32_t kHalfBytes = kHalfRows * kPG * 4;
    const float* src = ft.half_tab + (size_t)q * 2 * kHalfRows * kPG;
    fence_async_smem();   // the regions were last touched through the generic proxy (T)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&landed)), "r"(2 * kHalfBytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(hxh)),
                 "l"(src), "r"(kHalfBytes), "r"(smem_u32(&landed))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(hyh)),
                 "l"(src + kHalfRows * kPG), "r"(kHalfBytes), "r"(smem_u32(&landed))
                 : "memory");
  }
  lmax = __int_as_float(s_max[w3]);
  const float scale = lmax > 0.f ? (float)(32767.0 / (double)lmax) : 1.0f;   // pipeline.py:194-198
  if (valid && p.raw) {
#pragma unroll
    for (int x = 0; x < kN; ++x) p.raw[(size_t)item * kN * kN + s * kN + x] = v[pos_of(x)];
  }
  uint32_t* fq = reinterpret_cast<uint32_t*>(smem + w3 * L.win_bytes);                   // [y][kP] re | im << 16
  float2* U = reinterpret_cast<float2*>(smem + w3 * L.win_bytes + kN * kP * 4);           // [m][kP]
  if (lane_on) {
#pragma unroll
    for (int x = 0; x < kN; ++x) {
      const int r = __float2int_rn(__fmul_rn(v[pos_of(x)].x, scale));
      const int m = __float2int_rn(__fmul_rn(v[pos_of(x)].y, scale));
      fq[s * kP + x] = (uint32_t)(r & 0xffff) | ((uint32_t)m << 16);
      v[pos_of(x)] = make_float2((float)r, (float)m);   // integer-valued field for the overlap
    }
    if (s == 0) s_scale[w3] = scale;
  }
  if (valid && s == 0) p.scale[item] = scale;

  // ------------------------------------------- first overlap contraction, from registers (row y = s)
  if (PB && G > 0) mbar_wait(&landed, 1);   // the half tables have landed (second phase of the barrier)
  if (G > 0 && lane_on) {
    constexpr int CX = kN / 2;   // axis origin x = 21: x = 21 +- d for d = 1..20, plus x = 21 and x = 0
    const bool xsym = (ft.hsym >> (2 * q)) & 1;
    const int GQ = GP >> 2;
    if (xsym) {   // h_m(c - d) = (-1)^m h_m(c + d): even orders see F(c + d) + F(c - d), odd orders the difference
#pragma unroll
      for (int d = 1; d < CX; ++d) {
        const float2 a = v[pos_of(CX + d)], c = v[pos_of(CX - d)];
        v[pos_of(CX + d)] = cadd(a, c);
        v[pos_of(CX - d)] = csub(a, c);
      }
    }
    if constexpr (PB) {   // launched only for symmetric bases of at most kPG orders
      TAIL_MARK(10);
      overlap_x_half(hxh, v, U, s, G);
      TAIL_MARK(11);
    } else if (xsym) {
#pragma unroll 1
      for (int mq = 0; mq < GQ; ++mq) {
        const float* hq = hxT + 4 * mq;
        float4 ar, ai;
        {
          const float4 h0 = *reinterpret_cast<const float4*>(hq + CX * GP);
          const float4 h1 = *reinterpret_cast<const float4*>(hq);
          const float2 a = v[pos_of(CX)], c = v[pos_of(0)];
          ar = make_float4(fmaf(c.x, h1.x, a.x * h0.x), fmaf(c.x, h1.y, a.x * h0.y), fmaf(c.x, h1.z, a.x * h0.z),
                           fmaf(c.x, h1.w, a.x * h0.w));
          ai = make_float4(fmaf(c.y, h1.x, a.y * h0.x), fmaf(c.y, h1.y, a.y * h0.y), fmaf(c.y, h1.z, a.y * h0.z),
                           fmaf(c.y, h1.w, a.y * h0.w));
        }
#pragma unroll
        for (int d = 1; d < CX; ++d) {
          const float4 h = *reinterpret_cast<const float4*>(hq + (CX + d) * GP);
          const float2 sv = v[pos_of(CX + d)], dv = v[pos_of(CX - d)];
          ar.x = fmaf(sv.x, h.x, ar.x); ai.x = fmaf(sv.y, h.x, ai.x);
          ar.y = fmaf(dv.x, h.y, ar.y); ai.y = fmaf(dv.y, h.y, ai.y);
          ar.z = fmaf(sv.x, h.z, ar.z); ai.z = fmaf(sv.y, h.z, ai.z);
          ar.w = fmaf(dv.x, h.w, ar.w); ai.w = fmaf(dv.y, h.w, ai.w);
        }
        U[(4 * mq + 0) * kP + s] = make_float2(ar.x, ai.x);
        U[(4 * mq + 1) * kP + s] = make_float2(ar.y, ai.y);
        U[(4 * mq + 2) * kP + s] = make_float2(ar.z, ai.z);
        U[(4 * mq + 3) * kP + s] = make_float2(ar.w, ai.w);
      }
    } else {
#pragma unroll 1
      for (int mq = 0; mq < GQ; ++mq) {
        const float* hq = hxT + 4 * mq;
        float4 ar = make_float4(0.f, 0.f, 0.f, 0.f), ai = ar;
#pragma unroll
        for (int x = 0; x < kN; ++x) {
          const float4 h = *reinterpret_cast<const float4*>(hq + x * GP);
          const float2 a = v[pos_of(x)];
          ar.x = fmaf(a.x, h.x, ar.x); ai.x = fmaf(a.y, h.x, ai.x);
          ar.y = fmaf(a.x, h.y, ar.y); ai.y = fmaf(a.y, h.y, ai.y);
          ar.z = fmaf(a.x, h.z, ar.z); ai.z = fmaf(a.y, h.z, ai.z);
          ar.w = fmaf(a.x, h.w, ar.w); ai.w = fmaf(a.y, h.w, ai.w);
        }
        U[(4 * mq + 0) * kP + s] = make_float2(ar.x, ai.x);
        U[(4 * mq + 1) * kP + s] = make_float2(ar.y, ai.y);
        U[(4 * mq + 2) * kP + s] = make_float2(ar.z, ai.z);
        U[(4 * mq + 3) * kP + s] = make_float2(ar.w, ai.w);
      }
    }
  }
  __syncthreads();

  // ------------------------------------------------------------------ phase 3 (CTA-wide)
  TAIL_MARK(12);
  const int item0 = i0 + q + P * (task * kWin);
  // parameter-basis variant: threads 0..47 = (window, m) run the second contraction while the other 80 store
  constexpr int kYThr = PB ? kWin * kPG : 0;
  if (PB && tid < kYThr) {
    const int w = tid / kPG, m = tid - w * kPG;
    const int it = item0 + P * w;
    if (G > 0 && it < i1 && m < G) {
      const float2* Um = reinterpret_cast<const float2*>(smem + w * L.win_bytes + kN * kP * 4) + m * kP;
      const float d = __fdiv_rn(g.dxdy[q], s_scale[w]);
      float2* out = p.coefs + (size_t)it * g.M;
      if constexpr (PB) overlap_y_half(hyh, Um, m, G, d, out);
    }
    TAIL_MARK(13);
    return;
  }
#pragma unroll 1
  for (int w = 0; w < kWin; ++w) {   // int16 planes, natural [y][x], coalesced (pipeline.py:188-199)
    const int it = item0 + P * w;
    if (it >= i1) break;
    const uint32_t* fw = reinterpret_cast<const uint32_t*>(smem + w * L.win_bytes);
    uint32_t* fro = reinterpret_cast<uint32_t*>(p.fr + (size_t)it * kN * kN);
    uint32_t* fio = reinterpret_cast<uint32_t*>(p.fi + (size_t)it * kN * kN);
    for (int i = tid - kYThr; i < kN * kN / 2; i += kThr - kYThr) {
      const int y = i / (kN / 2), xp = i - y * (kN / 2);
      const uint32_t a = fw[y * kP + 2 * xp], c = fw[y * kP + 2 * xp + 1];
      fro[i] = __byte_perm(a, c, 0x5410);
      fio[i] = __byte_perm(a, c, 0x7632);
    }
  }
  if (!PB && G > 0) {   // second contraction; the dequantisation 1/scale (engine.py:367-369) once per coefficient
    const bool ysym = (ft.hsym >> (2 * q + 1)) & 1;
    constexpr int CY = kN / 2;
    const int M = g.M;
    for (int t = tid; t < kWin * M; t += kThr) {
      const int w = t / M, i = t - w * M;
      const int it = item0 + P * w;
      if (it >= i1) break;
      const int m = p.t.mode_m[i], n = p.t.mode_n[i];
      const float2* Um = reinterpret_cast<const float2*>(smem + w * L.win_bytes + kN * kP * 4) + m * kP;
      const float* hn = hyT + n;
      float ax, ay;
      if (ysym) {
        const float sg = (n & 1) ? -1.f : 1.f;
        const float2 u0 = Um[CY], u1 = Um[0];
        const float h0 = hn[CY * GP], h1 = hn[0];
        ax = fmaf(u1.x, h1, u0.x * h0);
        ay = fmaf(u1.y, h1, u0.y * h0);
#pragma unroll 5
        for (int d = 1; d < CY; ++d) {
          const float2 vp = Um[CY + d], vm = Um[CY - d];
          const float hv = hn[(CY + d) * GP];
          ax = fmaf(fmaf(sg, vm.x, vp.x), hv, ax);
          ay = fmaf(fmaf(sg, vm.y, vp.y), hv, ay);
        }
      } else {
        ax = 0.f;
        ay = 0.f;
#pragma unroll 6
        for (int y = 0; y < kN; ++y) {
          const float2 u = Um[y];
          const float hv = hn[y * GP];
          ax = fmaf(u.x, hv, ax);
          ay = fmaf(u.y, hv, ay);
        }
      }
      const float d = __fdiv_rn(g.dxdy[q], s_scale[w]);
      p.coefs[(size_t)it * M + i] = make_float2(ax * d, ay * d);
    }
  }
}

#ifdef HOLO_TAIL_TRACE
extern "C" int hpg_debug_tail_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, g_tail_trace, sizeof(g_tail_trace)) == cudaSuccess ? 0 : 1;
}
#endif

__global__ void __launch_bounds__(kThr, 4)
    tail42r_kernel(const __grid_constant__ RunParams p, const __grid_constant__ FastTables ft, int i0, int i1,
                   const float* __restrict__ win, TailRLayout L) {
  tail_body<false>(p, ft, i0, i1, win, L);
}

// half-table variant: symmetric bases of at most kPG orders, five CTAs per SM
__global__ void __launch_bounds__(kThr, 5)
    tail42p_kernel(const __grid_constant__ RunParams p, const __grid_constant__ FastTables ft, int i0, int i1,
                   const float* __restrict__ win, TailRLayout L) {
  tail_body<true>(p, ft, i0, i1, win, L);
}

bool tailr_supported(const Geometry& g, const void* rcal) {
  (void)rcal;   // applied with the removal phase (one wavelength: table q of the calibration)
  return g.wh == kN && g.ww == kN && g.gh == kN && g.gw == kN && g.G <= 48 && g.L == 1 && g.P <= kMaxPol &&
         tailr_layout(g.G).total <= 110 * 1024;
}

cudaError_t launch_tailr(const RunParams& p, const FastTables& ft, cudaStream_t s, int i0, int i1, const float* win) {
  const int G = p.coefs ? p.g.G : 0;
  const int n = i1 - i0, P = p.g.P;
  const int per_pol = (n + P - 1) / P;
  const int grid = std::max(1, P * ((per_pol + kWin - 1) / kWin));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThr);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see griddepcontrol.wait in the kernel
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool all_sym = (ft.hsym & ((1 << (2 * P)) - 1)) == (1 << (2 * P)) - 1;
  const char* env = getenv("HOLO_TAILR_SMEM_BASIS");   // diagnostic: keep the full shared-memory basis variant
  if (G > 0 && G <= kPG && all_sym && ft.half_tab && !(env && env[0] == '1')) {
    TailRLayout L = tailr_layout(0);   // no basis region: the half tables live behind Fq + U of windows 0 and 1
    cudaError_t e = ensure_smem_optin((const void*)tail42p_kernel, (size_t)L.total);
    if (e != cudaSuccess) return e;
    cfg.dynamicSmemBytes = (size_t)L.total;
    return cudaLaunchKernelEx(&cfg, tail42p_kernel, p, ft, i0, i1, win, L);
  }
  const TailRLayout L = tailr_layout(G);
  cudaError_t e = ensure_smem_optin((const void*)tail42r_kernel, (size_t)L.total);
  if (e != cudaSuccess) return e;
  cfg.dynamicSmemBytes = (size_t)L.total;
  return cudaLaunchKernelEx(&cfg, tail42r_kernel, p, ft, i0, i1, win, L);
}

}  // namespace holo
