// Field tail of the 128-window / 42 x 42 geometry: W -> 42 x 42 IFFT -> removal phase, calibrations ->
// int16 packing -> HG overlap (holopipe/pipeline.py:130-199, engine.py:234-272, hgbasis.py:101-116).
//
// One warp PAIR per window, no CTA-wide barrier: a pair owns a window buffer in shared memory and walks
// its window through every step with a 64-thread named barrier only, so the windows of an SM are
// independent and the per-step parallelism (294 / 252 small DFTs per IFFT axis) fills the 64 lanes.
//
// The 42-point inverse DFT uses the Good-Thomas prime-factor map (42 = 6 x 7, gcd 1): input n =
// (7 n1 + 6 n2) mod 42, output k = (7 k1 + 36 k2) mod 42, so
//     X[k] = sum_n2 e^{2 pi i n2 k2 / 7} sum_n1 e^{2 pi i n1 k1 / 6} x[n]
// -- a DFT-6 over n1 for each n2, then a DFT-7 over n2 for each k1, NO twiddle factors.  Both passes
// work in place (a DFT-6 writes k1 where it read n1); natural index k ends at position
// pos(k) = (7 (k mod 6) + 6 (k mod 7)) mod 42, which the epilogue reads through.
#include <algorithm>

#include "holo_internal.h"

namespace holo {

namespace {

constexpr int kN = 42;          // field side (wh = ww = 42)
constexpr int kPC = 43;         // buffer pitch (float2) of one column sequence: odd -> spread banks
constexpr int kWinPerCta = 8;   // windows in flight per CTA
constexpr int kWarpsPerWin = 2;  // one warp pair (64 lanes) per window
constexpr int kTailWarps = kWinPerCta * kWarpsPerWin;
constexpr int kLanes = 32 * kWarpsPerWin;

HOLO_DEV int pfa_pos(int k) { return (7 * (k % 6) + 6 * (k % 7)) % kN; }
HOLO_DEV int pfa_in(int a, int b) { return (7 * a + 6 * b) % kN; }   // position of (n1 | k1 = a, n2 | k2 = b)
// position of output k2 of the DFT-7 task with a = 7 k1 (a + 6 k2 < 42 + 36: one conditional subtract)
HOLO_DEV int pfa_in_fast(int a, int k2) { return a + 6 * k2 >= kN ? a + 6 * k2 - kN : a + 6 * k2; }

}  // namespace

// per-warp shared-memory layout (bytes): F / U [42][43] float2 | Fq [42][42] int16x2
struct TailLayout {
  int buf_bytes;    // max(42*43, 42*GP) float2
  int warp_bytes;   // buf + Fq, 16-byte aligned
  int basis_off;    // per-CTA basis tables [P][(42 + 42) * GP] float, after the warp regions
  int total;
};

inline TailLayout tail_layout(int G, int P) {
  TailLayout L;
  const int GP = std::max(4, (G + 3) & ~3);
  L.buf_bytes = std::max(kN * kPC, kN * GP) * 8;
  L.warp_bytes = (L.buf_bytes + kN * kN * 4 + 15) & ~15;
  L.basis_off = kWinPerCta * L.warp_bytes;
  L.total = L.basis_off + (G > 0 ? P * (kN + kN) * GP * 4 : 0);
  return L;
}

namespace {

// in-place inverse DFT-6 / DFT-7 passes over the 42 sequences of one axis.  Sequence s, element e is at
// buf[s * SS + e * ES].  Tasks touch disjoint elements, so each lane loads the inputs of TWO tasks before
// it stores anything (otherwise every task's loads wait behind the previous task's stores).
template <int SS, int ES>
HOLO_DEV void pfa_pass6(float2* buf, int lane) {
  constexpr int kTasks = kN * 7;
#pragma unroll 1
  for (int t0 = lane; t0 < kTasks; t0 += 2 * kLanes) {
    const int t1 = t0 + kLanes;
    const bool two = t1 < kTasks;
    const int s0 = t0 / 7, a0 = 6 * (t0 - 7 * s0);
    const int s1 = two ? t1 / 7 : s0, a1 = two ? 6 * (t1 - 7 * s1) : a0;
    float2* q0 = buf + s0 * SS;
    float2* q1 = buf + s1 * SS;
    int p0[6], p1[6];
#pragma unroll
    for (int n1 = 0; n1 < 6; ++n1) {   // (7 n1 + 6 n2) mod 42 with 6 n2 = a < 42
      p0[n1] = a0 + 7 * n1 >= kN ? a0 + 7 * n1 - kN : a0 + 7 * n1;
      p1[n1] = a1 + 7 * n1 >= kN ? a1 + 7 * n1 - kN : a1 + 7 * n1;
    }
    float2 v[6], w[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      v[j] = q0[p0[j] * ES];
      w[j] = q1[p1[j] * ES];
    }
    dft6<true>(v);
    dft6<true>(w);
#pragma unroll
    for (int j = 0; j < 6; ++j) q0[p0[j] * ES] = v[j];
    if (two) {
#pragma unroll
      for (int j = 0; j < 6; ++j) q1[p1[j] * ES] = w[j];
    }
  }
}

template <int SS, int ES>
HOLO_DEV void pfa_pass7(float2* buf, int lane) {
  constexpr int kTasks = kN * 6;
#pragma unroll 1
  for (int t0 = lane; t0 < kTasks; t0 += 2 * kLanes) {
    const int t1 = t0 + kLanes;
    const bool two = t1 < kTasks;
    const int s0 = t0 / 6, a0 = 7 * (t0 - 6 * s0);
    const int s1 = two ? t1 / 6 : s0, a1 = two ? 7 * (t1 - 6 * s1) : a0;
    float2* q0 = buf + s0 * SS;
    float2* q1 = buf + s1 * SS;
    int p0[7], p1[7];
#pragma unroll
    for (int n2 = 0; n2 < 7; ++n2) {   // (7 k1 + 6 n2) mod 42 with 7 k1 = a <= 35
      p0[n2] = a0 + 6 * n2 >= kN ? a0 + 6 * n2 - kN : a0 + 6 * n2;
      p1[n2] = a1 + 6 * n2 >= kN ? a1 + 6 * n2 - kN : a1 + 6 * n2;
    }
    float2 v[7], w[7];
#pragma unroll
    for (int j = 0; j < 7; ++j) {
      v[j] = q0[p0[j] * ES];
      w[j] = q1[p1[j] * ES];
    }
    dft7<true>(v);
    dft7<true>(w);
#pragma unroll
    for (int j = 0; j < 7; ++j) q0[p0[j] * ES] = v[j];
    if (two) {
#pragma unroll
      for (int j = 0; j < 7; ++j) q1[p1[j] * ES] = w[j];
    }
  }
}

}  // namespace

// win: [items][2][42 r][42 c] float: Re / Im of K1's masked Fourier window
__global__ void __launch_bounds__(kTailWarps * 32, 1)
    tail42_kernel(const __grid_constant__ RunParams p, const __grid_constant__ FastTables ft, int i0, int i1,
                  const float* __restrict__ win, TailLayout L) {
  extern __shared__ __align__(16) char smem[];
  const Geometry& g = p.g;
  const int wslot = threadIdx.x / kLanes, lane = threadIdx.x - wslot * kLanes;   // window slot, lane in the pair
  const int bar_id = 1 + wslot;
  __shared__ float red[kWinPerCta][kWarpsPerWin];
  __shared__ int s_lo[kN], s_hi[kN], s_pos[kN], s_nat[kN];   // mask row range per column; PFA position of
  for (int i = threadIdx.x; i < kN; i += blockDim.x) {          // natural index k, and its inverse
    s_lo[i] = ft.crange[2 * i];
    s_hi[i] = ft.crange[2 * i + 1];
    s_pos[i] = pfa_pos(i);
    s_nat[pfa_pos(i)] = i;
  }
  auto pair_sync = [&]() {   // 64-thread named barrier of this window (warps reconverged first: bar.sync is .aligned)
    __syncwarp();
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(kLanes) : "memory");
  };
  const int G = (p.coefs && g.G > 0) ? g.G : 0;
  const int GP = max(4, (g.G + 3) & ~3);
  float2* __restrict__ buf = reinterpret_cast<float2*>(smem + wslot * L.warp_bytes);    // [c][r] pitch 43
  uint32_t* __restrict__ fq = reinterpret_cast<uint32_t*>(smem + wslot * L.warp_bytes + L.buf_bytes);  // [y][x]
  float* basis = reinterpret_cast<float*>(smem + L.basis_off);                           // [P][x|y][GP]

  if (G > 0) {   // basis of every pol, transposed [x][m] / [y][n] (hgbasis.py:95-99 profiles)
    for (int q = 0; q < g.P; ++q) {
      const float* hx = p.t.hx + (size_t)q * g.G * kN;
      const float* hy = p.t.hy + (size_t)q * g.G * kN;
      float* bq = basis + q * 2 * kN * GP;
      for (int i = threadIdx.x; i < kN * GP; i += blockDim.x) {
        const int x = i / GP, m = i - x * GP;
        bq[i] = m < G ? __ldg(&hx[m * kN + x]) : 0.f;
        bq[kN * GP + i] = m < G ? __ldg(&hy[m * kN + x]) : 0.f;
      }
    }
  }
  __syncthreads();

  const int nw = gridDim.x * kWinPerCta;
  for (int item = i0 + blockIdx.x * kWinPerCta + wslot; item < i1; item += nw) {
    const int b = item / g.P, q = item - b * g.P;
    const int w = p.wl ? p.wl[b] : 0;
    const int pl = q * g.L + w;
    // -------------- load the masked window planes [Re | Im][r][c] -> buf[c][r]
    const float* src = win + (size_t)(item - i0) * 2 * kN * kN;
    {   // element i = lane + 64 j: (r, c) advanced incrementally (64 = 42 + 22)
      int r = lane >= kN ? 1 : 0, c = lane >= kN ? lane - kN : lane;
#pragma unroll 4
      for (int i = lane; i < kN * kN; i += kLanes) {
        buf[c * kPC + r] = make_float2(__ldg(src + i), __ldg(src + kN * kN + i));
        c += kLanes - kN;
        r += 1;
        if (c >= kN) { c -= kN; r += 1; }
      }
    }
    pair_sync();
    // ---------------------------------------- inverse DFT along r (y): 42 columns, prime-factor 6 x 7
    pfa_pass6<kPC, 1>(buf, lane);
    pair_sync();
    pfa_pass7<kPC, 1>(buf, lane);
    pair_sync();
    // ---------------------------------------------- along c (x): 42 rows (positions), then epilogue
    pfa_pass6<1, kPC>(buf, lane);
    pair_sync();
    float2 bc = make_float2(1.f, 0.f);
    if (p.bcal) bc = p.bcal[(size_t)min(q, p.cal_pols - 1) * p.cal_batch + ((p.row_offset + b) % p.cal_batch)];
    const float2* rc = p.rcal ? p.rcal + ((size_t)(w % p.rcal_count) * g.P + q) * kN * kN : nullptr;
    const float2* ex = p.t.rem_x + pl * kN;
    const float2* ey = p.t.rem_y + pl * kN;
    float lmax = 0.f;
#pragma unroll 1
    for (int t = lane; t < kN * 6; t += kLanes) {   // last pass: DFT-7 along x with the removal phase fused
      const int pr = t / 6, k1 = t - 6 * pr;    // pr: position of the row (natural y below)
      const int y = s_nat[pr];
      const int a = 7 * k1;
      int pc[7];
#pragma unroll
      for (int n2 = 0; n2 < 7; ++n2) pc[n2] = a + 6 * n2 >= kN ? a + 6 * n2 - kN : a + 6 * n2;
      float2 v[7];
#pragma unroll
      for (int n2 = 0; n2 < 7; ++n2) v[n2] = buf[pc[n2] * kPC + pr];
      dft7<true>(v);
      const float2 eyq = __ldg(&ey[y]);
#pragma unroll
      for (int k2 = 0; k2 < 7; ++k2) {
        const int x = s_nat[pfa_in_fast(a, k2)];
        float2 o = cmul(cmul(v[k2], eyq), __ldg(&ex[x]));   // same operation order as ct_stage_final_rows
        if (p.bcal) o = cmul(o, bc);
        if (rc) o = cmul(o, __ldg(&rc[y * kN + x]));   // reference calibration (engine.py:250-255)
        lmax = fmaxf(lmax, fmaxf(fabsf(o.x), fabsf(o.y)));
        v[k2] = o;
      }
#pragma unroll
      for (int k2 = 0; k2 < 7; ++k2) buf[pc[k2] * kPC + pr] = v[k2];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    if ((lane & 31) == 0) red[wslot][lane >> 5] = lmax;
    pair_sync();
    lmax = fmaxf(red[wslot][0], red[wslot][1]);
    const float scale = lmax > 0.f ? (float)(32767.0 / (double)lmax) : 1.0f;   // pipeline.py:194-198
    // ----------------------------------------------------------- int16 packing, natural [y][x]
    uint32_t* fro = reinterpret_cast<uint32_t*>(p.fr + (size_t)item * kN * kN);
    uint32_t* fio = reinterpret_cast<uint32_t*>(p.fi + (size_t)item * kN * kN);
    {   // pair i = lane + 64 j of row y, columns x, x + 1 (21 pairs per row; 64 = 3 * 21 + 1)
      int y = lane / 21, x = 2 * (lane - 21 * (lane / 21));
      for (int i = lane; i < kN * kN / 2; i += kLanes) {
        const int py = s_pos[y];
        const float2 v0 = buf[s_pos[x] * kPC + py], v1 = buf[s_pos[x + 1] * kPC + py];
        if (p.raw) {
          p.raw[(size_t)item * kN * kN + y * kN + x] = v0;
          p.raw[(size_t)item * kN * kN + y * kN + x + 1] = v1;
        }
        const int r0 = __float2int_rn(__fmul_rn(v0.x, scale)), m0 = __float2int_rn(__fmul_rn(v0.y, scale));
        const int r1 = __float2int_rn(__fmul_rn(v1.x, scale)), m1 = __float2int_rn(__fmul_rn(v1.y, scale));
        fro[i] = (uint32_t)(r0 & 0xffff) | ((uint32_t)r1 << 16);
        fio[i] = (uint32_t)(m0 & 0xffff) | ((uint32_t)m1 << 16);
        *reinterpret_cast<uint2*>(&fq[y * kN + x]) =
            make_uint2((uint32_t)(r0 & 0xffff) | ((uint32_t)m0 << 16), (uint32_t)(r1 & 0xffff) | ((uint32_t)m1 << 16));
        x += 2;   // advance by 64 pairs = 3 rows + 1 pair
        y += 3;
        if (x >= kN) { x -= kN; y += 1; }
      }
    }
    if (lane == 0) p.scale[item] = scale;
    if (G == 0) {
      pair_sync();
      continue;
    }
    pair_sync();
    // --------------------------------------------------------------------- HG overlap (SIMT)
    // U[y][m] = sum_x Fq[y][x] hx[m][x] on the integer-valued field; the dequantisation 1/scale
    // (engine.py:367-369) is applied once per coefficient.
    const float* __restrict__ hxT = basis + q * 2 * kN * GP;   // [x][GP]
    const float* __restrict__ hyT = hxT + kN * GP;              // [y][GP]
    float2* __restrict__ U = buf;                                // [y][GP]
    const int GQ = GP >> 2;
    constexpr int CX = kN / 2, NPX = kN - 1 - CX;  // parity around the axis origin x = 21
    const bool xsym = (ft.hsym >> (2 * q)) & 1, ysym = (ft.hsym >> (2 * q + 1)) & 1;
    for (int t = lane; t < kN * GQ; t += kLanes) {
      const int y = t / GQ, mq = t - y * GQ;
      const uint32_t* __restrict__ row = fq + y * kN;
      float4 ar = make_float4(0.f, 0.f, 0.f, 0.f), ai = ar;
      if (xsym) {   // h_m(c - d) = (-1)^m h_m(c + d): orders 4mq, 4mq+2 take sums, 4mq+1, 4mq+3 differences
#pragma unroll 4
        for (int dd = 1; dd <= NPX; ++dd) {
          const uint32_t a = row[CX + dd], c = row[CX - dd];
          const float ar_ = (float)(int16_t)(a & 0xffff), ai_ = (float)(int16_t)(a >> 16);
          const float cr_ = (float)(int16_t)(c & 0xffff), ci_ = (float)(int16_t)(c >> 16);
          const float sr = ar_ + cr_, si = ai_ + ci_, dr = ar_ - cr_, di = ai_ - ci_;
          const float4 h = *reinterpret_cast<const float4*>(&hxT[(CX + dd) * GP + 4 * mq]);
          ar.x = fmaf(sr, h.x, ar.x); ai.x = fmaf(si, h.x, ai.x);
          ar.y = fmaf(dr, h.y, ar.y); ai.y = fmaf(di, h.y, ai.y);
          ar.z = fmaf(sr, h.z, ar.z); ai.z = fmaf(si, h.z, ai.z);
          ar.w = fmaf(dr, h.w, ar.w); ai.w = fmaf(di, h.w, ai.w);
        }
#pragma unroll
        for (int k = 0; k < 1 + (CX - NPX); ++k) {   // the origin, and x = 0 (even width)
          const int x = k == 0 ? CX : 0;
          const uint32_t a = row[x];
          const float vr = (float)(int16_t)(a & 0xffff), vi = (float)(int16_t)(a >> 16);
          const float4 h = *reinterpret_cast<const float4*>(&hxT[x * GP + 4 * mq]);
          ar.x = fmaf(vr, h.x, ar.x); ai.x = fmaf(vi, h.x, ai.x);
          ar.y = fmaf(vr, h.y, ar.y); ai.y = fmaf(vi, h.y, ai.y);
          ar.z = fmaf(vr, h.z, ar.z); ai.z = fmaf(vi, h.z, ai.z);
          ar.w = fmaf(vr, h.w, ar.w); ai.w = fmaf(vi, h.w, ai.w);
        }
      } else {
#pragma unroll 6
        for (int x = 0; x < kN; ++x) {
          const uint32_t a = row[x];
          const float vr = (float)(int16_t)(a & 0xffff), vi = (float)(int16_t)(a >> 16);
          const float4 h = *reinterpret_cast<const float4*>(&hxT[x * GP + 4 * mq]);
          ar.x = fmaf(vr, h.x, ar.x); ai.x = fmaf(vi, h.x, ai.x);
          ar.y = fmaf(vr, h.y, ar.y); ai.y = fmaf(vi, h.y, ai.y);
          ar.z = fmaf(vr, h.z, ar.z); ai.z = fmaf(vi, h.z, ai.z);
          ar.w = fmaf(vr, h.w, ar.w); ai.w = fmaf(vi, h.w, ai.w);
        }
      }
      float2* u = U + y * GP + 4 * mq;
      u[0] = make_float2(ar.x, ai.x);
      u[1] = make_float2(ar.y, ai.y);
      u[2] = make_float2(ar.z, ai.z);
      u[3] = make_float2(ar.w, ai.w);
    }
    pair_sync();
    const float d = __fdiv_rn(g.dxdy[q], scale);
    float2* out = p.coefs + (size_t)item * g.M;
    constexpr int CY = kN / 2, NPY = kN - 1 - CY;
    for (int i = lane; i < g.M; i += kLanes) {
      const int m = p.t.mode_m[i], n = p.t.mode_n[i];
      float ax = 0.f, ay = 0.f;
      if (ysym) {
        const float sg = (n & 1) ? -1.f : 1.f;
#pragma unroll 4
        for (int dd = 1; dd <= NPY; ++dd) {
          const float2 vp = U[(CY + dd) * GP + m], vm = U[(CY - dd) * GP + m];
          const float hv = hyT[(CY + dd) * GP + n];
          ax = fmaf(fmaf(sg, vm.x, vp.x), hv, ax);
          ay = fmaf(fmaf(sg, vm.y, vp.y), hv, ay);
        }
#pragma unroll
        for (int k = 0; k < 1 + (CY - NPY); ++k) {
          const int y = k == 0 ? CY : 0;
          const float2 v = U[y * GP + m];
          const float hv = hyT[y * GP + n];
          ax = fmaf(v.x, hv, ax);
          ay = fmaf(v.y, hv, ay);
        }
      } else {
#pragma unroll 6
        for (int y = 0; y < kN; ++y) {
          const float2 v = U[y * GP + m];
          const float hv = hyT[y * GP + n];
          ax = fmaf(v.x, hv, ax);
          ay = fmaf(v.y, hv, ay);
        }
      }
      out[i] = make_float2(ax * d, ay * d);
    }
    pair_sync();
  }
}

bool tail_supported(const Geometry& g) {
  return g.wh == kN && g.ww == kN && g.gh == kN && g.gw == kN && g.G <= 48 &&
         tail_layout(g.G, g.P).total <= 227 * 1024;
}

cudaError_t launch_tail(const RunParams& p, const FastTables& ft, int num_sms, cudaStream_t s, int i0, int i1,
                        const float* win) {
  const TailLayout L = tail_layout(p.coefs ? p.g.G : 0, p.g.P);
  cudaError_t e = ensure_smem_optin((const void*)tail42_kernel, (size_t)L.total);
  if (e != cudaSuccess) return e;
  const int n = i1 - i0;
  const int grid = std::max(1, std::min((n + kTailWarps - 1) / kTailWarps, num_sms));
  tail42_kernel<<<grid, kTailWarps * 32, L.total, s>>>(p, ft, i0, i1, win, L);
  return cudaGetLastError();
}

}  // namespace holo
