// Generic fused hot-path kernel: frame -> window -> R2C -> Fourier-window crop
// -> reduced IFFT -> tilt/defocus removal -> field summary -> int16 -> HG overlap.
//
// One persistent CTA processes one (batch row, polarisation) item at a time.
// The reference does this as four numpy stages with full-size intermediates
// (holopipe/engine.py:135-385); here every intermediate stays on chip (or in
// an L2-resident per-CTA slab for windows too large for shared memory) and
// only the frame window is read from HBM and only int16 fields, scales and
// coefficients are written.
//
// FFT strategy (pruned 2-D R2C):
//   row pass   : rows y and y+ny/2 packed as one complex sequence, Stockham
//                FFT along x, Hermitian split, keep only the ww needed bins
//                (holopipe/pipeline.py:79-104 fetches them from the r2c plane)
//   column pass: FFT along y of the ww kept columns, keep the wh needed rows,
//                multiply by mask * recentring phase (pipeline.py:72-76,114-127)
//   IFFT       : wh x ww inverse (pipeline.py:130-149), ifftshift folded into
//                the separable removal phase (pipeline.py:163-185)
#include <algorithm>
#include <mutex>

#include "holo_internal.h"

namespace holo {

__device__ __forceinline__ float2* region_ptr(const Region& r, char* smem, char* slab) {
  return reinterpret_cast<float2*>(r.in_smem ? smem + r.off : slab + r.off);
}

__device__ __forceinline__ int pmod(int v, int n) {
  int r = v % n;
  return r < 0 ? r + n : r;
}

__device__ __forceinline__ float load_px(const void* frames, int fmt, int transpose, int W, int H,
                                         int64_t f, int y, int x) {
  const int64_t base = f * (int64_t)W * H;
  if (fmt == 0) return __ldg(reinterpret_cast<const float*>(frames) + base + (int64_t)y * W + x);
  const unsigned short* u = reinterpret_cast<const unsigned short*>(frames);
  if (transpose) return (float)__ldg(u + base + (int64_t)x * H + y);
  return (float)__ldg(u + base + (int64_t)y * W + x);
}

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum of NV doubles (same order every call).
template <int NV>
__device__ void block_sum(double* v, double (*red)[32]) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (l == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[i][w] = v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double s = 0.0;
    for (int j = 0; j < nw; ++j) s += red[i][j];
    v[i] = s;
  }
}

// Block max of v with the smallest index among ties (numpy argmax semantics).
__device__ void block_argmax(float& v, int& idx, float* redf, int* redi) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
  __syncthreads();
  if (l == 0) { redf[w] = v; redi[w] = idx; }
  __syncthreads();
  v = redf[0]; idx = redi[0];
  for (int j = 1; j < nw; ++j)
    if (redf[j] > v || (redf[j] == v && redi[j] < idx)) { v = redf[j]; idx = redi[j]; }
}

__device__ float block_max(float v, float* redf) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (l == 0) redf[w] = v;
  __syncthreads();
  v = redf[0];
  for (int j = 1; j < nw; ++j) v = fmaxf(v, redf[j]);
  return v;
}

__device__ __forceinline__ FFTPlan make_plan(int n, int nst, const int* radix, const float2* tw) {
  FFTPlan p;
  p.n = n;
  p.nst = nst;
#pragma unroll
  for (int i = 0; i < 8; ++i) p.radix[i] = radix[i];
  p.tw = tw;
  return p;
}

// ---------------------------------------------------------------- row pass
// Window rows (y, y+ny/2) -> complex sequence; FFT along x; Hermitian split;
// keep bins kx_c = k0x + c - ww/2 (mod nx): R[c][y] (column-major, ny long).
__device__ void row_pass(const RunParams& p, int64_t f, int q, int k0x, float2* R, float2* S0,
                         float2* S1, const FFTPlan& pl) {
  const Geometry& g = p.g;
  const int nx = g.nx, ny = g.ny, ny2 = g.ny >> 1, ww = g.ww;
  const int col0 = g.col0[q], row0 = g.row0[q];
  for (int c0 = 0; c0 < ny2; c0 += p.lay.CH) {
    const int ch = min(p.lay.CH, ny2 - c0);
    for (int idx = threadIdx.x; idx < ch * nx; idx += blockDim.x) {
      const int s = idx / nx, x = idx - s * nx, y = c0 + s;
      const float a = load_px(p.frames, p.fmt, p.transpose, g.W, g.H, f, row0 + y, col0 + x);
      const float b = load_px(p.frames, p.fmt, p.transpose, g.W, g.H, f, row0 + y + ny2, col0 + x);
      S0[idx] = make_float2(a, b);
    }
    __syncthreads();
    const float2* Z = stockham<false>(S0, S1, pl, ch, nx, 1);
    for (int idx = threadIdx.x; idx < ch * ww; idx += blockDim.x) {
      const int c = idx / ch, s = idx - c * ch;
      const int kx = pmod(k0x + c - ww / 2, nx);
      const int km = kx ? nx - kx : 0;
      const float2 zk = Z[s * nx + kx], zm = Z[s * nx + km];
      R[c * ny + c0 + s] = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
      R[c * ny + c0 + s + ny2] = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- column pass
// FFT along y of each kept column; keep rows ky_r = k0y + r - wh/2 (mod ny);
// multiply by the (mask * recentring phase [/ sinc]) table -> Wout[r][c].
__device__ void col_pass(const RunParams& p, int k0y, const float2* wtab, float2* R, float2* S0,
                         const FFTPlan& pl, float2* Wout) {
  const Geometry& g = p.g;
  const int ny = g.ny, ww = g.ww, wh = g.wh;
  for (int c0 = 0; c0 < ww; c0 += p.lay.CC) {
    const int cc = min(p.lay.CC, ww - c0);
    const float2* res = stockham<false>(R + (size_t)c0 * ny, S0, pl, cc, ny, 1);
    for (int idx = threadIdx.x; idx < wh * cc; idx += blockDim.x) {
      const int j = idx / wh, r = idx - j * wh, c = c0 + j;
      const int ky = pmod(k0y + r - wh / 2, ny);
      Wout[r * ww + c] = cmul(res[j * ny + ky], __ldg(&wtab[r * ww + c]));
    }
    __syncthreads();
  }
}

// -------------------------------------------------------------- epilogue
struct Stats {
  double v[6];  // tot, sx, sy, s2, cwrap, swrap
};

__device__ void write_params(float* params, int P, int slots, int q, int slot, const double* v,
                             float maxabs, int argmax, double da, double ya0, double span) {
  const double tot = v[0];
  float out[7];
  out[0] = (float)(tot * da);
  if (tot > 0.0) {
    out[1] = (float)(v[1] / tot);
    out[2] = (float)(v[2] / tot);
    out[5] = (float)((tot * da) * (tot * da) / (v[3] * da));
    double th = atan2(v[5], v[4]);
    th = fmod(th, 2.0 * M_PI);
    if (th < 0) th += 2.0 * M_PI;
    out[6] = (float)(ya0 + th * span / (2.0 * M_PI));
  } else {
    out[1] = out[2] = out[5] = 0.f;
    out[6] = (float)ya0;
  }
  out[3] = maxabs;
  out[4] = __int_as_float(argmax);
#pragma unroll
  for (int k = 0; k < 7; ++k) params[((size_t)k * P + q) * slots + slot] = out[k];
}

// Overlap of the dequantised field F (gh x gw, in `F`) with the separable basis:
// U[y][m] = sum_x F[y][x] hx[m][x];  c(m,n) = dxdy * sum_y hy[n][y] U[y][m]
// (holopipe/hgbasis.py:101-116).
__device__ void overlap(const RunParams& p, int q, const float2* F, float2* U, float2* out) {
  const Geometry& g = p.g;
  const int G = g.G, gh = g.gh, gw = g.gw;
  const float* hx = p.t.hx + (size_t)q * G * gw;
  const float* hy = p.t.hy + (size_t)q * G * gh;
  for (int idx = threadIdx.x; idx < gh * G; idx += blockDim.x) {
    const int y = idx / G, m = idx - y * G;
    const float2* row = F + (size_t)y * gw;
    const float* h = hx + (size_t)m * gw;
    float ax = 0.f, ay = 0.f;
    for (int x = 0; x < gw; ++x) {
      const float2 v = row[x];
      const float hv = __ldg(&h[x]);
      ax = fmaf(v.x, hv, ax);
      ay = fmaf(v.y, hv, ay);
    }
    U[idx] = make_float2(ax, ay);
  }
  __syncthreads();
  const float d = g.dxdy[q];
  for (int i = threadIdx.x; i < g.M; i += blockDim.x) {
    const int m = p.t.mode_m[i], n = p.t.mode_n[i];
    const float* h = hy + (size_t)n * gh;
    float ax = 0.f, ay = 0.f;
    for (int y = 0; y < gh; ++y) {
      const float2 v = U[y * G + m];
      const float hv = __ldg(&h[y]);
      ax = fmaf(v.x, hv, ax);
      ay = fmaf(v.y, hv, ay);
    }
    out[i] = make_float2(ax * d, ay * d);
  }
  __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(NT) fused_kernel(const __grid_constant__ RunParams p) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double red[8][32];
  __shared__ float redf[32];
  __shared__ int redi[32];
  const Geometry& g = p.g;
  char* slab = p.lay.slab_bytes ? p.work + (int64_t)blockIdx.x * p.lay.slab_bytes : nullptr;
  float2* R = region_ptr(p.lay.R, smem, slab);
  float2* S0 = region_ptr(p.lay.S0, smem, slab);
  float2* S1 = region_ptr(p.lay.S1, smem, slab);
  float2* Wt = region_ptr(p.lay.Wt, smem, slab);
  float2* Gd = region_ptr(p.lay.Gd, smem, slab);
  double2* Acc = reinterpret_cast<double2*>(region_ptr(p.lay.Acc, smem, slab));
  const bool summary = (p.flags & 1u) != 0;
  const int ghw = g.gh * g.gw, whw = g.wh * g.ww;
  double* agg = summary ? reinterpret_cast<double*>(p.work + p.lay.agg_off +
                                                    (int64_t)blockIdx.x * p.lay.agg_per_cta)
                        : nullptr;
  if (agg)
    for (int i = threadIdx.x; i < g.P * ghw; i += blockDim.x) agg[i] = 0.0;

  const FFTPlan pl_nx = make_plan(g.nx, g.nst_nx, g.radix_nx, p.t.tw_nx);
  const FFTPlan pl_ny = make_plan(g.ny, g.nst_ny, g.radix_ny, p.t.tw_ny);
  const FFTPlan pl_gw = make_plan(g.gw, g.nst_gw, g.radix_gw, p.t.tw_gw);
  const FFTPlan pl_gh = make_plan(g.gh, g.nst_gh, g.radix_gh, p.t.tw_gh);
  const double da = g.dx * g.dy;
  const double span = g.dy * g.gh;

  const int items = p.B * g.P;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int b = item / g.P, q = item - b * g.P;
    const int w = p.wl ? p.wl[b] : 0;
    const int k0x = g.k0[q][w][0], k0y = g.k0[q][w][1];
    const float2* wtab = p.t.win_tab + (size_t)(q * g.L + w) * whw;

    for (int a = 0; a < p.A; ++a) {
      const int64_t f = p.members ? (int64_t)p.members[(int64_t)b * p.A + a] : (int64_t)b * p.A + a;
      row_pass(p, f, q, k0x, R, S0, S1, pl_nx);
      col_pass(p, k0y, wtab, R, S0, pl_ny, Wt);
      if (p.A > 1) {
        // constructive average (holopipe/engine.py:543-552), complex128 accumulator
        if (a == 0) {
          for (int i = threadIdx.x; i < whw; i += blockDim.x)
            Acc[i] = make_double2(Wt[i].x, Wt[i].y);
        } else {
          double v[2] = {0.0, 0.0};
          for (int i = threadIdx.x; i < whw; i += blockDim.x) {
            const double2 ac = Acc[i];
            const float2 m = Wt[i];
            v[0] += ac.x * m.x + ac.y * m.y;
            v[1] += ac.x * m.y - ac.y * m.x;
          }
          block_sum<2>(v, red);
          const double mag = hypot(v[0], v[1]);
          const double cr = mag > 0.0 ? v[0] / mag : 1.0, ci = mag > 0.0 ? -v[1] / mag : 0.0;
          for (int i = threadIdx.x; i < whw; i += blockDim.x) {
            const float2 m = Wt[i];
            double2 ac = Acc[i];
            ac.x += m.x * cr - m.y * ci;
            ac.y += m.x * ci + m.y * cr;
            Acc[i] = ac;
          }
        }
        __syncthreads();
      }
    }
    if (p.A > 1) {
      const double inv = 1.0 / p.A;
      for (int i = threadIdx.x; i < whw; i += blockDim.x)
        Wt[i] = make_float2((float)(Acc[i].x * inv), (float)(Acc[i].y * inv));
      __syncthreads();
    }
    if (p.windows) {
      float2* wo = p.windows + (size_t)item * whw;
      for (int i = threadIdx.x; i < whw; i += blockDim.x) wo[i] = Wt[i];
    }

    // ---------------- inverse transform on the (gh x gw) grid
    float2* grid = Wt;
    if (g.gh != g.wh || g.gw != g.ww) {  // resolution mode 0: centred embedding
      const int r0 = g.gh / 2 - g.wh / 2, c0 = g.gw / 2 - g.ww / 2;
      for (int i = threadIdx.x; i < ghw; i += blockDim.x) {
        const int y = i / g.gw, x = i - y * g.gw;
        const int r = y - r0, c = x - c0;
        Gd[i] = (r >= 0 && r < g.wh && c >= 0 && c < g.ww) ? Wt[r * g.ww + c] : make_float2(0.f, 0.f);
      }
      __syncthreads();
      grid = Gd;
    }
    float2* r1 = stockham<true>(grid, S0, pl_gw, g.gh, g.gw, 1);
    float2* F = stockham<true>(r1, r1 == grid ? S0 : grid, pl_gh, g.gw, 1, g.gw);

    // ---------------- removal phase, calibrations, summary, peak
    const float2* ex = p.t.rem_x + (size_t)(q * g.L + w) * g.gw;
    const float2* ey = p.t.rem_y + (size_t)(q * g.L + w) * g.gh;
    float2 bc = make_float2(1.f, 0.f);
    if (p.bcal) bc = p.bcal[(size_t)min(q, p.cal_pols - 1) * p.cal_batch + ((p.row_offset + b) % p.cal_batch)];
    const float2* rc = p.rcal ? p.rcal + ((size_t)(w % p.rcal_count) * g.P + q) * ghw : nullptr;
    float lmax = 0.f, amax = -1.f;
    int aidx = 0x7fffffff;
    double st[6] = {0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < ghw; i += blockDim.x) {
      const int y = i / g.gw, x = i - y * g.gw;
      float2 v = cmul(cmul(F[i], __ldg(&ey[y])), __ldg(&ex[x]));
      if (p.bcal) v = cmul(v, bc);
      if (rc) v = cmul(v, rc[i]);
      F[i] = v;
      lmax = fmaxf(lmax, fmaxf(fabsf(v.x), fabsf(v.y)));
      if (p.raw) p.raw[(size_t)item * ghw + i] = v;
      if (summary) {
        const float mag = hypotf(v.x, v.y);
        const double I = (double)mag * (double)mag;
        st[0] += I;
        st[1] += I * __ldg(&p.t.xad[x]);
        st[2] += I * __ldg(&p.t.yad[y]);
        st[3] += I * I;
        const double ang = 2.0 * M_PI * (__ldg(&p.t.yad[y]) - __ldg(&p.t.yad[0])) / span;
        double sn, cs;
        sincos(ang, &sn, &cs);
        st[4] += I * cs;
        st[5] += I * sn;
        if (mag > amax) { amax = mag; aidx = i; }
        agg[(size_t)q * ghw + i] += I;
      }
    }
    const float peak = block_max(lmax, redf);
    if (summary) {
      block_sum<6>(st, red);
      block_argmax(amax, aidx, redf, redi);
      if (threadIdx.x == 0 && p.params)
        write_params(p.params, g.P, p.param_slots, q, b, st, amax, aidx, da, p.t.yad[0], span);
    }
    const float scale = peak > 0.f ? (float)(32767.0 / (double)peak) : 1.0f;
    // ---------------- int16 packing (holopipe/pipeline.py:188-199), dequantised copy
    int16_t* fro = p.fr + (size_t)item * ghw;
    int16_t* fio = p.fi + (size_t)item * ghw;
    for (int i = threadIdx.x; i < ghw; i += blockDim.x) {
      const float2 v = F[i];
      const int qr = __float2int_rn(__fmul_rn(v.x, scale));
      const int qi = __float2int_rn(__fmul_rn(v.y, scale));
      fro[i] = (int16_t)qr;
      fio[i] = (int16_t)qi;
      F[i] = make_float2(__fdiv_rn((float)qr, scale), __fdiv_rn((float)qi, scale));
    }
    if (threadIdx.x == 0) p.scale[item] = scale;
    __syncthreads();
    if (p.coefs && g.G > 0) {
      float2* U = (F == S0) ? S1 : S0;
      if (F != S0 && F != S1) U = S1;
      overlap(p, q, F, U, p.coefs + (size_t)item * g.M);
    }
    __syncthreads();
  }
}

// Generic plane statistics (holopipe/analysis.py:39-94) of complex data
// [count][P][h][w]: one CTA per (frame, pol) item writes its seven parameters
// and accumulates |F|^2 into its own fp64 aggregate image (deterministic:
// the finalize kernel sums the per-CTA images in a fixed order).
struct PlaneArgs {
  const float2* data;
  int64_t count;
  int P, h, w;
  const double* xa;
  const double* ya;
  float* params;
  int slots;
  char* agg;           // per-CTA [P][h][w] doubles
  int64_t agg_per_cta; // bytes
  float* total;        // [h][w] or NULL
  double* pol_total;   // [P][h][w] or NULL
  int agg_slot;        // slot index of the aggregate column
  int nblocks;         // CTAs that produced partials (finalize)
};

__device__ void stats_loop(const PlaneArgs& a, int q, const float2* d, double* agg, double* st, float& amax,
                           int& aidx) {
  const int hw = a.h * a.w;
  const double span = (a.h > 1 ? fabs(a.ya[1] - a.ya[0]) : 1.0) * a.h;
  for (int i = threadIdx.x; i < hw; i += blockDim.x) {
    const int y = i / a.w, x = i - y * a.w;
    const float2 v = d[i];
    const float mag = hypotf(v.x, v.y);
    const double I = (double)mag * (double)mag;
    st[0] += I;
    st[1] += I * a.xa[x];
    st[2] += I * a.ya[y];
    st[3] += I * I;
    double sn, cs;
    sincos(2.0 * M_PI * (a.ya[y] - a.ya[0]) / span, &sn, &cs);
    st[4] += I * cs;
    st[5] += I * sn;
    if (mag > amax) { amax = mag; aidx = i; }
    agg[(size_t)q * hw + i] += I;
  }
}

__global__ void __launch_bounds__(kThreads) plane_stats_kernel(const PlaneArgs a) {
  __shared__ double red[8][32];
  __shared__ float redf[32];
  __shared__ int redi[32];
  const int hw = a.h * a.w;
  double* agg = reinterpret_cast<double*>(a.agg + (int64_t)blockIdx.x * a.agg_per_cta);
  for (int i = threadIdx.x; i < a.P * hw; i += blockDim.x) agg[i] = 0.0;
  __syncthreads();
  const double dx = a.w > 1 ? fabs(a.xa[1] - a.xa[0]) : 1.0;
  const double dy = a.h > 1 ? fabs(a.ya[1] - a.ya[0]) : 1.0;
  for (int64_t item = blockIdx.x; item < a.count * a.P; item += gridDim.x) {
    const int q = (int)(item % a.P);
    const int64_t f = item / a.P;
    double st[6] = {0, 0, 0, 0, 0, 0};
    float amax = -1.f;
    int aidx = 0x7fffffff;
    stats_loop(a, q, a.data + (size_t)item * hw, agg, st, amax, aidx);
    block_sum<6>(st, red);
    block_argmax(amax, aidx, redf, redi);
    if (threadIdx.x == 0)
      write_params(a.params, a.P, a.slots, q, (int)f, st, amax, aidx, dx * dy, a.ya[0], dy * a.h);
  }
}

// Aggregate slot: per-pixel sum of the per-CTA images in fixed CTA order, then
// the seven parameters on the summed intensity with MAXABS = max sqrt(sum)
// (analysis.py:88-91) and the total over pols (analysis.py:92).
__global__ void __launch_bounds__(kThreads) plane_finalize_kernel(const PlaneArgs a) {
  __shared__ double red[8][32];
  __shared__ int redi[32];
  const int q = blockIdx.x;
  const int hw = a.h * a.w;
  const int64_t stride = a.agg_per_cta / (int64_t)sizeof(double);
  const double* base = reinterpret_cast<const double*>(a.agg);
  const double dx = a.w > 1 ? fabs(a.xa[1] - a.xa[0]) : 1.0;
  const double dy = a.h > 1 ? fabs(a.ya[1] - a.ya[0]) : 1.0;
  const double span = dy * a.h;
  double st[6] = {0, 0, 0, 0, 0, 0};
  double amax = -1.0;
  int aidx = 0x7fffffff;
  for (int i = threadIdx.x; i < hw; i += blockDim.x) {
    const int y = i / a.w, x = i - y * a.w;
    double I = 0.0;
    for (int c = 0; c < a.nblocks; ++c) I += base[c * stride + (size_t)q * hw + i];
    st[0] += I;
    st[1] += I * a.xa[x];
    st[2] += I * a.ya[y];
    st[3] += I * I;
    double sn, cs;
    sincos(2.0 * M_PI * (a.ya[y] - a.ya[0]) / span, &sn, &cs);
    st[4] += I * cs;
    st[5] += I * sn;
    if (I > amax) { amax = I; aidx = i; }
    if (a.pol_total) a.pol_total[(size_t)q * hw + i] = I;
    if (a.total && q == 0) {
      double tI = I;
      for (int qq = 1; qq < a.P; ++qq)
        for (int c = 0; c < a.nblocks; ++c) tI += base[c * stride + (size_t)qq * hw + i];
      a.total[i] = (float)tI;
    }
  }
  block_sum<6>(st, red);
  float fm = (float)sqrt(fmax(amax, 0.0));
  // argmax on the fp64 intensity (sqrt is monotonic), ties -> first index
  {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, amax, o);
      const int oi = __shfl_xor_sync(0xffffffffu, aidx, o);
      if (ov > amax || (ov == amax && oi < aidx)) { amax = ov; aidx = oi; }
    }
    __syncthreads();
    if (l == 0) { red[6][w] = amax; redi[w] = aidx; }
    __syncthreads();
    amax = red[6][0];
    aidx = redi[0];
    for (int j = 1; j < nw; ++j)
      if (red[6][j] > amax || (red[6][j] == amax && redi[j] < aidx)) { amax = red[6][j]; aidx = redi[j]; }
    fm = (float)sqrt(fmax(amax, 0.0));
  }
  if (threadIdx.x == 0) write_params(a.params, a.P, a.slots, q, a.agg_slot, st, fm, aidx, dx * dy, a.ya[0], span);
}

// Overlap of already-quantised fields: one CTA per (row, pol).
__global__ void __launch_bounds__(kThreads) coefs_kernel(const __grid_constant__ RunParams p) {
  extern __shared__ __align__(16) char smem[];
  const Geometry& g = p.g;
  const int ghw = g.gh * g.gw;
  float2* F = reinterpret_cast<float2*>(smem);
  float2* U = F + ghw;
  for (int item = blockIdx.x; item < p.B * g.P; item += gridDim.x) {
    const float s = p.scale[item];
    for (int i = threadIdx.x; i < ghw; i += blockDim.x)
      F[i] = make_float2(__fdiv_rn((float)p.fr[(size_t)item * ghw + i], s),
                         __fdiv_rn((float)p.fi[(size_t)item * ghw + i], s));
    __syncthreads();
    overlap(p, item % g.P, F, U, p.coefs + (size_t)item * g.M);
  }
}

// ------------------------------------------------------- full R2C plane
// plane[f][q][ky][kx], kx < nx/2+1 (holopipe/pipeline.py:47-59).
__global__ void __launch_bounds__(kThreads) fourier_full_kernel(const __grid_constant__ RunParams p,
                                                               int64_t F, float2* plane) {
  extern __shared__ __align__(16) char smem[];
  const Geometry& g = p.g;
  char* slab = p.lay.slab_bytes ? p.work + (int64_t)blockIdx.x * p.lay.slab_bytes : nullptr;
  float2* R = region_ptr(p.lay.R, smem, slab);   // (nx/2+1) columns x ny
  float2* S0 = region_ptr(p.lay.S0, smem, slab);
  float2* S1 = region_ptr(p.lay.S1, smem, slab);
  const FFTPlan pl_nx = make_plan(g.nx, g.nst_nx, g.radix_nx, p.t.tw_nx);
  const FFTPlan pl_ny = make_plan(g.ny, g.nst_ny, g.radix_ny, p.t.tw_ny);
  const int nx = g.nx, ny = g.ny, ny2 = ny / 2, nh = nx / 2 + 1;
  for (int64_t item = blockIdx.x; item < F * g.P; item += gridDim.x) {
    const int64_t f = item / g.P;
    const int q = (int)(item - f * g.P);
    const int col0 = g.col0[q], row0 = g.row0[q];
    for (int c0 = 0; c0 < ny2; c0 += p.lay.CH) {
      const int ch = min(p.lay.CH, ny2 - c0);
      for (int idx = threadIdx.x; idx < ch * nx; idx += blockDim.x) {
        const int s = idx / nx, x = idx - s * nx, y = c0 + s;
        S0[idx] = make_float2(load_px(p.frames, p.fmt, p.transpose, g.W, g.H, f, row0 + y, col0 + x),
                              load_px(p.frames, p.fmt, p.transpose, g.W, g.H, f, row0 + y + ny2, col0 + x));
      }
      __syncthreads();
      const float2* Z = stockham<false>(S0, S1, pl_nx, ch, nx, 1);
      for (int idx = threadIdx.x; idx < ch * nh; idx += blockDim.x) {
        const int c = idx / ch, s = idx - c * ch;
        const int km = c ? nx - c : 0;
        const float2 zk = Z[s * nx + c], zm = Z[s * nx + km];
        R[c * ny + c0 + s] = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
        R[c * ny + c0 + s + ny2] = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
      }
      __syncthreads();
    }
    float2* out = plane + (size_t)item * ny * nh;
    for (int c0 = 0; c0 < nh; c0 += p.lay.CC) {
      const int cc = min(p.lay.CC, nh - c0);
      const float2* res = stockham<false>(R + (size_t)c0 * ny, S0, pl_ny, cc, ny, 1);
      for (int idx = threadIdx.x; idx < ny * cc; idx += blockDim.x) {
        const int ky = idx / cc, j = idx - ky * cc;
        out[(size_t)ky * nh + c0 + j] = res[j * ny + ky];
      }
      __syncthreads();
    }
  }
}

// Sum over the batch of |dequantised int16 field|^2 per pol, fp64, fixed order.
__global__ void field_intensity_kernel(const int16_t* fr, const int16_t* fi, const float* scale, int B, int P,
                                       int hw, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)P * hw) return;
  const int q = (int)(i / hw), pix = (int)(i - (int64_t)q * hw);
  double acc = 0.0;
  for (int b = 0; b < B; ++b) {
    const size_t o = ((size_t)b * P + q) * hw + pix;
    const double s = (double)scale[(size_t)b * P + q];
    const double re = (double)fr[o] / s, im = (double)fi[o] / s;
    acc += re * re + im * im;
  }
  out[i] = acc;
}

cudaError_t launch_field_intensity(const int16_t* fr, const int16_t* fi, const float* scale, int B, int P, int hw,
                                   double* out, cudaStream_t s) {
  const int64_t n = (int64_t)P * hw;
  field_intensity_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(fr, fi, scale, B, P, hw, out);
  return cudaGetLastError();
}

// applied = conj(proc) / max(|proc|^2, eps) with proc = a (+ i b), fp64 (engine.py:332-334)
__global__ void refcal_finish_kernel(const float2* a, const float2* b, int64_t n, float2* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float2 v = a[i];
  if (b) {   // a + i b, rounded to complex64 like the reference's complex64 field
    const float2 w = b[i];
    v = make_float2(v.x - w.y, v.y + w.x);
  }
  const double re = (double)v.x, im = (double)v.y;
  const double mag2 = fmax(re * re + im * im, 1e-6);
  out[i] = make_float2((float)(re / mag2), (float)(-im / mag2));
}

cudaError_t launch_refcal_finish(const float2* a, const float2* b, int64_t n, float2* out, cudaStream_t s) {
  refcal_finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, b, n, out);
  return cudaGetLastError();
}

// ------------------------------------------------------ large-window path
// Windows too large for one CTA's shared memory (config 3: 512^2 window, 164^2 field) run as
// four grid-wide kernels over chunks of items whose intermediates stay resident in L2:
//   lw_rows   row pairs (y, y + ny/2) -> complex FFT along x -> Hermitian split -> R[c][y]
//   lw_cols   FFT along y of kept columns -> crop (mask * recentring [/ sinc]) -> IFFT along r -> T[c][y']
//   lw_field  IFFT along c of field rows -> removal phase, calibrations -> F[y'][x'], per-item peak
//   lw_pack   int16 packing with scale = float32(32767 / peak) (holopipe/pipeline.py:188-199)
// Same algebra as row_pass / col_pass / the fused epilogue; every CTA works on one item.
// output position of bin n in the group's buffer (one pad per 8: conflict-free pass-3 stores)
HOLO_DEV int f512_pos(int n) { return n + (n >> 3); }

// 512-point forward FFT by a group of 64 threads, three radix-8 passes (x = t + 64 j in registers
// -> twiddle W512^(t k) -> S1[k][t]; DFT-8 over t1 of t = t0 + 8 t1 -> twiddle W64^(t0 m1) ->
// S2[k][m1][t0]; DFT-8 over t0 -> X[k + 8 m1 + 64 m2]).  S1 (8 x 72) also receives the output
// (bin n at f512_pos(n), 576 float2); S2 is 64 x 9.  Every pass ends in a CTA barrier (all groups in lockstep).
HOLO_DEV void fft512_group(float2 (&a)[8], int t, const float2* __restrict__ tw, float2* S1, float2* S2) {
  dft8<false>(a);
#pragma unroll
  for (int k = 0; k < 8; ++k) S1[k * 72 + t] = k ? cmul(a[k], __ldg(&tw[(t * k) & 511])) : a[k];
  __syncthreads();
  {
    const int k = t >> 3, t0 = t & 7;
    float2 c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = S1[k * 72 + t0 + 8 * j];
    dft8<false>(c);
#pragma unroll
    for (int m1 = 0; m1 < 8; ++m1)
      S2[(k * 8 + m1) * 9 + t0] = m1 ? cmul(c[m1], __ldg(&tw[(8 * t0 * m1) & 511])) : c[m1];
  }
  __syncthreads();
  {
    const int k = t >> 3, m1 = t & 7;
    float2 e[8];
#pragma unroll
    for (int t0 = 0; t0 < 8; ++t0) e[t0] = S2[(k * 8 + m1) * 9 + t0];
    dft8<false>(e);
#pragma unroll
    for (int m2 = 0; m2 < 8; ++m2) S1[f512_pos(k + 8 * m1 + 64 * m2)] = e[m2];   // S1 is free after pass 2
  }
  __syncthreads();
}
constexpr int kF512Group = 8 * 72 + 64 * 9;   // float2 of scratch per 512-point group

// Row pass for 512-wide windows: 16 row pairs per 512-thread CTA, two per 64-thread group; both pairs' frame
// rows are loaded before the first FFT so the second load's latency hides behind it.
constexpr int kRows512Sets = 2;
__global__ void __launch_bounds__(512) lw_rows512_kernel(const __grid_constant__ RunParams p, int i0, int i1,
                                                          float2* __restrict__ R) {
  extern __shared__ __align__(16) char smem[];
  const Geometry& g = p.g;
  const int ny = g.ny, ny2 = ny >> 1, ww = g.ww;
  const int nblk = ny2 / (8 * kRows512Sets);
  const int item = i0 + blockIdx.x / nblk, yb = (blockIdx.x % nblk) * 8 * kRows512Sets;
  if (item >= i1) return;
  const int b = item / g.P, q = item - b * g.P;
  const int w = p.wl ? p.wl[b] : 0;
  const int k0x = g.k0[q][w][0];
  const int grp = threadIdx.x >> 6, t = threadIdx.x & 63;
  float2* S1 = reinterpret_cast<float2*>(smem) + grp * kF512Group;
  float2* S2 = S1 + 8 * 72;
  float2 a[kRows512Sets][8];
#pragma unroll
  for (int st = 0; st < kRows512Sets; ++st) {
    const int y = yb + 8 * st + grp;
    if (p.fmt == 0) {
      const float* ra = reinterpret_cast<const float*>(p.frames) + (int64_t)b * g.W * g.H +
                        (int64_t)(g.row0[q] + y) * g.W + g.col0[q];
      const float* rb = ra + (int64_t)ny2 * g.W;
#pragma unroll
      // streaming (evict-first) loads: the frame is read once and must not push the row-pass output R,
      // which the column kernel reads back from L2, out to DRAM
      for (int j = 0; j < 8; ++j) a[st][j] = make_float2(__ldcs(ra + t + 64 * j), __ldcs(rb + t + 64 * j));
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        a[st][j] = make_float2(load_px(p.frames, p.fmt, p.transpose, g.W, g.H, b, g.row0[q] + y, g.col0[q] + t + 64 * j),
                               load_px(p.frames, p.fmt, p.transpose, g.W, g.H, b, g.row0[q] + y + ny2,
                                       g.col0[q] + t + 64 * j));
    }
  }
  float2* Ri = R + (size_t)(item - i0) * ww * ny;
  const float2* X0 = reinterpret_cast<const float2*>(smem);
#pragma unroll
  for (int st = 0; st < kRows512Sets; ++st) {
    const int y0 = yb + 8 * st;
    if (st > 0) __syncthreads();   // the previous set's bins are read out
    fft512_group(a[st], t, p.t.tw_nx, S1, S2);
    // Hermitian split of the kept bins; the 8 row pairs of the set write 8 consecutive y per column
    for (int idx = threadIdx.x; idx < 8 * ww; idx += blockDim.x) {
      const int c = idx >> 3, s = idx & 7;
      const int kx = pmod(k0x + c - ww / 2, 512);
      const int km = (512 - kx) & 511;
      const float2* X = X0 + s * kF512Group;
      const float2 zk = X[f512_pos(kx)], zm = X[f512_pos(km)];
      Ri[(size_t)c * ny + y0 + s] = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
      Ri[(size_t)c * ny + y0 + s + ny2] = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
    }
  }
}

HOLO_DEV void ifft164(float2* S0, float2* S1, float2* scr, int count, const float2* __restrict__ tw);

// Column pass for 512-high windows: 8 columns per 512-thread CTA; FFT along y (512), crop, window table
// -> W[c][r] in T.  FUSE164 (164-row field grids, config 3): the 164-point IFFT along r of the CTA's 8 columns
// follows in the same CTA (the FFT scratch is reused) and T receives the transformed columns directly.
template <bool FUSE164>
__global__ void __launch_bounds__(512) lw_cols512_kernel(const __grid_constant__ RunParams p, int i0, int i1,
                                                          const float2* __restrict__ R, float2* __restrict__ T) {
  extern __shared__ __align__(16) char smem[];
  const Geometry& g = p.g;
  const int ny = g.ny, ww = g.ww, wh = g.wh;
  const int nblk = (ww + 7) / 8;
  const int item = i0 + blockIdx.x / nblk, c0 = (blockIdx.x % nblk) * 8;
  if (item >= i1) return;
  const int b = item / g.P, q = item - b * g.P;
  const int w = p.wl ? p.wl[b] : 0;
  const int k0y = g.k0[q][w][1];
  const int cc = min(8, ww - c0);
  const int grp = threadIdx.x >> 6, t = threadIdx.x & 63;
  float2* S1 = reinterpret_cast<float2*>(smem) + grp * kF512Group;
  float2* S2 = S1 + 8 * 72;
  const float2* Rc = R + (size_t)(item - i0) * ww * ny + (size_t)(c0 + min(grp, cc - 1)) * ny;
  float2 a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = Rc[t + 64 * j];
  fft512_group(a, t, p.t.tw_ny, S1, S2);
  // The column is consumed (fft512_group synchronises the CTA, so the duplicate reads of a partial block are
  // done too): drop its 32 dirty lines from L2 instead of letting them be written back to DRAM -- R is scratch,
  // rewritten by the next slot's row pass.  (Measured: 18.3 MB of DRAM writes per 26-window slot before.)
  if (grp < cc && t < 32)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<const char*>(Rc) + t * 128) : "memory");
  // crop + window table -> Wg[c][r] (global, column-major); the IFFT along r runs in lw_ifft_y
  const float2* wtab = p.t.win_tab + (size_t)(q * g.L + w) * wh * ww;
  const float2* X0 = reinterpret_cast<const float2*>(smem);
  float2* Wg = T + (size_t)(item - i0) * ww * wh + (size_t)c0 * wh;
  if constexpr (FUSE164) {
    constexpr int kPer = (164 * 8 + 511) / 512;   // cropped values per thread
    float2 v[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int idx = threadIdx.x + 512 * u;
      if (idx < wh * cc) {
        const int j = idx / wh, r = idx - j * wh, c = c0 + j;
        const int ky = pmod(k0y + r - wh / 2, 512);
        v[u] = cmul(X0[j * kF512Group + f512_pos(ky)], __ldg(&wtab[r * ww + c]));
      }
    }
    __syncthreads();   // the FFT scratch is free: S0 | S1 | radix-41 sums
    float2* S0 = reinterpret_cast<float2*>(smem);
    float2* S1 = S0 + 8 * 164;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int idx = threadIdx.x + 512 * u;
      if (idx < wh * cc) S0[idx] = v[u];
    }
    __syncthreads();
    ifft164(S0, S1, S1 + 8 * 164, cc, p.t.tw_gh);
    for (int idx = threadIdx.x; idx < wh * cc; idx += blockDim.x) Wg[idx] = S0[idx];
  } else {
    for (int idx = threadIdx.x; idx < wh * cc; idx += blockDim.x) {
      const int j = idx / wh, r = idx - j * wh, c = c0 + j;
      const int ky = pmod(k0y + r - wh / 2, 512);
      Wg[idx] = cmul(X0[j * kF512Group + f512_pos(ky)], __ldg(&wtab[r * ww + c]));
    }
  }
}

// Inverse 164-point transforms (164 = 4 x 41) of `count` sequences (stride 164), S0 -> S0 via S1:
// the radix-4 Stockham stage, then the radix-41 stage split over (sequence, k, output pair) work
// items with the conjugate-pair sums staged in `scr` (count * 4 * 20 * 2 float2), so every thread
// of the CTA has work (one task per thread keeps 20-deep FMA chains on a few threads).
HOLO_DEV void ifft164(float2* S0, float2* S1, float2* scr, int count, const float2* __restrict__ tw) {
  constexpr int N = 164, L = 4, P = 41, H = 20;
  __shared__ float cs41[2][P];   // per-thread (divergent) indices: shared memory, not the constant cache
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    cs41[0][i] = kCos41[i];
    cs41[1][i] = kSin41[i];
  }
  stockham_stage_fixed<4, true>(S0, S1, N, 1, count, N, 1, tw, threadIdx.x, blockDim.x);
  __syncthreads();
  float2* SP = scr;
  float2* SM = scr + count * L * H;
  for (int i = threadIdx.x; i < count * L * H; i += blockDim.x) {   // (q, k, j)
    const int qk = i / H, j = i - qk * H + 1, q = qk >> 2, k = qk & 3;
    const float2* src = S1 + q * N;
    const float2 a = cmul(src[k * P + j], twid<true>(__ldg(&tw[(j * k) % N])));
    const float2 b = cmul(src[k * P + P - j], twid<true>(__ldg(&tw[((P - j) * k) % N])));
    SP[i] = cadd(a, b);
    SM[i] = csub(a, b);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < count * L * (H + 1); i += blockDim.x) {   // (q, k, t)
    const int qk = i / (H + 1), t = i - qk * (H + 1), q = qk >> 2, k = qk & 3;
    const float2 v0 = S1[q * N + k * P];
    const float2* sp = SP + qk * H;
    const float2* sm = SM + qk * H;
    float2* d = S0 + q * N;
    if (t == 0) {
      float2 tot = v0;
#pragma unroll
      for (int j = 0; j < H; ++j) tot = cadd(tot, sp[j]);
      d[k] = tot;
    } else {
      float2 re = v0, im = make_float2(0.f, 0.f);
      int e = 0;
#pragma unroll
      for (int j = 1; j <= H; ++j) {
        e += t; if (e >= P) e -= P;
        const float c = cs41[0][e], sn = cs41[1][e];
        re.x = fmaf(c, sp[j - 1].x, re.x);
        re.y = fmaf(c, sp[j - 1].y, re.y);
        im.x = fmaf(sn, sm[j - 1].x, im.x);
        im.y = fmaf(sn, sm[j - 1].y, im.y);
      }
      const float2 rr = rot90<true>(im);
      d[k + L * t] = cadd(re, rr);
      d[k + L * (P - t)] = csub(re, rr);
    }
  }
  __syncthreads();
}

// IFFT along r of kLwIfft columns per CTA (enough independent tasks for the radix-41 stage)
constexpr int kLwIfft = 16;
template <bool F164>
__global__ void __launch_bounds__(kThreads, 3) lw_ifft_y_kernel(const __grid_constant__ RunParams p, int i0, int i1,
                                                                 const float2* __restrict__ Wg, float2* __restrict__ T) {
  extern __shared__ __align__(16) char smem[];
  const Geometry& g = p.g;
  const int gh = g.gh, ww = g.ww;
  const int nblk = (ww + kLwIfft - 1) / kLwIfft;
  const int item = i0 + blockIdx.x / nblk, c0 = (blockIdx.x % nblk) * kLwIfft;
  if (item >= i1) return;
  const int cc = min(kLwIfft, ww - c0);
  float2* S0 = reinterpret_cast<float2*>(smem);
  float2* S1 = S0 + kLwIfft * gh;
  const float2* Wi = Wg + (size_t)(item - i0) * ww * gh + (size_t)c0 * gh;
  for (int i = threadIdx.x; i < cc * gh; i += blockDim.x) S0[i] = Wi[i];
  __syncthreads();
  const float2* tr;
  if constexpr (F164) {
    ifft164(S0, S1, S1 + kLwIfft * gh, cc, p.t.tw_gh);
    tr = S0;
  } else {
    const FFTPlan pg = make_plan(gh, g.nst_gh, g.radix_gh, p.t.tw_gh);
    tr = stockham<true>(S0, S1, pg, cc, gh, 1);
  }
  float2* Ti = T + (size_t)(item - i0) * ww * gh + (size_t)c0 * gh;
  for (int i = threadIdx.x; i < cc * gh; i += blockDim.x) Ti[i] = tr[i];
}

constexpr int kLwRows = 8;    // row pairs per lw_rows CTA
constexpr int kLwCols = 8;    // columns per lw_cols CTA
constexpr int kLwFRows = 16;  // field rows per lw_field CTA (tasks for the radix-41 stage)

__global__ void __launch_bounds__(kThreads) lw_rows_kernel(const __grid_constant__ RunParams p, int i0, int i1,
                                                            float2* __restrict__ R) {
  extern __shared__ __align__(16) char smem[];
  const Geometry& g = p.g;
  const int nx = g.nx, ny = g.ny, ny2 = ny >> 1, ww = g.ww;
  const int nblk = (ny2 + kLwRows - 1) / kLwRows;
  const int item = i0 + blockIdx.x / nblk, c0 = (blockIdx.x % nblk) * kLwRows;
  if (item >= i1) return;
  const int b = item / g.P, q = item - b * g.P;
  const int w = p.wl ? p.wl[b] : 0;
  const int k0x = g.k0[q][w][0];
  const int ch = min(kLwRows, ny2 - c0);
  float2* S0 = reinterpret_cast<float2*>(smem);
  float2* S1 = S0 + kLwRows * nx;
  const int col0 = g.col0[q], row0 = g.row0[q];
  for (int idx = threadIdx.x; idx < ch * nx; idx += blockDim.x) {
    const int sr = idx / nx, x = idx - sr * nx, y = c0 + sr;
    const float a = load_px(p.frames, p.fmt, p.transpose, g.W, g.H, b, row0 + y, col0 + x);
    const float bb = load_px(p.frames, p.fmt, p.transpose, g.W, g.H, b, row0 + y + ny2, col0 + x);
    S0[idx] = make_float2(a, bb);
  }
  __syncthreads();
  const FFTPlan pl = make_plan(nx, g.nst_nx, g.radix_nx, p.t.tw_nx);
  const float2* Z = stockham<false>(S0, S1, pl, ch, nx, 1);
  float2* Ri = R + (size_t)(item - i0) * ww * ny;
  for (int idx = threadIdx.x; idx < ch * ww; idx += blockDim.x) {
    const int c = idx / ch, sr = idx - c * ch;
    const int kx = pmod(k0x + c - ww / 2, nx);
    const int km = kx ? nx - kx : 0;
    const float2 zk = Z[sr * nx + kx], zm = Z[sr * nx + km];
    Ri[(size_t)c * ny + c0 + sr] = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
    Ri[(size_t)c * ny + c0 + sr + ny2] = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
  }
}

__global__ void __launch_bounds__(kThreads) lw_cols_kernel(const __grid_constant__ RunParams p, int i0, int i1,
                                                            const float2* __restrict__ R, float2* __restrict__ T) {
  extern __shared__ __align__(16) char smem[];
  const Geometry& g = p.g;
  const int ny = g.ny, ww = g.ww, wh = g.wh;
  const int nblk = (ww + kLwCols - 1) / kLwCols;
  const int item = i0 + blockIdx.x / nblk, c0 = (blockIdx.x % nblk) * kLwCols;
  if (item >= i1) return;
  const int b = item / g.P, q = item - b * g.P;
  const int w = p.wl ? p.wl[b] : 0;
  const int k0y = g.k0[q][w][1];
  const int cc = min(kLwCols, ww - c0);
  float2* S0 = reinterpret_cast<float2*>(smem);
  float2* S1 = S0 + kLwCols * ny;
  const float2* Ri = R + (size_t)(item - i0) * ww * ny + (size_t)c0 * ny;
  for (int i = threadIdx.x; i < cc * ny; i += blockDim.x) S0[i] = Ri[i];
  __syncthreads();
  const FFTPlan pl = make_plan(ny, g.nst_ny, g.radix_ny, p.t.tw_ny);
  const float2* res = stockham<false>(S0, S1, pl, cc, ny, 1);
  float2* Wc = res == S0 ? S1 : S0;   // [j][r], column-major window (gh == wh)
  const float2* wtab = p.t.win_tab + (size_t)(q * g.L + w) * wh * ww;
  for (int idx = threadIdx.x; idx < wh * cc; idx += blockDim.x) {
    const int j = idx / wh, r = idx - j * wh, c = c0 + j;
    const int ky = pmod(k0y + r - wh / 2, ny);
    Wc[idx] = cmul(res[j * ny + ky], __ldg(&wtab[r * ww + c]));
  }
  __syncthreads();
  // ifftshift and 1/(nx ny) live in the removal vectors (plan tables), so the IDFT is plain
  const FFTPlan pg = make_plan(g.gh, g.nst_gh, g.radix_gh, p.t.tw_gh);
  float2* other = Wc == S0 ? S1 : S0;
  const float2* tr = stockham<true>(Wc, other, pg, cc, wh, 1);
  float2* Ti = T + (size_t)(item - i0) * ww * g.gh + (size_t)c0 * g.gh;
  for (int i = threadIdx.x; i < cc * g.gh; i += blockDim.x) Ti[i] = tr[i];
}

template <bool F164>
__global__ void __launch_bounds__(kThreads, 3) lw_field_kernel(const __grid_constant__ RunParams p, int i0, int i1,
                                                                const float2* __restrict__ T, float2* __restrict__ Fo,
                                                                unsigned* __restrict__ peak) {
  extern __shared__ __align__(16) char smem[];
  __shared__ float redf[32];
  const Geometry& g = p.g;
  const int gh = g.gh, gw = g.gw;
  const int nblk = (gh + kLwFRows - 1) / kLwFRows;
  const int item = i0 + blockIdx.x / nblk, y0 = (blockIdx.x % nblk) * kLwFRows;
  if (item >= i1) return;
  const int b = item / g.P, q = item - b * g.P;
  const int w = p.wl ? p.wl[b] : 0;
  const int rr = min(kLwFRows, gh - y0);
  float2* S0 = reinterpret_cast<float2*>(smem);
  float2* S1 = S0 + kLwFRows * gw;
  const float2* Ti = T + (size_t)(item - i0) * gw * gh;
  for (int i = threadIdx.x; i < rr * gw; i += blockDim.x) {   // [s][c] <- T[c][y0 + s]
    const int c = i / rr, sr = i - c * rr;
    S0[sr * gw + c] = Ti[(size_t)c * gh + y0 + sr];
  }
  __syncthreads();
  const float2* Fr;
  if constexpr (F164) {
    ifft164(S0, S1, S1 + kLwFRows * gw, rr, p.t.tw_gw);
    Fr = S0;
  } else {
    const FFTPlan pl = make_plan(gw, g.nst_gw, g.radix_gw, p.t.tw_gw);
    Fr = stockham<true>(S0, S1, pl, rr, gw, 1);
  }
  const float2* ex = p.t.rem_x + (size_t)(q * g.L + w) * gw;
  const float2* ey = p.t.rem_y + (size_t)(q * g.L + w) * gh;
  float2 bc = make_float2(1.f, 0.f);
  if (p.bcal) bc = p.bcal[(size_t)min(q, p.cal_pols - 1) * p.cal_batch + ((p.row_offset + b) % p.cal_batch)];
  const float2* rc = p.rcal ? p.rcal + ((size_t)(w % p.rcal_count) * g.P + q) * gh * gw : nullptr;
  float2* Fi = Fo + (size_t)(item - i0) * gh * gw;
  float lmax = 0.f;
  for (int i = threadIdx.x; i < rr * gw; i += blockDim.x) {
    const int sr = i / gw, x = i - sr * gw, y = y0 + sr;
    float2 v = cmul(cmul(Fr[i], __ldg(&ey[y])), __ldg(&ex[x]));
    if (p.bcal) v = cmul(v, bc);
    if (rc) v = cmul(v, rc[(size_t)y * gw + x]);
    lmax = fmaxf(lmax, fmaxf(fabsf(v.x), fabsf(v.y)));
    Fi[(size_t)y * gw + x] = v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  if ((threadIdx.x & 31) == 0) redf[threadIdx.x >> 5] = lmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < (int)(blockDim.x >> 5); ++j) lmax = fmaxf(lmax, redf[j]);
    atomicMax(&peak[item - i0], __float_as_uint(lmax));   // non-negative floats order as unsigned
  }
}

__global__ void __launch_bounds__(kThreads) lw_pack_kernel(const __grid_constant__ RunParams p, int i0, int i1,
                                                            const float2* __restrict__ Fo,
                                                            const unsigned* __restrict__ peak) {
  const Geometry& g = p.g;
  const int ghw = g.gh * g.gw;
  const int per = (ghw + 2 * blockDim.x - 1) / (2 * blockDim.x);   // blocks per item
  const int item = i0 + blockIdx.x / per, part = blockIdx.x % per;
  if (item >= i1) return;
  const float lmax = __uint_as_float(peak[item - i0]);
  const float scale = lmax > 0.f ? (float)(32767.0 / (double)lmax) : 1.0f;
  const float2* Fi = Fo + (size_t)(item - i0) * ghw;
  int16_t* fro = p.fr + (size_t)item * ghw;
  int16_t* fio = p.fi + (size_t)item * ghw;
  for (int i = part * 2 * blockDim.x + threadIdx.x; i < min(ghw, (part + 1) * 2 * (int)blockDim.x); i += blockDim.x) {
    const float2 v = Fi[i];
    fro[i] = (int16_t)__float2int_rn(__fmul_rn(v.x, scale));
    fio[i] = (int16_t)__float2int_rn(__fmul_rn(v.y, scale));
    if (p.raw) p.raw[(size_t)item * ghw + i] = v;
  }
  if (part == 0 && threadIdx.x == 0) p.scale[item] = scale;
}

bool lw_supported(const Geometry& g, int A, const void* members, unsigned flags, const void* windows) {
  const size_t cols_smem = 2ull * kLwCols * g.ny * sizeof(float2);
  const size_t rows_smem = 2ull * kLwRows * g.nx * sizeof(float2);
  const size_t field_smem = (2ull * g.gw + 160) * kLwFRows * sizeof(float2);
  const bool coefs_fit = g.G == 0 || ((size_t)g.gh * g.gw + (size_t)g.gh * g.G) * sizeof(float2) <= 200 * 1024;
  return A == 1 && members == nullptr && g.mode == 1 && g.gh == g.wh && g.gw == g.ww && g.nx >= 256 &&
         g.ny >= 256 && (flags & 1u) == 0 && windows == nullptr && cols_smem <= 200 * 1024 &&
         rows_smem <= 200 * 1024 && field_smem <= 200 * 1024 && 2ull * kLwCols * g.gh * sizeof(float2) <= cols_smem &&
         (2ull * g.gh + 160) * kLwIfft * sizeof(float2) <= 200 * 1024 &&
         coefs_fit;
}

int64_t lw_chunk(const Geometry& g) {   // items per chunk: R + T + F of a chunk within ~80 MB of L2
  const int64_t per = (int64_t)g.ww * g.ny * 8 + 2 * (int64_t)g.gh * g.gw * 8 + 4;
  return std::max<int64_t>(1, (80ll << 20) / per);
}

// kLwLanes slots of 1/kLwLanes of an L2 chunk each, processed on as many internal streams so that one slot's
// kernels fill the tail waves of the others'.
constexpr int kLwLanes = 3;
int64_t lw_slot_items(const Geometry& g, int64_t items) {
  const int64_t half = std::max<int64_t>(1, (lw_chunk(g) + kLwLanes - 1) / kLwLanes);
  return std::max<int64_t>(1, std::min<int64_t>(items, half));
}
static size_t lw_slot_bytes(const Geometry& g, int64_t items) {
  const size_t b = (size_t)lw_slot_items(g, items) * ((size_t)g.ww * g.ny * 8 + 2 * (size_t)g.gh * g.gw * 8 + 16);
  return (b + 255) & ~size_t(255);
}

size_t lw_workspace(const Geometry& g, int64_t items) { return kLwLanes * lw_slot_bytes(g, items) + 1024; }

cudaError_t launch_coefs(const RunParams& p, int grid, cudaStream_t s);

cudaError_t launch_lw(const RunParams& p, int num_sms, cudaStream_t s) {
  const Geometry& g = p.g;
  const int items = p.B * g.P;
  const int64_t chunk = lw_slot_items(g, items);
  const int64_t n0 = chunk;
  const size_t slot_bytes = lw_slot_bytes(g, items);
  for (const void* k : {(const void*)lw_rows_kernel, (const void*)lw_cols_kernel, (const void*)lw_field_kernel<true>,
                        (const void*)lw_field_kernel<false>, (const void*)lw_rows512_kernel,
                        (const void*)lw_cols512_kernel<false>, (const void*)lw_cols512_kernel<true>,
                        (const void*)lw_ifft_y_kernel<true>, (const void*)lw_ifft_y_kernel<false>}) {
    const cudaError_t e = ensure_smem_optin(k, 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int rows_smem = 2 * kLwRows * g.nx * (int)sizeof(float2);
  const int cols_smem = 2 * kLwCols * g.ny * (int)sizeof(float2);
  const int field_smem = (2 * g.gw + 160) * kLwFRows * (int)sizeof(float2);
  // fork onto two internal streams (one per workspace slot) and join back onto s: stream-ordered for the caller
  constexpr int kMaxDev = 64;
  static cudaStream_t lanes_of[kMaxDev][kLwLanes] = {};
  static cudaEvent_t fork_of[kMaxDev] = {}, join_of[kMaxDev][kLwLanes] = {};
  static std::mutex lanes_mu;
  const bool two = items > chunk;
  int dev = 0;
  cudaGetDevice(&dev);
  if (two && (dev < 0 || dev >= kMaxDev)) return cudaErrorInvalidDevice;
  // the lanes and events of a device are shared: one launch enqueues fork .. join at a time
  std::unique_lock<std::mutex> lk(lanes_mu, std::defer_lock);
  if (two) {
    lk.lock();
    if (!fork_of[dev]) {   // created once per device, reused by every later launch
      for (int k = 0; k < kLwLanes; ++k) {
        cudaStreamCreateWithFlags(&lanes_of[dev][k], cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&join_of[dev][k], cudaEventDisableTiming);
      }
      cudaEventCreateWithFlags(&fork_of[dev], cudaEventDisableTiming);
    }
  }
  cudaStream_t* lanes = two ? lanes_of[dev] : nullptr;
  cudaEvent_t fork_ev = two ? fork_of[dev] : nullptr;
  cudaEvent_t* join_ev = two ? join_of[dev] : nullptr;
  if (two) {
    cudaEventRecord(fork_ev, s);
    for (int k = 0; k < kLwLanes; ++k) cudaStreamWaitEvent(lanes[k], fork_ev, 0);
  }
  int slot = 0;
  for (int i0 = 0; i0 < items; i0 += (int)chunk, slot = (slot + 1) % kLwLanes) {
    const int i1 = (int)std::min<int64_t>(items, i0 + chunk);
    const int n = i1 - i0;
    cudaStream_t s_ = two ? lanes[slot] : s;
    float2* R = reinterpret_cast<float2*>(p.work + slot * slot_bytes);
    float2* T = R + (size_t)n0 * g.ww * g.ny;
    float2* F = T + (size_t)n0 * g.gh * g.gw;
    unsigned* peak = reinterpret_cast<unsigned*>(F + (size_t)n0 * g.gh * g.gw);
    cudaMemsetAsync(peak, 0, (size_t)n * sizeof(unsigned), s_);
    if (g.nx == 512 && g.ny == 512) {
      const int f512 = 8 * kF512Group * (int)sizeof(float2);
      lw_rows512_kernel<<<n * (g.ny / 2 / (8 * kRows512Sets)), 512, f512, s_>>>(p, i0, i1, R);
      if (g.gh == 164 && g.wh == 164) {   // column FFT, crop and the 164-point IFFT along r in one kernel
        lw_cols512_kernel<true><<<n * ((g.ww + 7) / 8), 512, f512, s_>>>(p, i0, i1, R, T);
      } else {
        lw_cols512_kernel<false><<<n * ((g.ww + 7) / 8), 512, f512, s_>>>(p, i0, i1, R, F);   // window -> F (scratch)
        const int ys = (2 * g.gh + 160) * kLwIfft * (int)sizeof(float2);
        if (g.gh == 164)
          lw_ifft_y_kernel<true><<<n * ((g.ww + kLwIfft - 1) / kLwIfft), kThreads, ys, s_>>>(p, i0, i1, F, T);
        else
          lw_ifft_y_kernel<false><<<n * ((g.ww + kLwIfft - 1) / kLwIfft), kThreads, ys, s_>>>(p, i0, i1, F, T);
      }
    } else {
      lw_rows_kernel<<<n * ((g.ny / 2 + kLwRows - 1) / kLwRows), kThreads, rows_smem, s_>>>(p, i0, i1, R);
      lw_cols_kernel<<<n * ((g.ww + kLwCols - 1) / kLwCols), kThreads, cols_smem, s_>>>(p, i0, i1, R, T);
    }
    if (g.gw == 164)
      lw_field_kernel<true><<<n * ((g.gh + kLwFRows - 1) / kLwFRows), kThreads, field_smem, s_>>>(p, i0, i1, T, F, peak);
    else
      lw_field_kernel<false><<<n * ((g.gh + kLwFRows - 1) / kLwFRows), kThreads, field_smem, s_>>>(p, i0, i1, T, F, peak);
    const int per = (g.gh * g.gw + 2 * kThreads - 1) / (2 * kThreads);
    lw_pack_kernel<<<n * per, kThreads, 0, s_>>>(p, i0, i1, F, peak);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      if (two)   // still join, so the caller's stream never runs ahead of queued work
        for (int k = 0; k < kLwLanes; ++k) {
          cudaEventRecord(join_ev[k], lanes[k]);
          cudaStreamWaitEvent(s, join_ev[k], 0);
        }
      return e;
    }
  }
  if (two) {
    for (int k = 0; k < kLwLanes; ++k) {
      cudaEventRecord(join_ev[k], lanes[k]);
      cudaStreamWaitEvent(s, join_ev[k], 0);
    }
    lk.unlock();
  }
  if (p.coefs && g.G > 0) {
    const int grid = (int)std::min<int64_t>(items, (int64_t)num_sms * 4);
    return launch_coefs(p, grid, s);
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_fused(const RunParams& p, cudaStream_t s) {
  if (p.lay.slab_bytes > 0)   // large windows: latency-bound on the global slab, more warps per CTA
    fused_kernel<512><<<p.lay.grid, 512, p.lay.smem_bytes, s>>>(p);
  else
    fused_kernel<kThreads><<<p.lay.grid, kThreads, p.lay.smem_bytes, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_finalize(const RunParams& p, float* total, cudaStream_t s) {
  PlaneArgs a{};
  a.P = p.g.P; a.h = p.g.gh; a.w = p.g.gw;
  a.xa = p.t.xad; a.ya = p.t.yad;
  a.params = p.params; a.slots = p.param_slots;
  a.agg = p.work + p.lay.agg_off; a.agg_per_cta = p.lay.agg_per_cta;
  a.total = total; a.agg_slot = p.B; a.nblocks = p.lay.grid;
  plane_finalize_kernel<<<p.g.P, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_plane_summary(const float2* data, int64_t count, int P, int h, int w, const double* xa,
                                 const double* ya, float* params, int slots, float* total, double* pol_total,
                                 char* work, int grid, cudaStream_t s) {
  PlaneArgs a{};
  a.pol_total = pol_total;
  a.data = data; a.count = count; a.P = P; a.h = h; a.w = w; a.xa = xa; a.ya = ya;
  a.params = params; a.slots = slots; a.agg = work;
  a.agg_per_cta = ((int64_t)P * h * w * 8 + 255) / 256 * 256;
  a.total = total; a.agg_slot = (int)count; a.nblocks = grid;
  plane_stats_kernel<<<grid, kThreads, 0, s>>>(a);
  plane_finalize_kernel<<<P, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_coefs(const RunParams& p, int grid, cudaStream_t s) {
  const int smem = (p.g.gh * p.g.gw + p.g.gh * p.g.G) * (int)sizeof(float2);
  coefs_kernel<<<grid, kThreads, smem, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_fourier_full(const RunParams& p, int64_t F, float2* plane, cudaStream_t s) {
  fourier_full_kernel<<<p.lay.grid, kThreads, p.lay.smem_bytes, s>>>(p, F, plane);
  return cudaGetLastError();
}
template <typename K>
static cudaError_t raise_smem(K kernel) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - (int)fa.sharedSizeBytes);
}
cudaError_t set_smem_limits() {
  cudaError_t e = raise_smem(fused_kernel<kThreads>);
  if (e != cudaSuccess) return e;
  e = raise_smem(fused_kernel<512>);
  if (e != cudaSuccess) return e;
  e = raise_smem(fourier_full_kernel);
  if (e != cudaSuccess) return e;
  return raise_smem(coefs_kernel);
}

}  // namespace holo
