// Shared-memory mixed-radix FFT building blocks for sm_100a.
//
// Complex values are float2 (x = Re, y = Im).  A "stage table" is W_n^i =
// exp(-2 pi i * i / n) for i in [0, n) (forward sign), computed on the host in
// fp64 and rounded to float32; inverse transforms conjugate it on the fly.
//
// The batched Stockham stage below is the generic workhorse: it works on
// shared memory or on global scratch (generic pointers), any transform length,
// any element/sequence stride, radices 2..16 unrolled in registers and any
// other prime through a table-driven O(p^2) butterfly.  The register-resident
// fast paths for the hot window sizes live in holo_fused.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HOLO_DEV __device__ __forceinline__

HOLO_DEV float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
HOLO_DEV float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
HOLO_DEV float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
HOLO_DEV float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
HOLO_DEV float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
HOLO_DEV float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// multiply by -i (forward) or +i (inverse)
template <bool INV> HOLO_DEV float2 rot90(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}
template <bool INV> HOLO_DEV float2 twid(float2 w) { return INV ? cconj(w) : w; }

// ------------------------------------------------------------ butterflies
// In-register DFT of length P with sign -1 (forward) or +1 (INV); in place.

template <bool INV> HOLO_DEV void dft2(float2& a, float2& b) {
  float2 t = csub(a, b);
  a = cadd(a, b);
  b = t;
}

template <bool INV> HOLO_DEV void dft3(float2& x0, float2& x1, float2& x2) {
  const float s3 = 0.86602540378443864676f;
  float2 t1 = cadd(x1, x2);
  float2 d = csub(x1, x2);
  float2 m = make_float2(fmaf(-0.5f, t1.x, x0.x), fmaf(-0.5f, t1.y, x0.y));
  x0 = cadd(x0, t1);
  float2 r = rot90<INV>(cscale(d, s3));  // -i*s3*d (fwd)
  x1 = cadd(m, r);
  x2 = csub(m, r);
}

template <bool INV> HOLO_DEV void dft4(float2& x0, float2& x1, float2& x2, float2& x3) {
  float2 a = cadd(x0, x2), b = csub(x0, x2);
  float2 c = cadd(x1, x3), d = rot90<INV>(csub(x1, x3));
  x0 = cadd(a, c);
  x2 = csub(a, c);
  x1 = cadd(b, d);
  x3 = csub(b, d);
}

// odd length via conjugate-symmetric pairs; C[j] = cos(2 pi j/P), S[j] = sin(2 pi j/P)
template <int P, bool INV> HOLO_DEV void dft_odd(float2* x, const float* C, const float* S) {
  constexpr int H = (P - 1) / 2;
  float2 sp[H], sm[H];
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    sp[j - 1] = cadd(x[j], x[P - j]);
    sm[j - 1] = csub(x[j], x[P - j]);
  }
  float2 x0 = x[0];
  float2 tot = x0;
#pragma unroll
  for (int j = 0; j < H; ++j) tot = cadd(tot, sp[j]);
#pragma unroll
  for (int t = 1; t <= H; ++t) {
    float2 re = x0, im = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      int k = (j * t) % P;
      float c = C[k], s = S[k];
      re.x = fmaf(c, sp[j - 1].x, re.x);
      re.y = fmaf(c, sp[j - 1].y, re.y);
      im.x = fmaf(s, sm[j - 1].x, im.x);
      im.y = fmaf(s, sm[j - 1].y, im.y);
    }
    // forward: X_t = re - i*im ; X_{P-t} = re + i*im
    float2 r = rot90<INV>(im);
    x[t] = cadd(re, r);
    x[P - t] = csub(re, r);
  }
  x[0] = tot;
}

template <bool INV> HOLO_DEV void dft5(float2* x) {
  const float C[5] = {1.f, 0.30901699437494742f, -0.80901699437494742f, -0.80901699437494742f,
                      0.30901699437494742f};
  const float S[5] = {0.f, 0.95105651629515357f, 0.58778525229247313f, -0.58778525229247313f,
                      -0.95105651629515357f};
  dft_odd<5, INV>(x, C, S);
}

template <bool INV> HOLO_DEV void dft7(float2* x) {
  const float C[7] = {1.f, 0.62348980185873353f, -0.22252093395631440f, -0.90096886790241913f,
                      -0.90096886790241913f, -0.22252093395631440f, 0.62348980185873353f};
  const float S[7] = {0.f, 0.78183148246802981f, 0.97492791218182361f, 0.43388373911755812f,
                      -0.43388373911755812f, -0.97492791218182361f, -0.78183148246802981f};
  dft_odd<7, INV>(x, C, S);
}

template <bool INV> HOLO_DEV void dft6(float2* x) {
  // 6 = 2 x 3: even outputs from sums, odd outputs from twiddled differences
  const float c = 0.5f, s = 0.86602540378443864676f;
  float2 a0 = cadd(x[0], x[3]), a1 = cadd(x[1], x[4]), a2 = cadd(x[2], x[5]);
  float2 b0 = csub(x[0], x[3]), b1 = csub(x[1], x[4]), b2 = csub(x[2], x[5]);
  // w6^1 = c - i s (fwd), w6^2 = -c - i s (fwd)
  float2 w1 = make_float2(c, INV ? s : -s), w2 = make_float2(-c, INV ? s : -s);
  b1 = cmul(b1, w1);
  b2 = cmul(b2, w2);
  dft3<INV>(a0, a1, a2);
  dft3<INV>(b0, b1, b2);
  x[0] = a0; x[2] = a1; x[4] = a2;
  x[1] = b0; x[3] = b1; x[5] = b2;
}

template <bool INV> HOLO_DEV void dft8(float2* x) {
  const float r = 0.70710678118654752440f;
  // s = b + 2a ; t = c + 4d
  float2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
  float2 o0 = x[1], o1 = x[3], o2 = x[5], o3 = x[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  // o_c *= w8^c
  o1 = cmul(o1, make_float2(r, INV ? r : -r));
  o2 = rot90<INV>(o2);
  o3 = cmul(o3, make_float2(-r, INV ? r : -r));
  x[0] = cadd(e0, o0); x[4] = csub(e0, o0);
  x[1] = cadd(e1, o1); x[5] = csub(e1, o1);
  x[2] = cadd(e2, o2); x[6] = csub(e2, o2);
  x[3] = cadd(e3, o3); x[7] = csub(e3, o3);
}

template <bool INV> HOLO_DEV void dft16(float2* x) {
  // s = b + 4a, t = c + 4d: DFT4 over a, twiddle w16^{bc}, DFT4 over b
  const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f;
  const float r = 0.70710678118654752440f;
  float2 y[16];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    float2 a0 = x[b], a1 = x[b + 4], a2 = x[b + 8], a3 = x[b + 12];
    dft4<INV>(a0, a1, a2, a3);
    y[b * 4 + 0] = a0; y[b * 4 + 1] = a1; y[b * 4 + 2] = a2; y[b * 4 + 3] = a3;
  }
  const float sg = INV ? 1.f : -1.f;
  // twiddles w16^{bc}, b,c in 1..3
  y[1 * 4 + 1] = cmul(y[5], make_float2(c1, sg * s1));
  y[1 * 4 + 2] = cmul(y[6], make_float2(r, sg * r));
  y[1 * 4 + 3] = cmul(y[7], make_float2(s1, sg * c1));
  y[2 * 4 + 1] = cmul(y[9], make_float2(r, sg * r));
  y[2 * 4 + 2] = rot90<INV>(y[10]);
  y[2 * 4 + 3] = cmul(y[11], make_float2(-r, sg * r));
  y[3 * 4 + 1] = cmul(y[13], make_float2(s1, sg * c1));
  y[3 * 4 + 2] = cmul(y[14], make_float2(-r, sg * r));
  y[3 * 4 + 3] = cmul(y[15], make_float2(-c1, -sg * s1));
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float2 b0 = y[c], b1 = y[4 + c], b2 = y[8 + c], b3 = y[12 + c];
    dft4<INV>(b0, b1, b2, b3);
    x[c] = b0; x[c + 4] = b1; x[c + 8] = b2; x[c + 12] = b3;
  }
}

template <int P, bool INV> HOLO_DEV void dft_fixed(float2* x) {
  if constexpr (P == 2) dft2<INV>(x[0], x[1]);
  else if constexpr (P == 3) dft3<INV>(x[0], x[1], x[2]);
  else if constexpr (P == 4) dft4<INV>(x[0], x[1], x[2], x[3]);
  else if constexpr (P == 5) dft5<INV>(x);
  else if constexpr (P == 6) dft6<INV>(x);
  else if constexpr (P == 7) dft7<INV>(x);
  else if constexpr (P == 8) dft8<INV>(x);
  else if constexpr (P == 16) dft16<INV>(x);
}

// ------------------------------------------------------- Stockham stage
// Data layout: element e of sequence q at base[q*sstride + e*estride].
// Stage with radix P, current sub-length L (product of earlier radices):
//   m_in = n/L, m' = m_in/P; task (q', k), q' < m', k < L:
//   read  A[(k*m_in + q' + m'*s)]  * W_n^{s*k*m'},  DFT_P over s,
//   write B[((k + L*t)*m' + q')]                         (self-sorting).

struct FFTPlan {
  int n;
  int nst;          // number of stages
  int radix[8];
  const float2* tw; // W_n^i, i < n
};

template <int P, bool INV>
HOLO_DEV void stockham_stage_fixed(const float2* src, float2* dst, int n, int L, int count,
                                   int sstride, int estride, const float2* tw, int tid,
                                   int nthr) {
  const int m_in = n / L, mp = m_in / P;
  const int per = n / P;
  const int total = count * per;
  const bool seq_fast = (sstride == 1 && estride != 1);
  for (int task = tid; task < total; task += nthr) {
    int q, r;
    if (seq_fast) { q = task % count; r = task / count; }
    else { q = task / per; r = task - q * per; }
    const int k = r / mp, qp = r - k * mp;
    const float2* s = src + (size_t)q * sstride;
    float2* d = dst + (size_t)q * sstride;
    float2 v[P];
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = s[(size_t)(k * m_in + qp + mp * j) * estride];
    if (L > 1) {
#pragma unroll
      for (int j = 1; j < P; ++j) v[j] = cmul(v[j], twid<INV>(tw[(j * k * mp) % n]));
    }
    dft_fixed<P, INV>(v);
#pragma unroll
    for (int t = 0; t < P; ++t) d[(size_t)((k + L * t) * mp + qp) * estride] = v[t];
  }
}

template <bool INV>
HOLO_DEV void stockham_stage_generic(const float2* src, float2* dst, int n, int L, int P,
                                     int count, int sstride, int estride, const float2* tw,
                                     int tid, int nthr) {
  // odd prime radix P: inputs loaded and twiddled once, then the conjugate-pair
  // DFT (same algebra as dft_odd) with the W_P powers read from the W_n table
  constexpr int PMAX = 128;
  const int m_in = n / L, mp = m_in / P;
  const int per = n / P;
  const int total = count * per;
  const int np = n / P;  // W_P^{e} = W_n^{e * n/P}
  const int H = (P - 1) / 2;
  for (int task = tid; task < total; task += nthr) {
    const int q = task / per, r = task - q * per;
    const int k = r / mp, qp = r - k * mp;
    const float2* s = src + (size_t)q * sstride;
    float2* d = dst + (size_t)q * sstride;
    if (P <= PMAX && (P & 1)) {
      float2 sp[PMAX / 2], sm[PMAX / 2];
      float2 v0 = s[(size_t)(k * m_in + qp) * estride];
      float2 tot = v0;
      int e1 = 0, e2 = 0;  // (j k mp) mod n and ((P-j) k mp) mod n, updated incrementally
      const int stepw = (k * mp) % n;
      e2 = (P * stepw) % n;
      for (int j = 1; j <= H; ++j) {
        e1 += stepw; if (e1 >= n) e1 -= n;
        e2 -= stepw; if (e2 < 0) e2 += n;
        float2 a = s[(size_t)(k * m_in + qp + mp * j) * estride];
        float2 b = s[(size_t)(k * m_in + qp + mp * (P - j)) * estride];
        if (L > 1) {
          a = cmul(a, twid<INV>(tw[e1]));
          b = cmul(b, twid<INV>(tw[e2]));
        }
        sp[j - 1] = cadd(a, b);
        sm[j - 1] = csub(a, b);
        tot = cadd(tot, sp[j - 1]);
      }
      d[(size_t)(k * mp + qp) * estride] = tot;
      for (int t = 1; t <= H; ++t) {
        float2 re = v0, im = make_float2(0.f, 0.f);
        int e = 0;
        for (int j = 1; j <= H; ++j) {
          e += t; if (e >= P) e -= P;
          const float2 w = tw[e * np];            // cos(2 pi e/P) - i sin(2 pi e/P)
          const float c = w.x, sn = -w.y;
          re.x = fmaf(c, sp[j - 1].x, re.x);
          re.y = fmaf(c, sp[j - 1].y, re.y);
          im.x = fmaf(sn, sm[j - 1].x, im.x);
          im.y = fmaf(sn, sm[j - 1].y, im.y);
        }
        const float2 rr = rot90<INV>(im);
        d[(size_t)((k + L * t) * mp + qp) * estride] = cadd(re, rr);
        d[(size_t)((k + L * (P - t)) * mp + qp) * estride] = csub(re, rr);
      }
      continue;
    }
    for (int t = 0; t < P; ++t) {   // any other radix: direct O(P^2)
      float2 acc = make_float2(0.f, 0.f);
      for (int j = 0; j < P; ++j) {
        float2 v = s[(size_t)(k * m_in + qp + mp * j) * estride];
        int e = ((j * k * mp) % n + ((j * t) % P) * np) % n;
        float2 w = twid<INV>(tw[e]);
        acc.x = fmaf(v.x, w.x, fmaf(-v.y, w.y, acc.x));
        acc.y = fmaf(v.x, w.y, fmaf(v.y, w.x, acc.y));
      }
      d[(size_t)((k + L * t) * mp + qp) * estride] = acc;
    }
  }
}

// cos / sin (2 pi e / 41): constant-cache operands of the radix-41 stage (164 = 4 x 41 field grids)
__constant__ float kCos41[41] = {1.000000000e+00f, 9.882804238e-01f, 9.533963921e-01f, 8.961655570e-01f, 8.179293608e-01f, 7.205215936e-01f, 6.062254110e-01f, 4.777198185e-01f, 3.380168784e-01f, 1.903911092e-01f, 3.830273369e-02f, -1.146834254e-01f, -2.649815022e-01f, -4.090686372e-01f, -5.435675500e-01f, -6.653257002e-01f, -7.714891798e-01f, -8.595696070e-01f, -9.275024511e-01f, -9.736954239e-01f, -9.970658012e-01f, -9.970658012e-01f, -9.736954239e-01f, -9.275024511e-01f, -8.595696070e-01f, -7.714891798e-01f, -6.653257002e-01f, -5.435675500e-01f, -4.090686372e-01f, -2.649815022e-01f, -1.146834254e-01f, 3.830273369e-02f, 1.903911092e-01f, 3.380168784e-01f, 4.777198185e-01f, 6.062254110e-01f, 7.205215936e-01f, 8.179293608e-01f, 8.961655570e-01f, 9.533963921e-01f, 9.882804238e-01f};
__constant__ float kSin41[41] = {0.000000000e+00f, 1.526492842e-01f, 3.017205986e-01f, 4.437198379e-01f, 5.753186602e-01f, 6.934325008e-01f, 7.952928713e-01f, 8.785122509e-01f, 9.411400480e-01f, 9.817083200e-01f, 9.992661811e-01f, 9.934020898e-01f, 9.642534955e-01f, 9.125036165e-01f, 8.393654261e-01f, 7.465532216e-01f, 6.362424423e-01f, 5.110186794e-01f, 3.738170718e-01f, 2.278535089e-01f, 7.654925284e-02f, -7.654925284e-02f, -2.278535089e-01f, -3.738170718e-01f, -5.110186794e-01f, -6.362424423e-01f, -7.465532216e-01f, -8.393654261e-01f, -9.125036165e-01f, -9.642534955e-01f, -9.934020898e-01f, -9.992661811e-01f, -9.817083200e-01f, -9.411400480e-01f, -8.785122509e-01f, -7.952928713e-01f, -6.934325008e-01f, -5.753186602e-01f, -4.437198379e-01f, -3.017205986e-01f, -1.526492842e-01f};

// Runs every stage of `plan` (block-cooperative, __syncthreads between stages).
// Ping-pongs between a and b; returns the buffer that holds the result.
template <bool INV>
__device__ float2* stockham(float2* a, float2* b, const FFTPlan& plan, int count, int sstride,
                            int estride) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  float2 *src = a, *dst = b;
  int L = 1;
  for (int st = 0; st < plan.nst; ++st) {
    const int P = plan.radix[st];
    switch (P) {
      case 2: stockham_stage_fixed<2, INV>(src, dst, plan.n, L, count, sstride, estride, plan.tw, tid, nthr); break;
      case 3: stockham_stage_fixed<3, INV>(src, dst, plan.n, L, count, sstride, estride, plan.tw, tid, nthr); break;
      case 4: stockham_stage_fixed<4, INV>(src, dst, plan.n, L, count, sstride, estride, plan.tw, tid, nthr); break;
      case 5: stockham_stage_fixed<5, INV>(src, dst, plan.n, L, count, sstride, estride, plan.tw, tid, nthr); break;
      case 6: stockham_stage_fixed<6, INV>(src, dst, plan.n, L, count, sstride, estride, plan.tw, tid, nthr); break;
      case 7: stockham_stage_fixed<7, INV>(src, dst, plan.n, L, count, sstride, estride, plan.tw, tid, nthr); break;
      case 8: stockham_stage_fixed<8, INV>(src, dst, plan.n, L, count, sstride, estride, plan.tw, tid, nthr); break;
      case 16: stockham_stage_fixed<16, INV>(src, dst, plan.n, L, count, sstride, estride, plan.tw, tid, nthr); break;
      default: stockham_stage_generic<INV>(src, dst, plan.n, L, P, count, sstride, estride, plan.tw, tid, nthr); break;
    }
    __syncthreads();
    L *= P;
    float2* t = src; src = dst; dst = t;
  }
  return src;
}
