// C ABI (include/holo_b200.h): plan construction in fp64 on the host, device
// table upload, workspace sizing and kernel launches.  No exceptions cross the
// boundary; every entry point returns an hpg_status.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <map>
#include <mutex>
#include <tuple>

#include <cuda_fp16.h>

#include "../../include/holo_b200.h"
#include "holo_internal.h"

namespace holo {
cudaError_t launch_fused(const RunParams& p, cudaStream_t s);
cudaError_t launch_finalize(const RunParams& p, float* total, cudaStream_t s);
cudaError_t launch_coefs(const RunParams& p, int grid, cudaStream_t s);
cudaError_t launch_fourier_full(const RunParams& p, int64_t F, float2* plane, cudaStream_t s);
cudaError_t set_smem_limits();
bool fast_supported(const Geometry& g, int A, int fmt, int transpose, int fill, const void* rcal,
                    unsigned flags, const void* windows);
cudaError_t launch_fast(const RunParams& p, const FastTables& ft, int num_sms, cudaStream_t s);
bool tc_supported(const Geometry& g, int A, int fmt, int transpose, int fill, const void* rcal, unsigned flags,
                  const void* windows);
cudaError_t launch_fast_tc(const RunParams& p, const FastTables& ft, int num_sms, cudaStream_t s);
bool tc2_supported(const Geometry& g, int A, int fmt, int transpose, int fill, const void* rcal, unsigned flags,
                   const void* windows);
size_t tc2_workspace(int64_t items);
bool lw_supported(const Geometry& g, int A, const void* members, unsigned flags, const void* windows);
size_t lw_workspace(const Geometry& g, int64_t items);
int64_t lw_chunk(const Geometry& g);
int64_t lw_slot_items(const Geometry& g, int64_t items);
int64_t tc2_chunk();
cudaError_t launch_lw(const RunParams& p, int num_sms, cudaStream_t s);
cudaError_t launch_tc2(const RunParams& p, const FastTables& ft, int num_sms, cudaStream_t s);
cudaError_t launch_plane_summary(const float2* data, int64_t count, int P, int h, int w, const double* xa,
                                 const double* ya, float* params, int slots, float* total, double* pol_total,
                                 char* work, int grid, cudaStream_t s);
cudaError_t launch_field_intensity(const int16_t* fr, const int16_t* fi, const float* scale, int B, int P, int hw,
                                   double* out, cudaStream_t s);
cudaError_t launch_refcal_finish(const float2* a, const float2* b, int64_t n, float2* out, cudaStream_t s);
}  // namespace holo

using namespace holo;

static thread_local std::string g_last_error;

// Device blocks of destroyed plans, handed to later plans of the same size on the same device.
// AutoAlign builds a plan per evaluation (holopipe/align.py:25-29 re-runs the pipeline with new
// parameters); cudaMalloc + cudaFree of the table block cost ~0.6 ms per evaluation, several times
// the evaluation itself.  A block is pooled only after the device is idle (cudaFree semantics).
static std::mutex g_pool_mu;
static std::vector<std::tuple<int, size_t, void*>> g_pool;
constexpr size_t kPoolMax = 64;

static cudaError_t pool_alloc(int device, size_t bytes, void** p) {
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (size_t i = 0; i < g_pool.size(); ++i)
      if (std::get<0>(g_pool[i]) == device && std::get<1>(g_pool[i]) == bytes) {
        *p = std::get<2>(g_pool[i]);
        g_pool.erase(g_pool.begin() + (std::ptrdiff_t)i);
        return cudaSuccess;
      }
  }
  return cudaMalloc(p, bytes);
}

static void pool_free(int device, size_t bytes, void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (g_pool.size() < kPoolMax) g_pool.emplace_back(device, bytes, p);
  else cudaFree(p);
}
namespace holo {
cudaError_t ensure_smem_optin(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{dev, func}];
  if (bytes <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}
}  // namespace holo

static thread_local int g_last_launches = 0;   // kernels the last hpg_run on this thread launched

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
static int cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? HPG_MEMORYALLOCATION : HPG_ERROR;
}

struct hpg_plan {
  Geometry g;
  double xi[2][2] = {{0, 0}, {0, 0}};   // fractional beam centre in window pixels (engine.py:147-150)
  void* tc_dev = nullptr;              // tensor-core DFT matrices (lazy)
  DevTables t;
  FastTables ft{};
  int fill = 0;
  void* dev = nullptr;         // one allocation for every table
  size_t dev_bytes = 0, tc_bytes = 0;
  std::vector<float> xa, ya;   // host copies of the axes
  std::vector<float> hx, hy;   // host copies of the dequantised basis
  int device = 0;
  int num_sms = 148;
};

namespace {

constexpr double kPi = 3.14159265358979323846;

double radians(double deg) { return deg * (kPi / 180.0); }

// round half to even, like Python's round() and numpy.rint
long long rint_even(double v) { return (long long)std::nearbyint(v); }

double sinc(double x) {
  if (x == 0.0) return 1.0;
  const double y = kPi * x;
  return std::sin(y) / y;
}

int radix_plan(int n, int* radix) {
  int e2 = 0, m = n;
  while (m % 2 == 0) { m /= 2; ++e2; }
  int e3 = 0;
  while (m % 3 == 0) { m /= 3; ++e3; }
  std::vector<int> r;
  while (e2 >= 4) { r.push_back(16); e2 -= 4; }
  if (e2 == 3) r.push_back(8);
  else if (e2 == 2) r.push_back(4);
  else if (e2 == 1) {
    if (e3 > 0) { r.push_back(6); --e3; }
    else r.push_back(2);
  }
  for (; e3 > 0; --e3) r.push_back(3);
  for (int p : {5, 7}) while (m % p == 0) { r.push_back(p); m /= p; }
  for (int p = 11; m > 1; p += 2)
    while (m % p == 0) { r.push_back(p); m /= p; }
  if (r.empty()) r.push_back(1);
  if (r.size() > 8) return -1;
  for (size_t i = 0; i < 8; ++i) radix[i] = i < r.size() ? r[i] : 1;
  return n == 1 ? 0 : (int)r.size();
}

void twiddles(int n, std::vector<float2>& out) {
  for (int i = 0; i < n; ++i) {
    const double a = 2.0 * kPi * (double)i / (double)n;
    out.push_back(make_float2((float)std::cos(a), (float)(-std::sin(a))));
  }
}

// Normalised Hermite-Gaussian profiles (holopipe/hgbasis.py:42-70), fp64.
std::vector<double> hg_profiles(int G, const std::vector<float>& axis, double waist) {
  const size_t n = axis.size();
  std::vector<double> h((size_t)G * n);
  const double s2 = std::sqrt(2.0), c0 = std::pow(kPi, -0.25);
  for (size_t i = 0; i < n; ++i) {
    const double u = s2 * ((double)axis[i] - 0.0) / waist;
    double hp = c0 * std::exp(-0.5 * u * u);
    h[i] = hp;
    if (G > 1) {
      double hc = s2 * u * hp;
      h[n + i] = hc;
      for (int k = 2; k < G; ++k) {
        const double hn = std::sqrt(2.0 / k) * u * hc - std::sqrt((k - 1.0) / k) * hp;
        h[(size_t)k * n + i] = hn;
        hp = hc;
        hc = hn;
      }
    }
  }
  const double d = n > 1 ? std::fabs((double)axis[1] - (double)axis[0]) : 1.0;
  for (int k = 0; k < G; ++k) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += h[(size_t)k * n + i] * h[(size_t)k * n + i];
    double nrm = std::sqrt(s * d);
    if (nrm == 0.0) nrm = 1.0;
    for (size_t i = 0; i < n; ++i) h[(size_t)k * n + i] /= nrm;
  }
  return h;
}

// int16 quantisation + float32 dequantisation of the profiles (hgbasis.py:84-93).
void quantised_basis(int G, const std::vector<float>& axis, double waist, float* out,
                     std::vector<int16_t>* q16 = nullptr, std::vector<float>* scales = nullptr) {
  const std::vector<double> h = hg_profiles(G, axis, waist);
  const size_t n = axis.size();
  if (q16) q16->assign((size_t)G * n, 0);
  if (scales) scales->assign(G, 1.f);
  for (int k = 0; k < G; ++k) {
    double mx = 0.0;
    for (size_t i = 0; i < n; ++i) mx = std::fmax(mx, std::fabs(h[(size_t)k * n + i]));
    const float scale = 32767.0f / (float)mx;
    if (scales) (*scales)[k] = scale;
    for (size_t i = 0; i < n; ++i) {
      const double qv = std::nearbyint(h[(size_t)k * n + i] * (double)scale);
      const int16_t q = (int16_t)qv;
      out[(size_t)k * n + i] = (float)q / scale;
      if (q16) (*q16)[(size_t)k * n + i] = q;
    }
  }
}

// Tensor-core overlap operand (holo_fast.cu, TCO): int16 basis q = 32 (q >> 5) + (q & 31) split into
// two exactly-representable fp16 parts, in the UMMA K-major layout [row/8][kstep 3][khalf][row%8][8],
// rows = orders (GP16 = G rounded up to 16), K = the 42 axis samples padded to 48.
void tco_image(const std::vector<int16_t>& q, int G, int GP16, int n, uint16_t* hi, uint16_t* lo) {
  for (int m = 0; m < GP16; ++m)
    for (int k = 0; k < 48; ++k) {
      const int v = (m < G && k < n) ? q[(size_t)m * n + k] : 0;
      const size_t e = ((size_t)(m >> 3) * 3 + (k >> 4)) * 128 + (size_t)((k >> 3) & 1) * 64 + (m & 7) * 8 + (k & 7);
      hi[e] = __half_as_ushort(__float2half((float)(32 * (v >> 5))));
      lo[e] = __half_as_ushort(__float2half((float)(v & 31)));
    }
}

template <typename T>
size_t push(std::vector<char>& blob, const std::vector<T>& v) {
  size_t off = (blob.size() + 255) & ~size_t(255);
  blob.resize(off + v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
  return off;
}

int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// Shared-memory / workspace placement of the fused kernel's buffers.
Layout make_layout(const hpg_plan* P, int B, int A, unsigned flags, bool full_plane) {
  const Geometry& g = P->g;
  Layout L{};
  const int64_t f2 = sizeof(float2);
  const int cols = full_plane ? g.nx / 2 + 1 : g.ww;
  int64_t nR = (int64_t)cols * g.ny;
  int64_t nS = std::max<int64_t>((int64_t)g.gh * g.gw, (int64_t)g.gh * std::max(g.G, 1));
  nS = std::max<int64_t>(nS, (int64_t)std::min(g.ny / 2, 16) * g.nx);
  nS = std::max<int64_t>(nS, (int64_t)std::min(cols, 16) * g.ny);
  if (full_plane) nS = std::max<int64_t>((int64_t)std::min(g.ny / 2, 16) * g.nx, (int64_t)std::min(cols, 16) * g.ny);
  L.CH = (int)std::max<int64_t>(1, std::min<int64_t>(g.ny / 2, nS / g.nx));
  L.CC = (int)std::max<int64_t>(1, std::min<int64_t>(cols, nS / g.ny));
  const int64_t nW = full_plane ? 0 : (int64_t)g.wh * g.ww;
  const int64_t nG = (!full_plane && (g.gh != g.wh || g.gw != g.ww)) ? (int64_t)g.gh * g.gw : 0;
  const int64_t nAcc = (!full_plane && A > 1) ? 2 * (int64_t)g.wh * g.ww : 0;  // double2
  struct Item { Region* r; int64_t bytes; };
  Item items[] = {{&L.S0, nS * f2}, {&L.S1, nS * f2}, {&L.Wt, nW * f2}, {&L.R, nR * f2},
                  {&L.Gd, nG * f2}, {&L.Acc, nAcc * f2}};
  const int64_t budget = 200 * 1024;  // < 227 KB opt-in minus static reduction buffers
  int64_t total = 0;
  for (auto& it : items) total += align_up(it.bytes, 256);
  int64_t soff = 0, goff = 0;
  for (auto& it : items) {
    const int64_t b = align_up(it.bytes, 256);
    if (total <= budget || soff + b <= budget) {
      it.r->in_smem = 1;
      it.r->off = soff;
      soff += b;
    } else {
      it.r->in_smem = 0;
      it.r->off = goff;
      goff += b;
    }
  }
  L.smem_bytes = (int)soff;
  L.slab_bytes = goff;
  return L;
}

}  // namespace

// Tensor-core DFT matrices of a plan (row DFT A1 for holo_fast_tc.cu / holo_tc2.cu, column DFT A2 for
// holo_tc2.cu), fp16 hi + lo, computed in fp64 on first use so that plans created for the SIMT
// kernels (e.g. one per AutoAlign evaluation) do not pay for them.
static cudaError_t ensure_tc_tables(const hpg_plan* Pc) {
  hpg_plan* P = const_cast<hpg_plan*>(Pc);
  if (P->tc_dev) return cudaSuccess;
  const Geometry& g = P->g;
  const double (&xi)[2][2] = P->xi;
  // Both tables are stored column-major, [pol][hi | lo][column (f16x2)][row n], so that a warp loading its
  // 32 TMEM lanes reads 32 consecutive words per instruction.
  // tensor-core row DFT (holo_fast_tc.cu): A[n][x], n < 64 -> Re, n >= 64 -> Im of
  // exp(-2 pi i kx_c x / nx) * px[c] = exp(-2 pi i kx_c (x - xi_x + nx/2) / nx), c = n mod 64,
  // split into fp16 hi + lo; rows c >= ww are zero.  Only for nx == 128, wavelength 0.
  std::vector<uint32_t> a_tc;
  if (g.nx == 128 && g.ww <= 64) {
    a_tc.assign((size_t)g.P * 2 * 128 * 64, 0u);
    for (int q = 0; q < g.P; ++q) {
      const int kx = g.k0[q][0][0];
      for (int n = 0; n < 128; ++n) {
        const int c = n & 63;
        if (c >= g.ww) continue;
        const double kc = (double)(kx + c - g.ww / 2);
        for (int x2 = 0; x2 < 64; ++x2) {
          uint16_t hh[2], ll[2];
          for (int e = 0; e < 2; ++e) {
            const int x = 2 * x2 + e;
            const double ang = -2.0 * kPi * kc * ((double)x - xi[q][0] + g.nx / 2.0) / g.nx;
            const double v = n < 64 ? std::cos(ang) : std::sin(ang);
            const __half h = __double2half(v);
            const __half l = __double2half(v - (double)__half2float(h));
            hh[e] = __half_as_ushort(h);
            ll[e] = __half_as_ushort(l);
          }
          a_tc[(((size_t)q * 2 + 0) * 64 + x2) * 128 + n] = (uint32_t)hh[0] | ((uint32_t)hh[1] << 16);
          a_tc[(((size_t)q * 2 + 1) * 64 + x2) * 128 + n] = (uint32_t)ll[0] | ((uint32_t)ll[1] << 16);
        }
      }
    }
  }
  if (a_tc.empty()) a_tc.push_back(0u);
  // the same matrix with packed, interleaved rows for the two-kernel path (holo_tc2.cu): row 2c -> Re, 2c + 1 -> Im;
  // the fill-factor envelope (pipeline.py:99-103; separable inside the Nyquist band, see the fast-path tables
  // in hpg_plan_create) is folded into the rows here and into the rows of the column-DFT matrix below
  auto env = [&](int k, int n) {   // 1 / sinc of the signed bin k of an n-point axis
    if (!P->fill) return 1.0;
    int t = k % n;
    if (t < 0) t += n;
    return 1.0 / sinc((double)(t <= n / 2 ? t : n - t) / n);
  };
  std::vector<uint32_t> a_tcp;
  if (g.nx == 128 && g.ww <= 64) {
    a_tcp.assign((size_t)g.P * 2 * 128 * 64, 0u);
    for (int q = 0; q < g.P; ++q) {
      const int kx = g.k0[q][0][0];
      for (int n = 0; n < 2 * g.ww; ++n) {
        const int c = n >> 1;
        const double kc = (double)(kx + c - g.ww / 2), ex = env(kx + c - g.ww / 2, g.nx);
        for (int x2 = 0; x2 < 64; ++x2) {
          uint16_t hh[2], ll[2];
          for (int e = 0; e < 2; ++e) {
            const int x = 2 * x2 + e;
            const double ang = -2.0 * kPi * kc * ((double)x - xi[q][0] + g.nx / 2.0) / g.nx;
            const double v = ((n & 1) ? std::sin(ang) : std::cos(ang)) * ex;
            const __half h = __double2half(v);
            const __half l = __double2half(v - (double)__half2float(h));
            hh[e] = __half_as_ushort(h);
            ll[e] = __half_as_ushort(l);
          }
          a_tcp[(((size_t)q * 2 + 0) * 64 + x2) * 128 + n] = (uint32_t)hh[0] | ((uint32_t)hh[1] << 16);
          a_tcp[(((size_t)q * 2 + 1) * 64 + x2) * 128 + n] = (uint32_t)ll[0] | ((uint32_t)ll[1] << 16);
        }
      }
    }
  }
  if (a_tcp.empty()) a_tcp.push_back(0u);
  // tensor-core column DFT (holo_tc2.cu): rows r < wh -> Cr, rows 64 + r -> Ci of
  // C[r][y] = exp(-2 pi i ky_r y / ny) * py[r] = exp(-2 pi i ky_r (y - xi_y + ny/2) / ny),
  // ky_r = k0y + r - wh/2; K = y (0..127), fp16 hi + lo.  ny == 128, wh <= 64, wavelength 0.
  std::vector<uint32_t> a2_tc;
  if (g.ny == 128 && g.wh <= 64) {
    a2_tc.assign((size_t)g.P * 2 * 128 * 64, 0u);
    for (int q = 0; q < g.P; ++q) {
      const int ky = g.k0[q][0][1];
      for (int n = 0; n < 128; ++n) {
        const int r = n & 63;
        if (r >= g.wh) continue;
        const double kr = (double)(ky + r - g.wh / 2);
        for (int y2 = 0; y2 < 64; ++y2) {
          uint16_t hh[2], ll[2];
          for (int e = 0; e < 2; ++e) {
            const int y = 2 * y2 + e;
            const double ang = -2.0 * kPi * kr * ((double)y - xi[q][1] + g.ny / 2.0) / g.ny;
            const double v = n < 64 ? std::cos(ang) : std::sin(ang);
            const __half h = __double2half(v);
            const __half l = __double2half(v - (double)__half2float(h));
            hh[e] = __half_as_ushort(h);
            ll[e] = __half_as_ushort(l);
          }
          a2_tc[(((size_t)q * 2 + 0) * 64 + y2) * 128 + n] = (uint32_t)hh[0] | ((uint32_t)hh[1] << 16);
          a2_tc[(((size_t)q * 2 + 1) * 64 + y2) * 128 + n] = (uint32_t)ll[0] | ((uint32_t)ll[1] << 16);
        }
      }
    }
  }
  if (a2_tc.empty()) a2_tc.push_back(0u);
  // column DFT as the B operand of holo_tc2.cu's column GEMM (the data, the row-DFT accumulator converted to
  // fp16 in TMEM, is the A operand): B[n][y] in the canonical K-major no-swizzle shared-memory layout,
  // rows n < 48 -> Cr[r = n][y], rows 48 + r -> Ci[r][y] (zero for r >= wh), hi part then lo part,
  // [kstep 8][row/8 12][khalf 2][row%8 8][8 halves] = 24 KB per part.
  std::vector<uint16_t> c2_tc;
  if (g.ny == 128 && g.wh <= 48) {
    const size_t part = 8 * 12 * 2 * 8 * 8;   // halves per part
    c2_tc.assign((size_t)g.P * 2 * part, 0);
    for (int q = 0; q < g.P; ++q) {
      const int ky = g.k0[q][0][1];
      for (int n = 0; n < 96; ++n) {
        const int r = n % 48;
        if (r >= g.wh) continue;
        const double kr = (double)(ky + r - g.wh / 2), ey = env(ky + r - g.wh / 2, g.ny);
        for (int y = 0; y < 128; ++y) {
          const double ang = -2.0 * kPi * kr * ((double)y - xi[q][1] + g.ny / 2.0) / g.ny;
          const double v = (n < 48 ? std::cos(ang) : std::sin(ang)) * ey;
          const __half h = __double2half(v);
          const __half l = __double2half(v - (double)__half2float(h));
          const size_t off = (size_t)(y >> 4) * (12 * 128) + ((size_t)(n >> 3) * 2 + ((y >> 3) & 1)) * 64 +
                             (size_t)(n & 7) * 8 + (y & 7);   // kmaj_off in halves
          c2_tc[((size_t)q * 2 + 0) * part + off] = __half_as_ushort(h);
          c2_tc[((size_t)q * 2 + 1) * part + off] = __half_as_ushort(l);
        }
      }
    }
  }
  if (c2_tc.empty()) c2_tc.push_back(0);
  std::vector<char> blob;
  const size_t o1 = push(blob, a_tc), o2 = push(blob, a2_tc), o3 = push(blob, c2_tc), o4 = push(blob, a_tcp);
  cudaError_t e = pool_alloc(P->device, blob.size(), &P->tc_dev);
  if (e != cudaSuccess) { P->tc_dev = nullptr; return e; }
  P->tc_bytes = blob.size();
  e = cudaMemcpy(P->tc_dev, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  P->ft.a_tc = reinterpret_cast<const uint32_t*>(static_cast<char*>(P->tc_dev) + o1);
  P->ft.a2_tc = reinterpret_cast<const uint32_t*>(static_cast<char*>(P->tc_dev) + o2);
  P->ft.a_tcp = reinterpret_cast<const uint32_t*>(static_cast<char*>(P->tc_dev) + o4);
  P->ft.c2_tc = reinterpret_cast<const uint4*>(static_cast<char*>(P->tc_dev) + o3);
  return cudaSuccess;
}

extern "C" {

int hpg_version(void) { return 1; }

const char* hpg_last_error(void) { return g_last_error.c_str(); }

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static const bool g_plan_timing = getenv("HOLO_PLAN_TIMING") != nullptr;

int hpg_plan_create(const hpg_plan_desc* d, hpg_plan** out) {
  const double t_start = g_plan_timing ? now_us() : 0.0;
  if (!d || !out) return fail(HPG_NULLPOINTER, "null argument");
  *out = nullptr;
  if (d->pol_count < 1 || d->pol_count > 2) return fail(HPG_INVALIDPOLARISATION, "pol_count");
  if (d->fft_nx < 2 || d->fft_ny < 2 || (d->fft_ny & 1) || d->frame_width < 1 || d->frame_height < 1)
    return fail(HPG_INVALIDDIMENSION, "window dimensions");
  if (d->wavelength_count < 1 || d->wavelength_count > kMaxWl || !d->wavelengths)
    return fail(HPG_INVALIDARGUMENT, "wavelength_count");
  if (d->pixel_size <= 0 || d->wavelength_centre <= 0) return fail(HPG_INVALIDARGUMENT, "pixel/wavelength");
  if (d->group_count < 0) return fail(HPG_INVALIDARGUMENT, "group_count");
  hpg_plan* P = new (std::nothrow) hpg_plan();
  if (!P) return fail(HPG_MEMORYALLOCATION, "host allocation");
  Geometry& g = P->g;
  std::memset(&g, 0, sizeof(g));
  g.W = d->frame_width;
  g.H = d->frame_height;
  g.P = d->pol_count;
  g.nx = d->fft_nx;
  g.ny = d->fft_ny;
  g.mode = d->resolution_mode;
  g.L = d->wavelength_count;
  g.G = d->group_count;
  g.M = g.G * (g.G + 1) / 2;
  const double p = d->pixel_size;
  // window box (holopipe/pipeline.py:62-69)
  const double fr = std::sin(radians(d->window_radius_deg)) / d->wavelength_centre;
  g.ww = (int)std::min<long long>(2 * ((long long)std::floor(fr * g.nx * p) + 1), g.nx);
  g.wh = (int)std::min<long long>(2 * ((long long)std::floor(fr * g.ny * p) + 1), g.ny);
  if (g.ww < 2 || g.wh < 2) { delete P; return fail(HPG_INVALIDDIMENSION, "window radius too small"); }
  if (g.mode == 0) { g.gh = g.ny; g.gw = g.nx; }
  else { g.gh = g.wh; g.gw = g.ww; }
  if (g.gw & 1 || g.gh & 1) { delete P; return fail(HPG_INVALIDDIMENSION, "odd IFFT grid"); }
  // window origins (pipeline.py:23-44) and fractional centres (engine.py:147-150)
  double xi[2][2];
  for (int q = 0; q < g.P; ++q) {
    int x0 = 0, x1 = g.W;
    if (g.P == 2) { x0 = q == 0 ? 0 : g.W / 2; x1 = q == 0 ? g.W / 2 : g.W; }
    if (g.nx > x1 - x0 || g.ny > g.H) { delete P; return fail(HPG_INVALIDDIMENSION, "fft window does not fit the frame region"); }
    const double xc = d->beam_centre[0][q] / p + g.W / 2.0;
    const double yc = d->beam_centre[1][q] / p + g.H / 2.0;
    long long c0 = rint_even(xc) - g.nx / 2, r0 = rint_even(yc) - g.ny / 2;
    c0 = std::min<long long>(std::max<long long>(c0, x0), x1 - g.nx);
    r0 = std::min<long long>(std::max<long long>(r0, 0), g.H - g.ny);
    g.col0[q] = (int)c0;
    g.row0[q] = (int)r0;
    xi[q][0] = d->beam_centre[0][q] / p + g.W / 2.0 - c0;
    xi[q][1] = d->beam_centre[1][q] / p + g.H / 2.0 - r0;
  }
  // carrier bins (engine.py:191-194)
  for (int q = 0; q < g.P; ++q)
    for (int w = 0; w < g.L; ++w) {
      const double lam = d->wavelengths[w];
      g.k0[q][w][0] = (int)rint_even(std::sin(radians(d->tilt_deg[0][q])) * g.nx * p / lam);
      g.k0[q][w][1] = (int)rint_even(std::sin(radians(d->tilt_deg[1][q])) * g.ny * p / lam);
    }
  // field axes (pipeline.py:152-160)
  P->xa.resize(g.gw);
  P->ya.resize(g.gh);
  for (int i = 0; i < g.gw; ++i)
    P->xa[i] = g.mode == 0 ? (float)((double)(i - g.nx / 2) * p)
                           : (float)((double)(i - g.ww / 2) * p * ((double)g.nx / g.ww));
  for (int i = 0; i < g.gh; ++i)
    P->ya[i] = g.mode == 0 ? (float)((double)(i - g.ny / 2) * p)
                           : (float)((double)(i - g.wh / 2) * p * ((double)g.ny / g.wh));
  g.dx = g.gw > 1 ? std::fabs((double)P->xa[1] - (double)P->xa[0]) : 1.0;
  g.dy = g.gh > 1 ? std::fabs((double)P->ya[1] - (double)P->ya[0]) : 1.0;
  for (int q = 0; q < g.P; ++q) g.dxdy[q] = (float)(g.dx * g.dy);
  // FFT plans
  g.nst_nx = radix_plan(g.nx, g.radix_nx);
  g.nst_ny = radix_plan(g.ny, g.radix_ny);
  g.nst_gw = radix_plan(g.gw, g.radix_gw);
  g.nst_gh = radix_plan(g.gh, g.radix_gh);
  if (g.nst_nx < 0 || g.nst_ny < 0 || g.nst_gw < 0 || g.nst_gh < 0) { delete P; return fail(HPG_INVALIDDIMENSION, "FFT size"); }

  std::vector<float2> tw_nx, tw_ny, tw_gw, tw_gh;
  twiddles(g.nx, tw_nx); twiddles(g.ny, tw_ny); twiddles(g.gw, tw_gw); twiddles(g.gh, tw_gh);
  // window table: mask * recentring phase (/ sinc envelope)  (pipeline.py:72-127)
  const int whw = g.wh * g.ww;
  std::vector<float2> wtab((size_t)g.P * g.L * whw);
  std::vector<float2> remx((size_t)g.P * g.L * g.gw), remy((size_t)g.P * g.L * g.gh);
  for (int q = 0; q < g.P; ++q)
    for (int w = 0; w < g.L; ++w) {
      const int kx = g.k0[q][w][0], ky = g.k0[q][w][1];
      const double lam = d->wavelengths[w];
      float2* T = &wtab[((size_t)q * g.L + w) * whw];
      // the recentring phase is separable: one cos / sin per column and per row (same fp64 values)
      std::vector<double> cxr(g.ww), cxi(g.ww);
      for (int c = 0; c < g.ww; ++c) {
        const double tx = (double)(kx + c - g.ww / 2);
        const double ax = 2.0 * kPi * tx * (xi[q][0] - g.nx / 2.0) / g.nx;
        cxr[c] = std::cos(ax);
        cxi[c] = std::sin(ax);
      }
      for (int r = 0; r < g.wh; ++r) {
        const double dfy = (double)(r - g.wh / 2) / (g.ny * p);
        const double ty = (double)(ky + r - g.wh / 2);
        const double ay = 2.0 * kPi * ty * (xi[q][1] - g.ny / 2.0) / g.ny;
        const double pyr = std::cos(ay), pyi = std::sin(ay);
        for (int c = 0; c < g.ww; ++c) {
          const double dfx = (double)(c - g.ww / 2) / (g.nx * p);
          const bool in = dfy * dfy + dfx * dfx <= fr * fr + 1e-30;
          // product of the two separable phases in complex128 (pipeline.py:125-127)
          const double pxr = cxr[c], pxi = cxi[c];
          const double re = pyr * pxr - pyi * pxi;
          const double im = pyr * pxi + pyi * pxr;
          // complex64 cast, then the mask (bool * c64)
          float fre = in ? (float)re : 0.f, fim = in ? (float)im : 0.f;
          if (d->fill_factor) {
            int txm = (kx + c - g.ww / 2) % g.nx; if (txm < 0) txm += g.nx;
            int tym = (ky + r - g.wh / 2) % g.ny; if (tym < 0) tym += g.ny;
            const int sx = txm <= g.nx / 2 ? txm : g.nx - txm;
            const double fyw = (double)(tym > g.ny / 2 ? tym - g.ny : tym) / g.ny;
            double env = sinc(fyw) * sinc((double)sx / g.nx);
            if (std::fabs(env) < 1e-3) env = 1e-3;
            const float fe = (float)env;
            fre = fre / fe;
            fim = fim / fe;
          }
          T[(size_t)r * g.ww + c] = make_float2(fre, fim);
        }
      }
      // removal phase, separable (pipeline.py:163-185), with ifftshift sign
      // (-1)^(x+y) and the 1/(nx*ny) inverse normalisation (pipeline.py:146-149)
      const double fxl = std::sin(radians(d->removal_tilt_deg[0][q])) / lam;
      const double fyl = std::sin(radians(d->removal_tilt_deg[1][q])) / lam;
      const double rx = fxl - kx / (g.nx * p), ry = fyl - ky / (g.ny * p);
      const double cst = 2.0 * kPi * (fxl * d->removal_beam_centre[0][q] + fyl * d->removal_beam_centre[1][q]) -
                         kPi * (kx + ky);
      const double quad = kPi * d->defocus[q] / lam;
      const double norm = 1.0 / ((double)g.nx * g.ny);
      for (int x = 0; x < g.gw; ++x) {
        const double xv = (double)P->xa[x];
        const double ph = 2.0 * kPi * rx * xv + quad * xv * xv;
        const double sg = (x & 1) ? -1.0 : 1.0;
        remx[((size_t)q * g.L + w) * g.gw + x] = make_float2((float)(sg * std::cos(ph)), (float)(-sg * std::sin(ph)));
      }
      for (int y = 0; y < g.gh; ++y) {
        const double yv = (double)P->ya[y];
        const double ph = cst + 2.0 * kPi * ry * yv + quad * yv * yv;
        const double sg = ((y & 1) ? -1.0 : 1.0) * norm;
        remy[((size_t)q * g.L + w) * g.gh + y] = make_float2((float)(sg * std::cos(ph)), (float)(-sg * std::sin(ph)));
      }
    }
  // basis (hgbasis.py:76-93); centre 0, waist per pol
  const int G = std::max(g.G, 0);
  P->hx.assign((size_t)g.P * G * g.gw, 0.f);
  P->hy.assign((size_t)g.P * G * g.gh, 0.f);
  std::vector<int16_t> mm, mn;
  const int GP16 = std::max(16, (G + 15) & ~15);
  const bool tco_ok = G > 0 && GP16 <= 48 && g.gw == 42 && g.gh == 42;
  const size_t tco_part = (size_t)GP16 * 48;   // halves per operand part
  std::vector<uint16_t> tco_img(tco_ok ? (size_t)g.P * 4 * tco_part : 1, 0);
  std::vector<float> tco_inv(tco_ok ? (size_t)g.P * 2 * GP16 : 1, 0.f);
  if (G > 0) {
    for (int q = 0; q < g.P; ++q) {
      if (!(d->waist[q] > 0)) { delete P; return fail(HPG_INVALIDDIMENSION, "basis waist must be positive"); }
      std::vector<int16_t> qx, qy;
      std::vector<float> sx, sy;
      quantised_basis(G, P->xa, d->waist[q], &P->hx[(size_t)q * G * g.gw], &qx, &sx);
      quantised_basis(G, P->ya, d->waist[q], &P->hy[(size_t)q * G * g.gh], &qy, &sy);
      if (tco_ok) {
        uint16_t* img = &tco_img[(size_t)q * 4 * tco_part];
        tco_image(qx, G, GP16, g.gw, img, img + tco_part);
        tco_image(qy, G, GP16, g.gh, img + 2 * tco_part, img + 3 * tco_part);
        for (int m = 0; m < G; ++m) {
          tco_inv[((size_t)q * 2 + 0) * GP16 + m] = 1.f / sx[m];
          tco_inv[((size_t)q * 2 + 1) * GP16 + m] = 1.f / sy[m];
        }
      }
    }
    for (int gg = 0; gg < G; ++gg)
      for (int m = gg; m >= 0; --m) { mm.push_back((int16_t)m); mn.push_back((int16_t)(gg - m)); }
  } else {
    mm.push_back(0); mn.push_back(0);
  }
  // fast-path tables (holo_fast.cu): separable recentring phases and the
  // circular mask as a row range per column
  std::vector<float2> pxv((size_t)g.P * g.L * g.ww), pyv((size_t)g.P * g.L * g.wh);
  std::vector<int16_t> crange((size_t)g.ww * 2);
  for (int q = 0; q < g.P; ++q)
    for (int w = 0; w < g.L; ++w) {
      const size_t pl = (size_t)q * g.L + w;
      const int kx = g.k0[q][w][0], ky = g.k0[q][w][1];
      for (int c = 0; c < g.ww; ++c) {
        const double ax = 2.0 * kPi * (double)(kx + c - g.ww / 2) * (xi[q][0] - g.nx / 2.0) / g.nx;
        // fill-factor envelope (pipeline.py:99-103) folded in: sinc(fx) sinc(fy) >= (2/pi)^2 inside
        // the Nyquist band, so the 1e-3 floor never binds and the envelope is separable
        double ex = 1.0;
        if (d->fill_factor) {
          int txm = (kx + c - g.ww / 2) % g.nx; if (txm < 0) txm += g.nx;
          ex = sinc((double)(txm <= g.nx / 2 ? txm : g.nx - txm) / g.nx);
        }
        pxv[pl * g.ww + c] = make_float2((float)(std::cos(ax) / ex), (float)(std::sin(ax) / ex));
      }
      for (int r = 0; r < g.wh; ++r) {
        const double ay = 2.0 * kPi * (double)(ky + r - g.wh / 2) * (xi[q][1] - g.ny / 2.0) / g.ny;
        double ey = 1.0;
        if (d->fill_factor) {
          int tym = (ky + r - g.wh / 2) % g.ny; if (tym < 0) tym += g.ny;
          ey = sinc((double)(tym > g.ny / 2 ? tym - g.ny : tym) / g.ny);
        }
        pyv[pl * g.wh + r] = make_float2((float)(std::cos(ay) / ey), (float)(std::sin(ay) / ey));
      }
    }
  for (int c = 0; c < g.ww; ++c) {
    const double dfx = (double)(c - g.ww / 2) / (g.nx * p);
    int lo = g.wh, hi = -1;
    for (int r = 0; r < g.wh; ++r) {
      const double dfy = (double)(r - g.wh / 2) / (g.ny * p);
      if (dfy * dfy + dfx * dfx <= fr * fr + 1e-30) { lo = std::min(lo, r); hi = std::max(hi, r); }
    }
    crange[2 * c] = (int16_t)lo;
    crange[2 * c + 1] = (int16_t)hi;
  }
  for (int q = 0; q < 2; ++q) { P->xi[q][0] = xi[q][0]; P->xi[q][1] = xi[q][1]; }
  P->fill = d->fill_factor;
  std::vector<char> blob;
  const size_t o_px = push(blob, pxv), o_py = push(blob, pyv), o_cr = push(blob, crange), o_unused = 0;
  const size_t o_timg = push(blob, tco_img), o_tinv = push(blob, tco_inv);
  const size_t o_nx = push(blob, tw_nx), o_ny = push(blob, tw_ny), o_gw = push(blob, tw_gw), o_gh = push(blob, tw_gh);
  const size_t o_w = push(blob, wtab), o_rx = push(blob, remx), o_ry = push(blob, remy);
  std::vector<float> hxv = P->hx, hyv = P->hy;
  if (hxv.empty()) hxv.push_back(0.f);
  if (hyv.empty()) hyv.push_back(0.f);
  const size_t o_hx = push(blob, hxv), o_hy = push(blob, hyv);
  // half tables of the register-resident tail (holo_tailr.cu): [pol][x | y][22 rows: axis index 0, then
  // n/2 .. n-1][16 orders], transposed and zero-padded, for 42-point axes and at most 16 orders
  std::vector<float> half_tab;
  if (G > 0 && G <= 16 && g.gw == 42 && g.gh == 42) {
    half_tab.assign((size_t)g.P * 2 * 22 * 16, 0.f);
    for (int q = 0; q < g.P; ++q)
      for (int ax = 0; ax < 2; ++ax)
        for (int j = 0; j < 22; ++j)
          for (int m = 0; m < G; ++m) {
            const int x = j == 0 ? 0 : 20 + j;
            half_tab[(((size_t)q * 2 + ax) * 22 + j) * 16 + m] = (ax == 0 ? P->hx : P->hy)[((size_t)q * G + m) * 42 + x];
          }
  }
  const bool half_ok = !half_tab.empty();
  if (half_tab.empty()) half_tab.push_back(0.f);
  const size_t o_half = push(blob, half_tab);
  const size_t o_xa = push(blob, P->xa), o_ya = push(blob, P->ya);
  std::vector<double> xad(P->xa.begin(), P->xa.end()), yad(P->ya.begin(), P->ya.end());
  const size_t o_xad = push(blob, xad), o_yad = push(blob, yad);
  const size_t o_mm = push(blob, mm), o_mn = push(blob, mn);
  const double t_host = g_plan_timing ? now_us() : 0.0;
  cudaGetDevice(&P->device);
  cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, P->device);
  cudaError_t e = pool_alloc(P->device, blob.size(), &P->dev);
  const double t_alloc = g_plan_timing ? now_us() : 0.0;
  if (e != cudaSuccess) { delete P; return cuda_fail(e, "cudaMalloc(plan tables)"); }
  P->dev_bytes = blob.size();
  e = cudaMemcpy(P->dev, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(P->dev); delete P; return cuda_fail(e, "cudaMemcpy(plan tables)"); }
  char* base = static_cast<char*>(P->dev);
  P->t.tw_nx = reinterpret_cast<const float2*>(base + o_nx);
  P->t.tw_ny = reinterpret_cast<const float2*>(base + o_ny);
  P->t.tw_gw = reinterpret_cast<const float2*>(base + o_gw);
  P->t.tw_gh = reinterpret_cast<const float2*>(base + o_gh);
  P->t.win_tab = reinterpret_cast<const float2*>(base + o_w);
  P->t.rem_x = reinterpret_cast<const float2*>(base + o_rx);
  P->t.rem_y = reinterpret_cast<const float2*>(base + o_ry);
  P->t.hx = reinterpret_cast<const float*>(base + o_hx);
  P->t.hy = reinterpret_cast<const float*>(base + o_hy);
  P->t.xa = reinterpret_cast<const float*>(base + o_xa);
  P->t.ya = reinterpret_cast<const float*>(base + o_ya);
  P->t.xad = reinterpret_cast<const double*>(base + o_xad);
  P->t.yad = reinterpret_cast<const double*>(base + o_yad);
  P->t.mode_m = reinterpret_cast<const int16_t*>(base + o_mm);
  P->t.mode_n = reinterpret_cast<const int16_t*>(base + o_mn);
  P->ft.px = reinterpret_cast<const float2*>(base + o_px);
  P->ft.py = reinterpret_cast<const float2*>(base + o_py);
  P->ft.crange = reinterpret_cast<const int16_t*>(base + o_cr);
  (void)o_unused;
  P->ft.a_tc = nullptr;    // tensor-core DFT matrices: built on first use (ensure_tc_tables)
  P->ft.a2_tc = nullptr;
  P->ft.c2_tc = nullptr;
  P->ft.tco_img = tco_ok ? reinterpret_cast<const uint4*>(base + o_timg) : nullptr;
  P->ft.tco_inv = reinterpret_cast<const float*>(base + o_tinv);
  P->ft.tco_gp = tco_ok ? GP16 : 0;
  // HG parity on the symmetric part of the field axes (pipeline.py:152-160 puts the origin at index w / 2),
  // verified bit for bit on the quantised profiles: the fast kernel then folds each +-d pair of the overlap
  P->ft.half_tab = half_ok ? reinterpret_cast<const float*>(base + o_half) : nullptr;
  P->ft.hsym = 0;
  for (int q = 0; q < g.P && G > 0; ++q) {
    for (int ax = 0; ax < 2; ++ax) {
      const int n = ax == 0 ? g.gw : g.gh;
      const float* h = ax == 0 ? &P->hx[(size_t)q * G * n] : &P->hy[(size_t)q * G * n];
      const int c = n / 2;
      bool sym = true;
      for (int m = 0; m < G && sym; ++m)
        for (int dd = 1; c + dd < n && sym; ++dd)
          sym = h[(size_t)m * n + c - dd] == ((m & 1) ? -h[(size_t)m * n + c + dd] : h[(size_t)m * n + c + dd]);
      if (sym) P->ft.hsym |= 1 << (2 * q + ax);
    }
  }
  const double t_copy = g_plan_timing ? now_us() : 0.0;
  e = set_smem_limits();
  if (g_plan_timing)
    fprintf(stderr, "hpg_plan_create: host %.0f us, malloc %.0f us, copy %.0f us (%zu B), smem limits %.0f us\n",
            t_host - t_start, t_alloc - t_host, t_copy - t_alloc, blob.size(), now_us() - t_copy);
  if (e != cudaSuccess) { cudaFree(P->dev); delete P; return cuda_fail(e, "cudaFuncSetAttribute"); }
  *out = P;
  return HPG_SUCCESS;
}

int hpg_plan_destroy(hpg_plan* P) {
  if (!P) return fail(HPG_NULLPOINTER, "null plan");
  if (P->dev || P->tc_dev) {
    // kernels still in flight may read the tables: wait for the plan's device like cudaFree would
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != P->device) cudaSetDevice(P->device);
    cudaDeviceSynchronize();
    if (cur != P->device && cur >= 0) cudaSetDevice(cur);
    pool_free(P->device, P->dev_bytes, P->dev);
    pool_free(P->device, P->tc_bytes, P->tc_dev);
  }
  delete P;
  return HPG_SUCCESS;
}

int hpg_plan_get_info(const hpg_plan* P, hpg_plan_info* info) {
  if (!P || !info) return fail(HPG_NULLPOINTER, "null argument");
  std::memset(info, 0, sizeof(*info));
  const Geometry& g = P->g;
  info->wh = g.wh; info->ww = g.ww; info->gh = g.gh; info->gw = g.gw;
  info->mode_count = g.M;
  for (int q = 0; q < 2; ++q) {
    info->col0[q] = g.col0[q];
    info->row0[q] = g.row0[q];
    for (int w = 0; w < kMaxWl; ++w) {
      info->k0[q][w][0] = g.k0[q][w][0];
      info->k0[q][w][1] = g.k0[q][w][1];
    }
  }
  return HPG_SUCCESS;
}

int hpg_plan_get_axes(const hpg_plan* P, float* x, float* y) {
  if (!P || !x || !y) return fail(HPG_NULLPOINTER, "null argument");
  std::memcpy(x, P->xa.data(), P->xa.size() * sizeof(float));
  std::memcpy(y, P->ya.data(), P->ya.size() * sizeof(float));
  return HPG_SUCCESS;
}

int hpg_plan_get_basis(const hpg_plan* P, float* hx, float* hy) {
  if (!P || !hx || !hy) return fail(HPG_NULLPOINTER, "null argument");
  std::memcpy(hx, P->hx.data(), P->hx.size() * sizeof(float));
  std::memcpy(hy, P->hy.data(), P->hy.size() * sizeof(float));
  return HPG_SUCCESS;
}

static int grid_for(const hpg_plan* P, const Layout& L, int64_t items, const void* kernel_tag) {
  (void)kernel_tag;
  int per_sm = L.smem_bytes <= 100 * 1024 ? 2 : 1;
  int64_t grid = (int64_t)P->num_sms * per_sm;
  if (items < grid) grid = items;
  return (int)std::max<int64_t>(grid, 1);
}

static void finish_layout(const hpg_plan* P, Layout& L, int64_t items, unsigned flags) {
  L.grid = grid_for(P, L, items, nullptr);
  L.agg_off = align_up(L.slab_bytes * L.grid, 256);
  L.agg_per_cta = (flags & HPG_FLAG_SUMMARY) ? align_up((int64_t)P->g.P * P->g.gh * P->g.gw * 8, 256) : 0;
}

int hpg_workspace_size(const hpg_plan* P, int32_t B, uint32_t flags, size_t* bytes) {
  if (!P || !bytes) return fail(HPG_NULLPOINTER, "null argument");
  Layout L = make_layout(P, B, 2, flags, false);  // worst case: averaging enabled
  finish_layout(P, L, (int64_t)B * P->g.P, flags);
  const int64_t fused = L.agg_off + L.agg_per_cta * L.grid;
  Layout F = make_layout(P, B, 1, 0, true);
  finish_layout(P, F, (int64_t)P->num_sms * 2, 0);
  *bytes = (size_t)std::max<int64_t>(std::max<int64_t>(fused, F.slab_bytes * F.grid), 256);
  *bytes = std::max(*bytes, tc2_workspace((int64_t)B * P->g.P));   // Fourier windows between the TC2 kernels
  if (lw_supported(P->g, 1, nullptr, flags, nullptr))                  // large-window path intermediates
    *bytes = std::max(*bytes, lw_workspace(P->g, (int64_t)B * P->g.P));
  return HPG_SUCCESS;
}

static int fill_params(const hpg_plan* P, const hpg_batch* b, const hpg_outputs* o, unsigned flags,
                       RunParams& rp) {
  std::memset(&rp, 0, sizeof(rp));
  rp.g = P->g;
  rp.t = P->t;
  rp.frames = b->frames;
  rp.fmt = b->frame_format;
  rp.transpose = b->transpose;
  rp.B = b->batch_count;
  rp.A = std::max(1, b->avg_count);
  rp.members = b->members;
  rp.wl = b->wl_of_row;
  rp.bcal = static_cast<const float2*>(b->batch_cal);
  rp.cal_pols = b->cal_pols;
  rp.cal_batch = b->cal_batch;
  rp.row_offset = b->row_offset;
  rp.rcal = static_cast<const float2*>(b->ref_cal);
  rp.rcal_count = std::max(1, b->ref_cal_count);
  rp.flags = flags;
  if (b->layout_width > 0) {
    rp.g.W = b->layout_width;
    rp.g.H = b->layout_height;
    for (int q = 0; q < P->g.P; ++q) {
      rp.g.col0[q] = b->layout_col0[q];
      rp.g.row0[q] = b->layout_row0[q];
    }
  }
  if (o) {
    rp.fr = o->field_r;
    rp.fi = o->field_i;
    rp.scale = o->field_scale;
    rp.coefs = static_cast<float2*>(o->coefs);
    rp.raw = static_cast<float2*>(o->raw_fields);
    rp.windows = static_cast<float2*>(o->windows);
    rp.params = o->field_params;
    rp.param_slots = o->param_slots;
    rp.work = static_cast<char*>(o->workspace);
  }
  return HPG_SUCCESS;
}

int hpg_last_launch_count(void) { return g_last_launches; }

int hpg_run(const hpg_plan* P, const hpg_batch* b, const hpg_outputs* o, uint32_t flags, void* stream) {
  g_last_launches = 0;
  if (!P || !b || !o) return fail(HPG_NULLPOINTER, "null argument");
  if (!b->frames || !o->field_r || !o->field_i || !o->field_scale) return fail(HPG_NULLPOINTER, "null buffer");
  if (b->batch_count < 1) return fail(HPG_INVALIDDIMENSION, "batch_count");
  const int A = std::max(1, b->avg_count);
  if (!b->members && (int64_t)b->batch_count * A > b->frame_count)
    return fail(HPG_INVALIDDIMENSION, "frame buffer holds fewer frames than batch*avg");
  if (b->frame_format != 0 && b->frame_format != 1) return fail(HPG_INVALIDARGUMENT, "frame_format");
  if (b->layout_width > 0) {
    for (int q = 0; q < P->g.P; ++q)
      if (b->layout_col0[q] < 0 || b->layout_row0[q] < 0 || b->layout_col0[q] + P->g.nx > b->layout_width ||
          b->layout_row0[q] + P->g.ny > b->layout_height)
        return fail(HPG_INVALIDDIMENSION, "layout override does not contain the FFT window");
  }
  if (b->batch_cal && (b->cal_pols < 1 || b->cal_batch < 1)) return fail(HPG_INVALIDARGUMENT, "batch calibration dims");
  if (b->row_offset < 0) return fail(HPG_INVALIDARGUMENT, "row_offset");
  if ((flags & HPG_FLAG_SUMMARY) && o->field_params && o->param_slots < b->batch_count + 1)
    return fail(HPG_INVALIDDIMENSION, "param_slots");
  RunParams rp;
  fill_params(P, b, o, flags, rp);
  rp.lay = make_layout(P, b->batch_count, A, flags, false);
  finish_layout(P, rp.lay, (int64_t)b->batch_count * P->g.P, flags);
  const int64_t need = rp.lay.agg_off + rp.lay.agg_per_cta * rp.lay.grid;
  if ((rp.lay.slab_bytes > 0 || (flags & HPG_FLAG_SUMMARY)) && (!o->workspace || (int64_t)o->workspace_bytes < need))
    return fail(HPG_INVALIDARGUMENT, "workspace too small (hpg_workspace_size)");
  cudaError_t e;
  const int64_t items = (int64_t)b->batch_count * P->g.P;
  // Two-kernel tensor-core path (holo_tc2.cu): asked for with HPG_FLAG_TC2, and chosen automatically for
  // batches of at least 6 windows per SM with a basis of at most 16 orders -- below that its persistent
  // set-up and second launch cost more than they save, and larger bases run the tensor-core overlap of the
  // fused kernel.  HPG_FLAG_SIMT / HPG_FLAG_TC / HPG_FLAG_GENERIC keep their kernels.
  const bool tc2_ok = !(flags & (HPG_FLAG_GENERIC | HPG_FLAG_SIMT)) && !b->members &&
                      tc2_supported(rp.g, A, b->frame_format, b->transpose, P->fill, b->ref_cal, flags, o->windows);
  const bool tc2_auto = tc2_ok && !(flags & HPG_FLAG_TC) && items >= 6 * (int64_t)P->num_sms && rp.g.G <= 16 &&
                        o->workspace && o->workspace_bytes >= tc2_workspace(items) && !getenv("HOLO_NO_TC2");
  if (tc2_ok && ((flags & HPG_FLAG_TC2) || tc2_auto)) {
    if (!o->workspace || o->workspace_bytes < tc2_workspace((int64_t)b->batch_count * P->g.P))
      return fail(HPG_INVALIDARGUMENT, "workspace too small (hpg_workspace_size)");
    e = ensure_tc_tables(P);
    if (e == cudaSuccess) e = launch_tc2(rp, P->ft, P->num_sms, static_cast<cudaStream_t>(stream));
    g_last_launches = 2 * (int)((items + tc2_chunk() - 1) / tc2_chunk());
  } else if ((flags & HPG_FLAG_TC) && !(flags & (HPG_FLAG_GENERIC | HPG_FLAG_SIMT)) && !b->members &&
      tc_supported(rp.g, A, b->frame_format, b->transpose, P->fill, b->ref_cal, flags, o->windows))
  {
    e = ensure_tc_tables(P);
    if (e == cudaSuccess) e = launch_fast_tc(rp, P->ft, P->num_sms, static_cast<cudaStream_t>(stream));
    g_last_launches = 1;
  }
  else if (!(flags & HPG_FLAG_GENERIC) && fast_supported(rp.g, A, b->frame_format, b->transpose, P->fill, b->ref_cal, flags, o->windows) &&
      !b->members) {
    e = launch_fast(rp, P->ft, P->num_sms, static_cast<cudaStream_t>(stream));
    g_last_launches = 1;
  }
  else if (!(flags & HPG_FLAG_GENERIC) && lw_supported(rp.g, A, b->members, flags, o->windows)) {
    if (!o->workspace || o->workspace_bytes < lw_workspace(rp.g, (int64_t)b->batch_count * P->g.P))
      return fail(HPG_INVALIDARGUMENT, "workspace too small (hpg_workspace_size)");
    e = launch_lw(rp, P->num_sms, static_cast<cudaStream_t>(stream));
    // rows, cols (+ the 164-point IFFT along y when fused), [ifft_y,] field, pack
    const bool fused164 = rp.g.gh == 164 && rp.g.wh == 164;
    const int per_chunk = (rp.g.nx == 512 && rp.g.ny == 512 && !fused164) ? 5 : 4;
    const int64_t slot = lw_slot_items(rp.g, items);
    g_last_launches = per_chunk * (int)((items + slot - 1) / slot) +
                      ((rp.coefs && rp.g.G > 0) ? 1 : 0);
  } else {
    e = launch_fused(rp, static_cast<cudaStream_t>(stream));
    g_last_launches = 1;
  }
  if (e != cudaSuccess) return cuda_fail(e, "fused kernel launch");
  return HPG_SUCCESS;
}

int hpg_finalize_summary(const hpg_plan* P, const hpg_batch* b, const hpg_outputs* o, float* total,
                         void* stream) {
  if (!P || !b || !o || !o->workspace) return fail(HPG_NULLPOINTER, "null argument");
  RunParams rp;
  fill_params(P, b, o, HPG_FLAG_SUMMARY, rp);
  rp.lay = make_layout(P, b->batch_count, std::max(1, b->avg_count), HPG_FLAG_SUMMARY, false);
  finish_layout(P, rp.lay, (int64_t)b->batch_count * P->g.P, HPG_FLAG_SUMMARY);
  cudaError_t e = launch_finalize(rp, total, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "finalize kernel launch");
  return HPG_SUCCESS;
}

int hpg_fourier_full(const hpg_plan* P, const hpg_batch* b, void* plane, void* workspace, size_t ws_bytes,
                     void* stream) {
  if (!P || !b || !b->frames || !plane) return fail(HPG_NULLPOINTER, "null argument");
  RunParams rp;
  fill_params(P, b, nullptr, 0, rp);
  rp.work = static_cast<char*>(workspace);
  const int64_t F = b->frame_count;
  rp.lay = make_layout(P, 1, 1, 0, true);
  finish_layout(P, rp.lay, F * P->g.P, 0);
  if (rp.lay.slab_bytes > 0 && (!workspace || (int64_t)ws_bytes < rp.lay.slab_bytes * rp.lay.grid))
    return fail(HPG_INVALIDARGUMENT, "workspace too small");
  cudaError_t e = launch_fourier_full(rp, F, static_cast<float2*>(plane), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fourier kernel launch");
  return HPG_SUCCESS;
}

static int plane_grid(int64_t count, int P) { return (int)std::min<int64_t>(count * P, 148); }

size_t hpg_plane_summary_workspace(int64_t count, int32_t P, int32_t h, int32_t w) {
  return (size_t)plane_grid(count, P) * (size_t)align_up((int64_t)P * h * w * 8, 256);
}

int hpg_plane_summary(const void* data, int64_t count, int32_t P, int32_t h, int32_t w, const double* xa,
                      const double* ya, float* params, int32_t slots, float* total, double* pol_total, void* work,
                      size_t work_bytes, void* stream) {
  if (!data || !xa || !ya || !params || !work) return fail(HPG_NULLPOINTER, "null argument");
  if (count < 1 || P < 1 || h < 1 || w < 1) return fail(HPG_INVALIDDIMENSION, "empty plane");
  if (slots < count + 1) return fail(HPG_INVALIDDIMENSION, "slots");
  if (work_bytes < hpg_plane_summary_workspace(count, P, h, w)) return fail(HPG_INVALIDARGUMENT, "workspace too small");
  cudaError_t e = launch_plane_summary(static_cast<const float2*>(data), count, P, h, w, xa, ya, params, slots,
                                       total, pol_total, static_cast<char*>(work), plane_grid(count, P),
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "plane summary launch");
  return HPG_SUCCESS;
}

int hpg_field_intensity(const int16_t* fr, const int16_t* fi, const float* scale, int32_t B, int32_t P, int32_t h,
                        int32_t w, double* out, void* stream) {
  if (!fr || !fi || !scale || !out) return fail(HPG_NULLPOINTER, "null argument");
  if (B < 1 || P < 1 || h < 1 || w < 1) return fail(HPG_INVALIDDIMENSION, "dimensions");
  cudaError_t e = launch_field_intensity(fr, fi, scale, B, P, h * w, out, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "field intensity launch");
  return HPG_SUCCESS;
}

int hpg_ref_calibration_finish(const void* a, const void* b, int64_t n, void* applied, void* stream) {
  if (!a || !applied) return fail(HPG_NULLPOINTER, "null argument");
  if (n < 1) return fail(HPG_INVALIDDIMENSION, "count");
  cudaError_t e = launch_refcal_finish(static_cast<const float2*>(a), static_cast<const float2*>(b), n,
                                       static_cast<float2*>(applied), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "reference calibration launch");
  return HPG_SUCCESS;
}

int hpg_upload_windows(const hpg_plan* P, const void* host, int32_t fmt, int64_t F, void* dst, void* stream) {
  if (!P || !host || !dst) return fail(HPG_NULLPOINTER, "null argument");
  if (F < 1) return fail(HPG_INVALIDDIMENSION, "frame_count");
  const Geometry& g = P->g;
  const size_t es = fmt == 1 ? 2 : 4;
  for (int q = 0; q < g.P; ++q) {
    cudaMemcpy3DParms m = {};
    m.srcPtr = make_cudaPitchedPtr(const_cast<void*>(host), (size_t)g.W * es, (size_t)g.W, (size_t)g.H);
    m.srcPos = make_cudaPos((size_t)g.col0[q] * es, (size_t)g.row0[q], 0);
    m.dstPtr = make_cudaPitchedPtr(dst, (size_t)g.P * g.nx * es, (size_t)g.P * g.nx, (size_t)g.ny);
    m.dstPos = make_cudaPos((size_t)q * g.nx * es, 0, 0);
    m.extent = make_cudaExtent((size_t)g.nx * es, (size_t)g.ny, (size_t)F);
    m.kind = cudaMemcpyHostToDevice;
    cudaError_t e = cudaMemcpy3DAsync(&m, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy3DAsync");
  }
  return HPG_SUCCESS;
}

int hpg_extract_coefs(const hpg_plan* P, const int16_t* fr, const int16_t* fi, const float* scale,
                      int32_t B, void* coefs, void* stream) {
  if (!P || !fr || !fi || !scale || !coefs) return fail(HPG_NULLPOINTER, "null argument");
  if (P->g.G < 1) return HPG_SUCCESS;
  RunParams rp;
  std::memset(&rp, 0, sizeof(rp));
  rp.g = P->g;
  rp.t = P->t;
  rp.B = B;
  rp.fr = const_cast<int16_t*>(fr);
  rp.fi = const_cast<int16_t*>(fi);
  rp.scale = const_cast<float*>(scale);
  rp.coefs = static_cast<float2*>(coefs);
  const int grid = (int)std::min<int64_t>((int64_t)B * P->g.P, (int64_t)P->num_sms * 4);
  cudaError_t e = launch_coefs(rp, grid, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "coefs kernel launch");
  return HPG_SUCCESS;
}

}  // extern "C"

extern "C" int hpg_host_register(void* ptr, size_t bytes) {
  if (!ptr || bytes == 0) return HPG_NULLPOINTER;
  const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
  if (e == cudaSuccess) return HPG_SUCCESS;
  cudaGetLastError();   // not sticky: clear it so later calls do not report it
  return e == cudaErrorHostMemoryAlreadyRegistered ? HPG_INVALIDARGUMENT : fail(HPG_ERROR, cudaGetErrorString(e));
}

extern "C" int hpg_host_unregister(void* ptr) {
  if (!ptr) return HPG_NULLPOINTER;
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e == cudaSuccess) return HPG_SUCCESS;
  cudaGetLastError();
  return HPG_INVALIDARGUMENT;
}
