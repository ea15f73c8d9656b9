// Transfer-matrix metric reductions (holopipe/analysis.py:104-188) on the GPU.
//
// The reference builds the (rows x cols) complex128 transfer matrix from the
// coefficients and calls numpy / LAPACK per wavelength.  Here one pass over
// the complex64 coefficients produces, in fp64:
//   row_power[r]   = sum_j |A_rj|^2                           (IL, SNR rows)
//   diag_power[r]  = |A_r,d|^2,  d = r + diag_offset          (DIAG*, SNR*)
//   group_power[r] = sum_{j: label_j == label_d} |A_rj|^2     (SNRMG)
//   gram           = X X^H with X = A (rows <= cols) or A^T   (MDL eigenvalues)
// These are additive over row shards, so a multi-GPU caller all-reduces them
// (NCCL) and finishes the nine metrics on the host from O(rows + cols^2) data.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/holo_b200.h"

namespace {

struct MArgs {
  const float2* coefs;
  int rows, cols, ld;
  const int32_t* row_ids;
  const int32_t* col_offset;
  const int32_t* col_count;
  const int32_t* labels;
  int ndiag, diag_offset;
  int gram_rows;
  double* row_power;
  double* diag_power;
  double* group_power;
  double2* gram;
};

__device__ __forceinline__ double2 elem(const MArgs& a, int r, int j) {
  const int off = a.col_offset ? a.col_offset[r] : 0;
  const int cnt = a.col_count ? a.col_count[r] : a.cols;
  if (j < off || j >= off + cnt) return make_double2(0.0, 0.0);
  const float2 v = a.coefs[(size_t)a.row_ids[r] * a.ld + j];
  return make_double2(v.x, v.y);
}

__global__ void row_kernel(const MArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= a.rows) return;
  const int r = warp, d = r + a.diag_offset;
  const bool has_diag = d < a.ndiag;
  const int lab = has_diag && a.labels ? a.labels[d] : -1;
  double rp = 0.0, gp = 0.0;
  for (int j = lane; j < a.cols; j += 32) {
    const double2 v = elem(a, r, j);
    const double p = v.x * v.x + v.y * v.y;
    rp += p;
    if (has_diag && a.labels && a.labels[j] == lab) gp += p;
  }
  for (int o = 16; o; o >>= 1) {
    rp += __shfl_xor_sync(0xffffffffu, rp, o);
    gp += __shfl_xor_sync(0xffffffffu, gp, o);
  }
  if (lane == 0) {
    a.row_power[r] = rp;
    if (has_diag) {
      const double2 v = elem(a, r, d);
      a.diag_power[r] = v.x * v.x + v.y * v.y;
      a.group_power[r] = a.labels ? gp : a.diag_power[r];
    } else {
      a.diag_power[r] = -1.0;
      a.group_power[r] = -1.0;
    }
  }
}

// H[i][j] = sum_k X[i][k] conj(X[j][k]); X = A (gram_rows) or A^T.
constexpr int T = 16;
__global__ void gram_kernel(const MArgs a) {
  __shared__ double2 xi[T][T + 1], xj[T][T + 1];
  const int n = a.gram_rows ? a.rows : a.cols;
  const int K = a.gram_rows ? a.cols : a.rows;
  const int i = blockIdx.y * T + threadIdx.y, j = blockIdx.x * T + threadIdx.x;
  double sr = 0.0, si = 0.0;
  for (int k0 = 0; k0 < K; k0 += T) {
    const int kk = k0 + threadIdx.x;
    const int ii = blockIdx.y * T + threadIdx.y, jj = blockIdx.x * T + threadIdx.y;
    double2 vi = make_double2(0, 0), vj = make_double2(0, 0);
    if (kk < K && ii < n) vi = a.gram_rows ? elem(a, ii, kk) : elem(a, kk, ii);
    if (kk < K && jj < n) vj = a.gram_rows ? elem(a, jj, kk) : elem(a, kk, jj);
    xi[threadIdx.y][threadIdx.x] = vi;
    xj[threadIdx.y][threadIdx.x] = vj;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const double2 u = xi[threadIdx.y][k], v = xj[threadIdx.x][k];
      sr += u.x * v.x + u.y * v.y;
      si += u.y * v.x - u.x * v.y;
    }
    __syncthreads();
  }
  if (i < n && j < n) a.gram[(size_t)i * n + j] = make_double2(sr, si);
}

// out[r][p][o] = sum_{m < use} T[o][m] x[r][p][m], fp64 accumulation (the reference's complex128
// einsum, holopipe/engine.py:375-380).  block != 0: T is block-diagonal by mode group (the HG->LG
// matrix, hgbasis.py:126-152), so output o of group g only reads inputs [g(g+1)/2, g(g+1)/2 + g].
__global__ void coef_transform_kernel(const float2* __restrict__ x, int64_t rows, int pols, int m_in,
                                      const double2* __restrict__ t, int m_out, int use, int ld, int block,
                                      float2* __restrict__ out) {
  extern __shared__ double2 xs[];
  const int64_t rp = blockIdx.x;   // one (row, pol) per CTA
  const float2* xr = x + rp * m_in;
  for (int m = threadIdx.x; m < use; m += blockDim.x) {
    const float2 v = xr[m];
    xs[m] = make_double2(v.x, v.y);
  }
  __syncthreads();
  for (int o = threadIdx.x; o < m_out; o += blockDim.x) {
    int lo = 0, hi = use;
    if (block) {
      int g = (int)((sqrt(8.0 * o + 1.0) - 1.0) * 0.5);
      while ((g + 1) * (g + 2) / 2 <= o) ++g;
      while (g * (g + 1) / 2 > o) --g;
      lo = g * (g + 1) / 2;
      hi = min(use, lo + g + 1);
    }
    const double2* tr = t + (int64_t)o * ld;
    double re = 0.0, im = 0.0;
    for (int m = lo; m < hi; ++m) {
      const double2 a = __ldg(&tr[m]), b = xs[m];
      re = fma(a.x, b.x, fma(-a.y, b.y, re));
      im = fma(a.x, b.y, fma(a.y, b.x, im));
    }
    out[rp * m_out + o] = make_float2((float)re, (float)im);
  }
}

}  // namespace

extern "C" int hpg_coef_transform(const void* coefs, int64_t rows, int32_t pols, int32_t modes_in,
                                  const void* transform, int32_t modes_out, int32_t use, int32_t ld,
                                  int32_t block_diagonal, void* out, void* stream) {
  if (!coefs || !transform || !out) return HPG_NULLPOINTER;
  if (rows < 0 || pols < 1 || modes_in < 1 || modes_out < 1 || use < 1 || use > modes_in || ld < use)
    return HPG_INVALIDDIMENSION;
  if (rows == 0) return HPG_SUCCESS;
  const size_t smem = (size_t)use * sizeof(double2);
  if (smem > 200 * 1024) return HPG_INVALIDDIMENSION;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(coef_transform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
    return HPG_ERROR;
  coef_transform_kernel<<<(unsigned)(rows * pols), 256, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const float2*>(coefs), rows, pols, modes_in, static_cast<const double2*>(transform), modes_out,
      use, ld, block_diagonal, static_cast<float2*>(out));
  return cudaGetLastError() == cudaSuccess ? HPG_SUCCESS : HPG_ERROR;
}

extern "C" int hpg_metric_partials(const hpg_metric_args* m, void* stream) {
  if (!m || !m->coefs || !m->row_ids || !m->row_power || !m->diag_power || !m->group_power)
    return HPG_NULLPOINTER;
  if (m->rows < 1 || m->cols < 1) return HPG_INVALIDDIMENSION;
  MArgs a;
  a.coefs = static_cast<const float2*>(m->coefs);
  a.rows = m->rows;
  a.cols = m->cols;
  a.ld = m->ld > 0 ? m->ld : m->cols;
  a.row_ids = m->row_ids;
  a.col_offset = m->col_offset;
  a.col_count = m->col_count;
  a.labels = m->labels;
  a.ndiag = m->ndiag;
  a.diag_offset = m->diag_offset;
  a.gram_rows = m->gram_rows;
  a.row_power = m->row_power;
  a.diag_power = m->diag_power;
  a.group_power = m->group_power;
  a.gram = static_cast<double2*>(m->gram);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  row_kernel<<<(a.rows * 32 + 255) / 256, 256, 0, s>>>(a);
  if (a.gram) {
    const int n = a.gram_rows ? a.rows : a.cols;
    dim3 grid((n + T - 1) / T, (n + T - 1) / T), block(T, T);
    gram_kernel<<<grid, block, 0, s>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HPG_SUCCESS : HPG_ERROR;
}
