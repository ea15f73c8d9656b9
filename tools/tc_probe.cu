// tcgen05 probe: D[128x128] (fp32, TMEM) = A[128xK] (fp16, TMEM) * B[KxN]^T-stored
// (fp16, smem, K-major, no swizzle).  Validates descriptors / TMEM layouts used by
// the tensor-core row DFT, against a host fp64 reference.
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int M = 128, N = 128, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// canonical K-major SWIZZLE_NONE: [K/16][N/8][2][8 rows][8 halves]; 16-B rows
__device__ __forceinline__ int b_off_halves(int n, int k) {
  const int ks = k >> 4, kh = (k >> 3) & 1, kk = k & 7, ng = n >> 3, r = n & 7;
  return (((ks * (N / 8) + ng) * 2 + kh) * 8 + r) * 8 + kk;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;
}

__global__ void __launch_bounds__(128) probe(const __half* A, const __half* B, float* D) {
  __shared__ __align__(1024) __half sB[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i - n * K;
    sB[b_off_halves(n, k)] = B[n * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  // A into TMEM columns [0, K/2): row m = lane m, 2 halves per 32-bit column
  {
    const int m = warp * 32 + lane;
    uint32_t r[32];
#pragma unroll
    for (int c = 0; c < K / 2; ++c) {
      __half2 h = __halves2half2(A[m * K + 2 * c], A[m * K + 2 * c + 1]);
      r[c] = *reinterpret_cast<uint32_t*>(&h);
    }
    const uint32_t taddr = tm + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t d_t = tm + 128;  // D at columns [128, 256)
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t bdesc = make_desc(smem_u32(sB) + s * (N * 16 * 2), 128, 256);
      const uint32_t a_t = tm + s * 8;
      const uint32_t acc = s > 0;
      asm volatile(
          "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d_t),
          "r"(a_t), "l"(bdesc), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&mbar)));
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
          : "=r"(done)
          : "r"(smem_u32(&mbar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const int m = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 32) {
      uint32_t r[32];
      const uint32_t taddr = d_t + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
            "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
            "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
            "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 32; ++j) D[m * N + c0 + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

int main() {
  std::vector<__half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) { float v = (rand() % 2001 - 1000) / 256.f; A[i] = __float2half(v); Af[i] = __half2float(A[i]); }
  for (int i = 0; i < N * K; ++i) { float v = (rand() % 2001 - 1000) / 512.f; B[i] = __float2half(v); Bf[i] = __half2float(B[i]); }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), N * K * 2, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  probe<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> D(M * N);
  cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)Af[m * K + k] * Bf[n * K + k];
      maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
      maxref = fmax(maxref, fabs(ref));
    }
  printf("max |err| %.3e  max |ref| %.3e  D[0]=%f D[1]=%f D[129]=%f\n", maxerr, maxref, D[0], D[1], D[129]);
  return maxerr < 1e-3 * maxref ? 0 : 1;
}
