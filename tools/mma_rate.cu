// tcgen05.mma issue/execute rate probe (sm_100a): one CTA per SM, one issuing thread, R x 24 MMAs of
// M = 128, K = 16 into one accumulator; cycles per MMA for operand-source / N / layout variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu && tools/mma_rate
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__device__ __forceinline__ uint32_t idesc(int M, int N) { return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24); }
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

// variant: 0 TS N128 noswz (3-product pattern) | 1 SS N128 noswz | 2 TS N96 | 3 TS N128 SW128 | 4 TS N256 noswz
//          5 TS N128 noswz, every MMA reads the same B slice | 6 TS N64 | 7 TS N128 noswz + 8 warps hammering smem
template <bool USE_ELECT>
__global__ void __launch_bounds__(384, 1) probe(int variant, int R, long long* out) {
  extern __shared__ __align__(1024) char smem[];   // 128 KB: B operand(s)
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;   // 1.0h
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (warp == 0) {
    const int N = variant == 2 ? 96 : variant == 4 ? 256 : variant == 6 ? 64 : 128;
    const uint32_t id = idesc(128, N);
    const uint32_t sb = smem_u32(smem);
    const int ng = N / 8;   // row groups
    long long t0 = 0, t1 = 0, t2 = 0;
    uint32_t elected = 0;
    asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0, 1, 0, p;}" : "=r"(elected));
    if (USE_ELECT ? elected != 0 : lane == 0) {
      t0 = clock64();
      for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int gk = 0; gk < 8; ++gk) {
          uint64_t bh, bl;
          if (variant == 3) {   // SW128 K-major: [K block 64][row][128 B], k-step = +32 B inside the atom
            bh = desc(sb + (gk >> 2) * 16384 + (gk & 3) * 32, 16, 1024, 2);
            bl = desc(sb + 32768 + (gk >> 2) * 16384 + (gk & 3) * 32, 16, 1024, 2);
          } else {
            const int g2 = variant == 5 ? 0 : gk;
            bh = desc(sb + g2 * ng * 256, 128, 256, 0);
            bl = desc(sb + 65536 + g2 * ng * 256, 128, 256, 0);
          }
          const uint32_t d = tm + 256;
          if (variant == 1) {
            const uint64_t ah = desc(sb + 98304 + gk * 4096, 128, 256, 0);
            mma_ss(d, ah, bh, id, gk != 0 || r != 0);
            mma_ss(d, ah, bh, id, 1);
            mma_ss(d, ah, bl, id, 1);
          } else {
            mma_ts(d, tm + gk * 8, bh, id, gk != 0 || r != 0);
            mma_ts(d, tm + 64 + gk * 8, bh, id, 1);
            mma_ts(d, tm + gk * 8, bl, id, 1);
          }
        }
      }
      t1 = clock64();
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    __syncwarp();
    uint32_t done = 0;
    while (!done)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}" : "=r"(done) : "r"(smem_u32(&bar)));
    if (USE_ELECT ? elected != 0 : lane == 0) {
      t2 = clock64();
      stop = 1;
      if (blockIdx.x == 0) {
        out[variant * 2] = t1 - t0;
        out[variant * 2 + 1] = t2 - t0;
      }
    }
  } else if (variant == 7 && warp >= 4) {   // shared-memory traffic like the K1 producers: 16-byte loads + stores
    uint4* q = reinterpret_cast<uint4*>(smem + 65536 + 32768) + (tid - 128);
    uint4 acc = make_uint4(0, 0, 0, 0);
    while (!stop) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint4 v = q[i * 256];
        acc.x ^= v.x;
        q[i * 256] = acc;
      }
    }
    if (acc.x == 0x12345) out[63] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* out;
  cudaMallocManaged(&out, 64 * sizeof(long long));
  cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int R = 20;
  const char* names[8] = {"TS N128 noswz", "SS N128 noswz", "TS N96 noswz", "TS N128 SW128", "TS N256 noswz",
                          "TS N128 same-B", "TS N64 noswz", "TS N128 noswz + smem traffic"};
  for (int v = 0; v < 16; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      if (v < 8) probe<false><<<148, 384, 128 * 1024>>>(v, R, out);
      else probe<true><<<148, 384, 128 * 1024>>>(v - 8, R, out + 16);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("variant %d: %s\n", v, cudaGetErrorString(e)); return 1; }
    }
    printf("%-30s %s issue %.1f cyc/MMA, complete %.1f cyc/MMA\n", names[v & 7], v < 8 ? "lane0" : "elect", out[2 * v] / (24.0 * R), out[2 * v + 1] / (24.0 * R));
  }
  return 0;
}
