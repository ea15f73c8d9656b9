// FP32 pipe probe (sm_100a): scalar FFMA / FADD against the packed FFMA2 / FADD2 (two fp32 lanes per register pair).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/f32x2_rate tools/f32x2_rate.cu && tools/f32x2_rate
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) { u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ffma1(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float fadd1(float a, float b) { float d; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }

template <int MODE>
__global__ void __launch_bounds__(512) probe(float* out, int iters, float x, float y) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
  u64* a2 = reinterpret_cast<u64*>(a);
  float2 xy = make_float2(x, y);
  const u64 X = *reinterpret_cast<u64*>(&xy);
  float r[16];   // per-thread (vector-register) second operands
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = 1.0f + threadIdx.x * 1e-6f * (i + 1);
  u64* r2 = reinterpret_cast<u64*>(r);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 4) {        // 16 scalar FFMA, three register operands
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = ffma1(a[i], r[i], r[(i + 1) & 15]);
    } else if (MODE == 5) { // 8 FFMA2, three register operands
#pragma unroll
      for (int i = 0; i < 8; ++i) a2[i] = ffma2(a2[i], r2[i], r2[(i + 1) & 7]);
    } else if (MODE == 6) { // 16 scalar FADD, two register operands
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fadd1(a[i], r[i]);
    } else if (MODE == 7) { // 8 FADD2, two register operands
#pragma unroll
      for (int i = 0; i < 8; ++i) a2[i] = fadd2(a2[i], r2[i]);
    } else if (MODE == 0) {        // 16 scalar FFMA
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = ffma1(a[i], x, y);
    } else if (MODE == 1) { // 8 FFMA2 (same 16 flops-lanes)
#pragma unroll
      for (int i = 0; i < 8; ++i) a2[i] = ffma2(a2[i], X, X);
    } else if (MODE == 2) { // 16 scalar FADD
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fadd1(a[i], x);
    } else {                // 8 FADD2
#pragma unroll
      for (int i = 0; i < 8; ++i) a2[i] = fadd2(a2[i], X);
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i] + r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) reinterpret_cast<long long*>(out)[1 << 20] = t1 - t0;
}

int main() {
  float* out;
  cudaMalloc(&out, (1 << 23) + 64);
  const int iters = 4096;
  const char* names[8] = {"FFMA  R,R,U,U", "FFMA2 R,R,U,U", "FADD  R,R,U", "FADD2 R,R,U",
                          "FFMA  R,R,R,R", "FFMA2 R,R,R,R", "FADD  R,R,R", "FADD2 R,R,R"};
  for (int m = 0; m < 8; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) probe<0><<<148 * 2, 512>>>(out, iters, 1.0001f, 0.5f);
      if (m == 1) probe<1><<<148 * 2, 512>>>(out, iters, 1.0001f, 0.5f);
      if (m == 2) probe<2><<<148 * 2, 512>>>(out, iters, 1.0001f, 0.5f);
      if (m == 3) probe<3><<<148 * 2, 512>>>(out, iters, 1.0001f, 0.5f);
      if (m == 4) probe<4><<<148 * 2, 512>>>(out, iters, 1.0001f, 0.5f);
      if (m == 5) probe<5><<<148 * 2, 512>>>(out, iters, 1.0001f, 0.5f);
      if (m == 6) probe<6><<<148 * 2, 512>>>(out, iters, 1.0001f, 0.5f);
      if (m == 7) probe<7><<<148 * 2, 512>>>(out, iters, 1.0001f, 0.5f);
      cudaDeviceSynchronize();
    }
    long long cyc;
    cudaMemcpy(&cyc, reinterpret_cast<long long*>(out) + (1 << 20), 8, cudaMemcpyDeviceToHost);
    // CTA 0's own span: 16 warps, 16 fp32 lane-results per thread per iteration (the SM's other CTA runs beside it)
    const double lanes = 2 * 512.0 * 16 * iters;
    printf("%s: %lld cycles, %.1f fp32 results / clk / SM, %.2f warp-instr / clk / SM\n", names[m], cyc, lanes / cyc,
           lanes / cyc / 32 / ((m & 1) ? 2 : 1));
  }
  return 0;
}
