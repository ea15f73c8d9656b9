// DRAM read rate of the window access pattern of BASELINE config 2 (1,000 frames of 256 x 640 float32; two
// 128 x 128 windows per frame: rows 64..191, columns 96..223 and 416..543) against a dense read of the same
// number of bytes.  Plain 16-byte loads, one warp per 512-byte window row, enough CTAs to fill the machine.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/window_read_rate tools/window_read_rate.cu
#include <cstdio>
#include <cstdint>

__global__ void __launch_bounds__(256) read_windows(const float4* __restrict__ frames, int F, int dense, int u16,
                                                    float* out) {
  // work item = (frame, pol, row): 128 float4 per 512-byte row -> one warp reads a row with one load per lane
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  const int items = F * 2 * 128;
  for (int it0 = warp * 4; it0 < items; it0 += nwarps * 4) {   // four rows in flight per warp
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int it = it0 + u;
      size_t off;   // in float4
      if (dense) {
        off = (size_t)it * 32 + lane;
      } else {
        const int f = it >> 8, q = (it >> 7) & 1, r = it & 127;
        off = ((size_t)f * 256 * 640 + (size_t)(64 + r) * 640 + (q ? 416 : 96)) / 4 + lane;
        if (u16) off = ((size_t)f * 256 * 640 + (size_t)(64 + r) * 640 + (q ? 416 : 96)) / 8 + (lane & 15);   // 256-byte rows
      }
      v[u] = __ldg(frames + off);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 123.456f) out[0] = acc;
}

int main() {
  const int F = 1000;
  const size_t bytes = (size_t)F * 256 * 640 * 4;
  float4* d;
  float* out;
  cudaMalloc(&d, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(d, 0, bytes);
  char* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[3] = {"f32 windows (512-byte row segments)", "dense read of the same bytes", "u16 windows (256-byte row segments)"};
  for (int mode = 0; mode < 6; ++mode) {
    float best = 1e9f;
    const bool do_flush = mode < 3;
    for (int rep = 0; rep < 6; ++rep) {
      if (do_flush) cudaMemset(flush, rep, 256 << 20);   // bench.py's L2 flush: leaves L2 full of dirty lines
      cudaEventRecord(a);
      read_windows<<<148 * 8, 256>>>(d, F, mode % 3 == 1, mode % 3 == 2, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best) best = ms;
    }
    const double mb = F * 2 * 128 * (mode % 3 == 2 ? 256.0 : 512.0) / 1e6;
    printf("%-40s %s %.1f MB in %.1f us = %.2f TB/s\n", names[mode % 3], do_flush ? "after a 256 MB flush write" : "back to back, no flush      ", mb, best * 1e3, mb / 1e6 / (best * 1e-3));
  }
  return 0;
}
