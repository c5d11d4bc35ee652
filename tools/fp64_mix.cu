// Do fp64 DMMA (mma.sync m8n8k4) and DFMA share the fp64 datapath on B200?
// Times three loops with the same per-warp instruction counts: DMMA only,
// DFMA only, both interleaved.  time(both) ~ max(A, B): separate pipes;
// ~ A + B: shared.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/fp64_mix.cu -o tools/fp64_mix
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int MODE>   // 1 DMMA, 2 DFMA, 3 both
__global__ void mix(int iters, double* out) {
  double c[8][2], f[16];
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int i = 0; i < 16; ++i) f[i] = 0.1 * i;
  for (int it = 0; it < iters; ++it) {
    if (MODE & 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    if (MODE & 2) {
      // 8 DMMA.8x8x4 = 2048 MAC per warp; 64 DFMA per lane = 2048 FMA per warp
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(f[i], b, a);
    }
  }
  double s = 0.0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < 16; ++i) s += f[i];
  if (s == 12345.678) out[0] = s;
}

template <int MODE>
float run(int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<MODE><<<blocks, threads>>>(iters / 10, out);
  cudaEventRecord(e0);
  mix<MODE><<<blocks, threads>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int warps = 4; warps <= 16; warps *= 2) {
    const int blocks = sms * 2, threads = 32 * warps, iters = 20000;
    const float a = run<1>(blocks, threads, iters, out), b = run<2>(blocks, threads, iters, out),
                c = run<3>(blocks, threads, iters, out);
    const double macs = 2048.0 * iters * blocks * warps;
    printf("{\"probe\": \"dmma_dfma_mix\", \"warps_per_block\": %d, \"dmma_ms\": %.3f, \"dfma_ms\": %.3f, "
           "\"both_ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"both_over_sum\": %.3f, "
           "\"both_over_max\": %.3f}\n",
           warps, a, b, c, 2 * macs / a / 1e9, 2 * macs / b / 1e9, c / (a + b), c / (a > b ? a : b));
  }
  return 0;
}
