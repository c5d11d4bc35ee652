// FP64 peak / fragment-layout probe for B200 (sm_100a).
//
// Measures, with CUDA events on the launching stream:
//   * DFMA throughput (independent FMA chains, full-chip grid)
//   * DMMA throughput for mma.sync f64 shapes m8n8k4, m16n8k4, m16n8k8, m16n8k16
//   * fp64 RED (atomicAdd, no return) throughput to L2-resident distinct addresses
// and checks the m16n8k8 f64 fragment layout against a host product.
// Prints one JSON object per measurement.  This is a tool, not part of the
// product path; its output is committed under profiles/ as the FP64 roofline
// denominator (MEASURED_PEAKS.json carries no FP64 figure).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void mma_m8n8k4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k4(double (&c)[4], const double (&a)[2], double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k8(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma_m16n8k16(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE, int ACC>
__global__ void dmma_kernel(double* out, int iters) {
  int lane = threadIdx.x & 31;
  double a8[8], b4[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a8[i] = 1e-3 * (lane + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b4[i] = 1e-3 * (lane - i);
  double c[ACC][4];
#pragma unroll
  for (int j = 0; j < ACC; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[j][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < ACC; ++j) {
      if (SHAPE == 0) { double cc[2] = {c[j][0], c[j][1]}; mma_m8n8k4(cc, a8[0], b4[0]); c[j][0] = cc[0]; c[j][1] = cc[1]; }
      if (SHAPE == 1) { double aa[2] = {a8[0], a8[1]}; mma_m16n8k4(c[j], aa, b4[0]); }
      if (SHAPE == 2) { double aa[4] = {a8[0], a8[1], a8[2], a8[3]}; double bb[2] = {b4[0], b4[1]}; mma_m16n8k8(c[j], aa, bb); }
      if (SHAPE == 3) { mma_m16n8k16(c[j], a8, b4); }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < ACC; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 12345.678) out[0] = s;
}

// m16n8k8 layout probe: A 16x8 row-major, B 8x8 (k x n), C 16x8.
__global__ void layout_probe(const double* A, const double* B, double* C) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[4] = {A[g * 8 + t], A[(g + 8) * 8 + t], A[g * 8 + t + 4], A[(g + 8) * 8 + t + 4]};
  double b[2] = {B[t * 8 + g], B[(t + 4) * 8 + g]};
  double c[4] = {0, 0, 0, 0};
  mma_m16n8k8(c, a, b);
  C[g * 8 + 2 * t] = c[0];
  C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2];
  C[(g + 8) * 8 + 2 * t + 1] = c[3];
}

__global__ void red_kernel(double* buf, long n, int iters) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (long j = i; j < n; j += stride) atomicAdd(&buf[j], 1.0);
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", prop.name, sms, prop.clockRate);
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;

  // DFMA: 148*4 blocks x 256 threads, 8 chains
  {
    int blocks = sms * 4, threads = 256, iters = 40000;
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaEventRecord(e0));
      dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
    }
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * blocks * threads * 8.0 * iters;
    printf("{\"probe\": \"dfma\", \"tflops\": %.3f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  // DMMA shapes
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const double macs[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
  for (int shape = 0; shape < 4; ++shape) {
    for (int warps = 4; warps <= 16; warps *= 2) {
      int blocks = sms * 2, threads = 32 * warps, iters = 4000;
      auto launch = [&]() {
        switch (shape) {
          case 0: dmma_kernel<0, 8><<<blocks, threads>>>(out, iters); break;
          case 1: dmma_kernel<1, 8><<<blocks, threads>>>(out, iters); break;
          case 2: dmma_kernel<2, 8><<<blocks, threads>>>(out, iters); break;
          case 3: dmma_kernel<3, 8><<<blocks, threads>>>(out, iters); break;
        }
      };
      launch();
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double flops = 2.0 * macs[shape] * 8 * iters * (double)blocks * warps;
      printf("{\"probe\": \"dmma_%s\", \"warps_per_block\": %d, \"tflops\": %.3f, \"ms\": %.3f}\n",
             names[shape], warps, flops / ms / 1e9, ms);
    }
  }
  // sustained DMMA m16n8k8 for ~4 s (power cap behaviour)
  {
    int blocks = sms * 2, threads = 256, iters = 20000;
    dmma_kernel<2, 8><<<blocks, threads>>>(out, iters);
    CK(cudaEventRecord(e0));
    int reps = 0;
    float total = 0;
    while (total < 4000.f) {
      dmma_kernel<2, 8><<<blocks, threads>>>(out, iters);
      ++reps;
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&total, e0, e1));
    }
    double flops = 2.0 * macs[2] * 8 * iters * (double)blocks * 8 * reps;
    printf("{\"probe\": \"dmma_m16n8k8_sustained\", \"tflops\": %.3f, \"ms\": %.3f, \"reps\": %d}\n",
           flops / total / 1e9, total, reps);
  }
  // layout probe
  {
    std::vector<double> hA(128), hB(64), hC(128), ref(128, 0.0);
    for (int i = 0; i < 128; ++i) hA[i] = std::sin(1.0 + i);
    for (int i = 0; i < 64; ++i) hB[i] = std::cos(2.0 + 3 * i);
    for (int m = 0; m < 16; ++m)
      for (int n = 0; n < 8; ++n)
        for (int k = 0; k < 8; ++k) ref[m * 8 + n] += hA[m * 8 + k] * hB[k * 8 + n];
    double *dA, *dB, *dC;
    CK(cudaMalloc(&dA, 1024));
    CK(cudaMalloc(&dB, 512));
    CK(cudaMalloc(&dC, 1024));
    CK(cudaMemcpy(dA, hA.data(), 1024, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB.data(), 512, cudaMemcpyHostToDevice));
    layout_probe<<<1, 32>>>(dA, dB, dC);
    CK(cudaMemcpy(hC.data(), dC, 1024, cudaMemcpyDeviceToHost));
    double err = 0;
    for (int i = 0; i < 128; ++i) err = std::fmax(err, std::fabs(hC[i] - ref[i]));
    printf("{\"probe\": \"layout_m16n8k8\", \"max_abs_err\": %.3e}\n", err);
  }
  // fp64 RED throughput into a 16 MiB (L2-resident) buffer
  {
    long n = 2 * 1024 * 1024;
    double* buf;
    CK(cudaMalloc(&buf, n * 8));
    CK(cudaMemset(buf, 0, n * 8));
    int iters = 50;
    red_kernel<<<sms * 8, 256>>>(buf, n, 2);
    CK(cudaEventRecord(e0));
    red_kernel<<<sms * 8, 256>>>(buf, n, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("{\"probe\": \"red_f64_l2\", \"gatom_per_s\": %.2f, \"ms\": %.3f}\n", n * (double)iters / ms / 1e6, ms);
  }
  return 0;
}
