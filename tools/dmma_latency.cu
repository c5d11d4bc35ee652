// Latency of dependent fp64 tensor-core (mma.sync m8n8k4, DMMA) and DFMA
// chains on one warp, and DMMA throughput of one warp with k independent
// accumulators (sm_100a).  Dev tool: prints cycles per instruction.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int K>
__global__ void chain(double* out, long long* cyc, int n) {
  double c[K][2];
  for (int k = 0; k < K; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3 + k;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) dmma(c[k][0], c[k][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < K; ++k) s += c[k][0] + c[k][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void fchain(double* out, long long* cyc, int n) {
  double x = threadIdx.x * 1e-3, a = 1.0000001, b = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int K>
void run(double* out, long long* cyc, int n) {
  chain<K><<<1, 32>>>(out, cyc, n);
  long long h;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"probe\": \"dmma_m8n8k4_one_warp\", \"independent_accumulators\": %d, \"cycles_per_dmma\": %.2f}\n", K,
         (double)h / (n * K));
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  const int n = 4096;
  run<1>(out, cyc, n);
  run<2>(out, cyc, n);
  run<4>(out, cyc, n);
  run<8>(out, cyc, n);
  run<16>(out, cyc, n);
  fchain<<<1, 32>>>(out, cyc, n);
  long long h;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"probe\": \"dfma_dependent_chain\", \"cycles_per_dfma\": %.2f}\n", (double)h / n);
  return 0;
}
