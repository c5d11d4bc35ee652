// Ceiling of the regeneration inner loop on one GPU: per entry one DADD, the
// rsqrt seed + third-order correction, and two FMAs (row and column sums),
// 18 independent entries per tile as in htlr_regen_sym.cu.  Prints entries/s
// for a few block sizes / occupancies.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_pos(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

template <int R, int C>
__global__ void probe(const double* in, double* out, int iters) {
  double dx[R][C], vc[C], wt[R], ra[R], ca[C];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    wt[r] = in[(t + r) & 1023];
    ra[r] = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) dx[r][c] = 1.0 + in[(t + r * C + c) & 1023];
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
    vc[c] = in[(t * 3 + c) & 1023];
    ca[c] = 0;
  }
  double yz = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double kv = rsqrt_pos(dx[r][c] + yz);
        ra[r] = fma(kv, vc[c], ra[r]);
        ca[c] = fma(kv, wt[r], ca[c]);
      }
    yz += 1e-3;
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) s += ra[r];
#pragma unroll
  for (int c = 0; c < C; ++c) s += ca[c];
  out[t] = s;
}

template <int R, int C>
void run(int blocks, int threads, const double* in, double* out) {
  const int iters = 2000;
  probe<R, C><<<blocks, threads>>>(in, out, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<R, C><<<blocks, threads>>>(in, out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double ent = (double)blocks * threads * iters * R * C;
  printf("{\"probe\": \"regen_entry\", \"tile\": \"%dx%d\", \"blocks\": %d, \"threads\": %d, \"entries_per_s\": %.4e, "
         "\"dp_ops_per_entry\": 8}\n", R, C, blocks, threads, ent / (ms * 1e-3));
}

int main() {
  double *in, *out;
  cudaMalloc(&in, 1024 * sizeof(double));
  cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
  cudaMemset(in, 0, 1024 * sizeof(double));
  for (int bpsm : {1, 2, 4, 8}) {
    run<3, 6>(148 * bpsm, 256, in, out);
  }
  run<3, 6>(148 * 2, 288, in, out);
  run<3, 6>(148 * 4, 288, in, out);
  run<6, 6>(148 * 4, 256, in, out);
  run<2, 6>(148 * 4, 256, in, out);
  return 0;
}
