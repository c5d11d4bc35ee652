// Accuracy probe of the rsqrt.approx.ftz.f64 seed and the Newton variants used
// by the mapped-grid regeneration kernels (dev tool).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void probe(const double* x, double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = x[i], y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
  out[4 * i] = y;
  double e = fma(-v, y * y, 1.0);
  double y1 = fma(0.5 * y, e, y);
  double e1 = fma(-v, y1 * y1, 1.0);
  out[4 * i + 1] = fma(0.5 * y1, e1, y1);                       // two Newton steps
  out[4 * i + 2] = fma(y * e, fma(0.375, e, 0.5), y);           // one third-order step
  out[4 * i + 3] = rsqrt(v);                                    // libdevice
}

int main() {
  const int n = 1 << 20;
  double *hx = new double[n], *ho = new double[4 * n];
  for (int i = 0; i < n; ++i) hx[i] = std::exp(-14.0 + 16.0 * (i + 0.5) / n) * (1.0 + 0.37 * std::sin(1.0 * i));
  double *dx, *dout;
  cudaMalloc(&dx, n * 8);
  cudaMalloc(&dout, 4 * n * 8);
  cudaMemcpy(dx, hx, n * 8, cudaMemcpyHostToDevice);
  probe<<<(n + 255) / 256, 256>>>(dx, dout, n);
  cudaMemcpy(ho, dout, 4 * n * 8, cudaMemcpyDeviceToHost);
  double err[4] = {0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
    long double ref = 1.0L / sqrtl((long double)hx[i]);
    for (int k = 0; k < 4; ++k) {
      double e = (double)fabsl(((long double)ho[4 * i + k] - ref) / ref);
      if (e > err[k]) err[k] = e;
    }
  }
  printf("{\"probe\": \"rsqrt\", \"seed\": %.3e, \"newton2\": %.3e, \"third_order\": %.3e, \"libdevice\": %.3e}\n",
         err[0], err[1], err[2], err[3]);
  return 0;
}
