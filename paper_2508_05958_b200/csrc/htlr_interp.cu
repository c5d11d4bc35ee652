// Device versions of the reference's interpolation / kernel building blocks
// for the public API surface (chebyshev.py:31-85, kernels.py:105-117):
// Chebyshev nodes, Lagrange factor matrices and pairwise kernel values.  The
// plan's construction uses the same formulas inline (htlr_build.cu).
#include "htlr_kernels.h"

namespace htlr {

__global__ void cheb_nodes_kernel(double lo, double hi, int p, double* out) {
  const int t = threadIdx.x;
  if (t >= p) return;
  double arg = __ddiv_rn(__dmul_rn((double)(2 * (t + 1) - 1), 3.141592653589793), (double)(2 * p));
  out[t] = __dadd_rn(__dmul_rn(__dmul_rn(0.5, __dadd_rn(hi, -lo)), cos(arg)), __dmul_rn(0.5, __dadd_rn(hi, lo)));
}

__global__ void lagrange_kernel(const double* __restrict__ pts, int64_t n, const double* __restrict__ nodes, int p,
                                double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * p) return;
  const int64_t i = e / p;
  const int t = (int)(e % p);
  const double x = pts[i];
  double prod = 1.0;
  bool first = true;
  for (int j = 0; j < p; ++j) {
    if (j == t) continue;
    const double f = __ddiv_rn(__dadd_rn(x, -nodes[j]), __dadd_rn(nodes[t], -nodes[j]));
    prod = first ? f : __dmul_rn(prod, f);
    first = false;
  }
  out[e] = prod;
}

__global__ void pairs_kernel(KernelParams kp, int d, const double* __restrict__ x, int64_t m1,
                             const double* __restrict__ y, int64_t m2, double* __restrict__ out,
                             int* __restrict__ coincident) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m1 * m2) return;
  const int64_t i = e / m2, j = e % m2;
  const double r2 = r2_of(d, x + i * d, y + j * d);
  if (kp.kind != 0 && r2 == 0.0) {
    *coincident = 1;
    out[e] = 0.0;
    return;
  }
  out[e] = kernel_from_r2(kp, r2);
}

void launch_cheb_nodes(double lo, double hi, int p, double* out, cudaStream_t st) {
  cheb_nodes_kernel<<<1, 64, 0, st>>>(lo, hi, p, out);
}

void launch_lagrange(const double* pts, int64_t n, const double* nodes, int p, double* out, cudaStream_t st) {
  if (n * p > 0) lagrange_kernel<<<(unsigned)((n * p + 255) / 256), 256, 0, st>>>(pts, n, nodes, p, out);
}

void launch_pairs(const KernelParams& kp, int d, const double* x, int64_t m1, const double* y, int64_t m2, double* out,
                  int* coincident, cudaStream_t st) {
  if (m1 * m2 > 0)
    pairs_kernel<<<(unsigned)((m1 * m2 + 255) / 256), 256, 0, st>>>(kp, d, x, m1, y, m2, out, coincident);
}

}  // namespace htlr
