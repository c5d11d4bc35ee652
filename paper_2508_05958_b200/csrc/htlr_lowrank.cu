// H-matrix baseline of the reference (blocks.py:76-86,167-187,262-264;
// operators.py:129-135,164-165) on the device.
//
// The reference's LowRankBlock stores u = Q of QR(kron(L_d..L_1)) (s^d x p^d),
// g = R_u (h^d G) R_v^T and v, and applies u (g (v^T x)).  The QR of a
// Kronecker product is the Kronecker product of the per-dimension QRs (up to
// column signs, which cancel in u g v^T), so with the per-level Q of the
// Tucker plan the baseline is u = kron(Q, .., Q) and g = the Tucker core: the
// same operator with the factors applied as dense s^d x p^d matrices instead
// of d mode products -- the representation whose storage and work the paper
// compares against.
#include "htlr_kernels.h"

namespace htlr {

// K[i][a] = prod_k Q[i_k][a_k], i and a F-order multi-indices (first fastest)
__global__ void kron_factor_kernel(const double* __restrict__ Q, int d, int s, int p, double* __restrict__ K) {
  const int P = (d == 2) ? p * p : p * p * p;
  const int64_t S = (d == 2) ? (int64_t)s * s : (int64_t)s * s * s;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < S * P; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / P;
    const int a = (int)(e % P);
    double v = Q[(i % s) * p + a % p] * Q[((i / s) % s) * p + (a / p) % p];
    if (d == 3) v *= Q[(i / ((int64_t)s * s)) * p + a / (p * p)];
    K[e] = v;
  }
}

// W[c][r][a] = sum_i K[i][a] u_c[i]  (u_c = cluster c's points, F-order)
__global__ void dense_upward_kernel(const double* __restrict__ u, double* __restrict__ W, int d, int n, int s, int p,
                                    int bits, int R, int K_pad, const double* __restrict__ K, int64_t c0) {
  const int64_t c = c0 + blockIdx.x;
  const int r = blockIdx.y;
  int cc[3];
  morton_decode(c, d, bits, cc);
  const int P = (d == 2) ? p * p : p * p * p;
  const int64_t S = (d == 2) ? (int64_t)s * s : (int64_t)s * s * s;
  double* dst = W + ((int64_t)c * R + r) * K_pad;
  for (int a = threadIdx.x; a < K_pad; a += blockDim.x) {
    double v = 0.0;
    if (a < P) {
      for (int64_t i = 0; i < S; ++i) {
        const int x = (int)(i % s), y = (int)((i / s) % s), z = (int)(i / ((int64_t)s * s));
        int64_t g = (int64_t)(cc[0] * s + x) + (int64_t)n * (cc[1] * s + y);
        if (d == 3) g += (int64_t)n * n * (cc[2] * s + z);
        v += K[i * P + a] * u[g * R + r];
      }
    }
    dst[a] = v;
  }
}

void launch_kron_factor(const double* Q, int d, int s, int p, double* K, cudaStream_t st) {
  kron_factor_kernel<<<1024, 256, 0, st>>>(Q, d, s, p, K);
}

void launch_dense_upward(const double* u, double* W, int d, int n, int side, int p, int level, int R, int K_pad,
                         const double* K, int64_t c0, int64_t nc, cudaStream_t st) {
  if (nc > 0) dense_upward_kernel<<<dim3((unsigned)nc, R), 256, 0, st>>>(u, W, d, n, side, p, level, R, K_pad, K, c0);
}

}  // namespace htlr
