// Shared device helpers for the B200 HTLR kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace htlr {

// ---------------------------------------------------------------------------
// kernel functions (kernels.py:88-103), arithmetic in the reference's order;
// __dmul_rn/__dadd_rn keep nvcc from contracting r^2 into FMAs so r^2 is the
// value numpy computes.
// ---------------------------------------------------------------------------
struct KernelParams {
  int kind;        // 0 gaussian, 1 slp2d, 2 slp3d
  double denom;    // gaussian: (2.0 * sigma) * sigma
  double scale;    // multiplies the reference formula
};

__device__ __forceinline__ double kernel_from_r2(const KernelParams& kp, double r2) {
  double v;
  if (kp.kind == 0) {
    v = exp(-r2 / kp.denom);
  } else if (kp.kind == 1) {
    v = (-0.5 * log(r2)) / (2.0 * 3.141592653589793);
  } else {
    v = 1.0 / ((4.0 * 3.141592653589793) * sqrt(r2));
  }
  return kp.scale == 1.0 ? v : kp.scale * v;
}

// Regeneration fast path (mapped grid): k(r^2) = kernel_coef * kernel_shape(r^2),
// division-free (rsqrt / log / exp with the constant hoisted and folded into
// the operand vector).  Each differs from the reference formula by <= a few
// ulp, far below the 1e-12 parity bar.
__host__ __device__ __forceinline__ double kernel_coef(const KernelParams& kp) {
  if (kp.kind == 0) return kp.scale;
  if (kp.kind == 1) return kp.scale * (-0.5 / (2.0 * 3.141592653589793));
  return kp.scale / (4.0 * 3.141592653589793);
}

// 1/sqrt(x) for normal positive x (squared distances of distinct points):
// MUFU.RSQ64H seed (measured max rel. error 9.1e-7, tools/rsqrt_probe.cu) and
// one third-order correction y (1 + e/2 + 3e^2/8), e = 1 - x y^2 (measured
// 1.1e-16, same as libdevice rsqrt) -- 5 fp64 ops, no slow path.
__device__ __forceinline__ double rsqrt_pos(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

template <int KIND>
__device__ __forceinline__ double kernel_shape(double r2, double neg_inv_denom) {
  if (KIND == 0) return exp(r2 * neg_inv_denom);
  if (KIND == 1) return log(r2);
  return rsqrt_pos(r2);
}

__device__ __forceinline__ double r2_of(int d, const double* x, const double* y) {
  double d0 = __dadd_rn(x[0], -y[0]);
  double r2 = __dmul_rn(d0, d0);
  double d1 = __dadd_rn(x[1], -y[1]);
  r2 = __dadd_rn(r2, __dmul_rn(d1, d1));
  if (d == 3) {
    double d2 = __dadd_rn(x[2], -y[2]);
    r2 = __dadd_rn(r2, __dmul_rn(d2, d2));
  }
  return r2;
}

// ---------------------------------------------------------------------------
// Chebyshev node of a domain interval (chebyshev.py:36-37), numpy's order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double cheb_node(double lo, double hi, int t1, int p) {
  double arg = __ddiv_rn(__dmul_rn((double)(2 * t1 - 1), 3.141592653589793), (double)(2 * p));
  double c = cos(arg);
  return __dadd_rn(__dmul_rn(__dmul_rn(0.5, __dadd_rn(hi, -lo)), c),
                   __dmul_rn(0.5, __dadd_rn(hi, lo)));
}

// ---------------------------------------------------------------------------
// GEMM A-operand tiling.  Every deduplicated core / near block is stored
// pre-tiled for mma.sync.m16n8k8.f64 so a CTA stage (MT rows x KC cols) is one
// contiguous chunk and each lane's fragment (a0..a3) is 32 contiguous bytes:
//   [row tile][k chunk][m16 block][k8 block][lane][4]
// lane = g*4 + t holds A[g][t], A[g+8][t], A[g][t+4], A[g+8][t+4].
// ---------------------------------------------------------------------------
constexpr int kKC = 32;

// MT < 0 selects the "thin" layout of gemm_thin_kernel (htlr_gemm.cu): one row
// tile of M_pad = -MT rows, stored per 32-wide K chunk as
//   [k4 (8)][m8 (M_pad/8)][lane][1],  lane = (m%8)*4 + k%4
// i.e. the mma.m8n8k4 A fragment of every 8x4 sub-block is 256 contiguous bytes.
__host__ __device__ __forceinline__ int64_t tiled_offset(int m, int k, int MT, int K_pad) {
  if (MT < 0) {
    // thin layout: [k chunk][k4 pair][m8 tile][lane][2] -- a lane's operands
    // of two consecutive k4 steps are adjacent (one 16-byte shared load)
    const int M_pad = -MT;
    const int kc = k / kKC, kk = k % kKC;
    const int lane = (m & 7) * 4 + (kk & 3);
    const int k4 = kk >> 2;
    return ((int64_t)kc * (kKC / 8) + (k4 >> 1)) * (int64_t)(M_pad / 8 * 64) + (int64_t)((m >> 3) * 32 + lane) * 2 +
           (k4 & 1);
  }
  int rt = m / MT, mm = m % MT;
  int kc = k / kKC, kk = k % kKC;
  int mi = mm >> 4, r16 = mm & 15;
  int ki = kk >> 3, c8 = kk & 7;
  int g = r16 & 7, hi = r16 >> 3;
  int t = c8 & 3, hk = c8 >> 2;
  int lane = g * 4 + t;
  int reg = hi + 2 * hk;
  int64_t chunk = (int64_t)rt * (K_pad / kKC) + kc;
  return chunk * (int64_t)(MT * kKC) + (int64_t)((mi * (kKC / 8) + ki) * 128 + lane * 4 + reg);
}

// ---------------------------------------------------------------------------
// Cluster numbering: Morton (Z) order with the reference's child order
// (np.ndindex, last dimension fastest, grids.py:226-230): coordinate a's bit b
// sits at bit d*b + (d-1-a).  Every subtree is a contiguous id range at every
// deeper level, the parent of id c is c >> d, and the order of leaf boxes is
// the reference's DFS order of cluster-tree leaves.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t morton_encode(const int* c, int d, int bits) {
  int64_t id = 0;
  for (int b = 0; b < bits; ++b)
    for (int a = 0; a < d; ++a) id |= (int64_t)((c[a] >> b) & 1) << (d * b + (d - 1 - a));
  return id;
}

__host__ __device__ __forceinline__ void morton_decode(int64_t id, int d, int bits, int* c) {
  c[0] = c[1] = c[2] = 0;
  for (int b = 0; b < bits; ++b)
    for (int a = 0; a < d; ++a) c[a] |= (int)((id >> (d * b + (d - 1 - a))) & 1) << b;
}

}  // namespace htlr
