// Mapped grid (BASELINE config 5): symmetric regeneration of the admissible
// cores and near blocks, one kernel evaluation per UNORDERED cluster pair.
//
// The kernels are symmetric, k(x, y) = k(y, x), and the block lists are
// symmetric ((tau, sigma) admissible <=> (sigma, tau) admissible, the same
// Chebyshev nodes / point coordinates on both sides), so the regenerated
// block of (sigma, tau) is the transpose of that of (tau, sigma) -- bit for
// bit, since r^2 is formed from squared per-axis differences.  Each CTA owns
// a target cluster tau and walks its sources sigma > tau only:
//
//   OUT[tau]   += coef * sum_j k(x_i, y_j) V[sigma][j]      (row sums)
//   OUT[sigma] += coef * sum_i k(x_i, y_j) V[tau][i]        (column sums)
//
// which halves the fp64 work of the dominant kernel of the mapped matvec
// (rsqrt seed + third-order correction + 2 FMAs per entry instead of 2 x
// (correction + 1 FMA)).  For the admissible levels V = W (source-weighted
// upward data), for the near field V = w (*) u (cell weight times input);
// the near self pair tau = tau (the diagonal excluded) is applied by the
// one-sided kernel of htlr_mapped.cu before this one.
//
// Thread layout (PP = p or the leaf side, P = PP^3 points per cluster):
// thread t = cg * 8 + s, column group cg = (j2, j3) (PP columns j1), slice s
// owns row units u = s + 8 k (k < PP^2 / 4), unit u = half (u & 1) of the
// rows i1 of row group rg = u >> 1 = (i2, i3).  Column sums are reduced
// over the 8 slices of a column group by shuffles and added with fp64 RED
// per sigma.  Row sums live in shared memory (thread-minor, loaded/stored once per 3 x PP tile) so that
// two CTAs fit an SM: the kernel is fp64-latency bound at one.  Sources are staged
// eight at a time with cp.async, double buffered.
#include <algorithm>

#include "htlr_kernels.h"

namespace htlr {

namespace {

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

}  // namespace

template <int PP, int KIND, int SB, int MINB, bool DXS = false>
__global__ void __launch_bounds__(PP * PP * 8, MINB)
    regen_sym_kernel(KernelParams kp, int level, const double* __restrict__ ax, const int* __restrict__ order,
                     const int64_t* __restrict__ uptr, const int* __restrict__ ucols, const double* __restrict__ V,
                     int64_t vstride, double* __restrict__ OUT, int64_t ostride, double coef) {
  constexpr int P = PP * PP * PP, HALF = PP / 2, U = PP * PP / 4;
  constexpr int SE = P + 3 * PP;   // staged doubles per source: V then 3 x PP coordinates
  extern __shared__ __align__(16) double sm[];
  double* stage = sm;                         // 2 x SB x SE
  double* tab = stage + 2 * SB * SE;          // SB x 3 x PP x PP   squared axis differences
  double* vt = tab + SB * 3 * PP * PP;        // P                  V[tau]
  double* xt = vt + P;                        // 3 x PP             tau coordinates
  double* racc = xt + 3 * PP;                 // U x HALF x NT      row sums (thread-minor)
  constexpr int NT = PP * PP * 8;
  const double nid = -1.0 / kp.denom;
  const int tau = order[blockIdx.x];
  const int t = threadIdx.x, cg = t >> 3, s = t & 7;
  const int j2 = cg % PP, j3 = cg / PP, ih = s & 1;
  const int64_t e0 = uptr[tau], ns = uptr[tau + 1] - e0;

  auto issue = [&](int64_t b) {   // stage sources [b*SB, b*SB + SB) into buffer b & 1
    double* dst = stage + (b & 1) * SB * SE;
    const int nsb = (int)min((int64_t)SB, ns - b * SB);
    for (int e = t; e < nsb * SE; e += blockDim.x) {
      const int q = e / SE, r = e % SE;
      const int sigma = ucols[e0 + b * SB + q];
      if (r < P) {
        cp_async8(dst + e, V + (int64_t)sigma * vstride + r);
      } else {
        const int a = (r - P) / PP, k = (r - P) % PP;
        int sc[3];
        morton_decode(sigma, 3, level, sc);
        cp_async8(dst + e, ax + (int64_t)sc[a] * PP + k);
      }
    }
    cp_async_commit();
  };

  {
    int tc[3];
    morton_decode(tau, 3, level, tc);
    for (int e = t; e < P + 3 * PP; e += blockDim.x) {
      if (e < P)
        vt[e] = V[(int64_t)tau * vstride + e];
      else
        xt[e - P] = ax[(int64_t)tc[(e - P) / PP] * PP + (e - P) % PP];
    }
  }
#pragma unroll
  for (int k = 0; k < U * HALF; ++k) racc[k * NT + t] = 0.0;

  const int64_t nbatch = (ns + SB - 1) / SB;
  if (nbatch > 0) issue(0);
  for (int64_t b = 0; b < nbatch; ++b) {
    if (b + 1 < nbatch)
      issue(b + 1);
    else
      cp_async_commit();   // empty group keeps the wait count uniform
    cp_async_wait1();
    __syncthreads();
    const double* sb = stage + (b & 1) * SB * SE;
    const int nsb = (int)min((int64_t)SB, ns - b * SB);
    for (int e = t; e < nsb * 3 * PP * PP; e += blockDim.x) {
      const int q = e / (3 * PP * PP), r = e % (3 * PP * PP);
      const int a = r / (PP * PP), i = (r / PP) % PP, j = r % PP;
      const double df = __dadd_rn(xt[a * PP + i], -sb[q * SE + P + a * PP + j]);
      tab[e] = __dmul_rn(df, df);
    }
    __syncthreads();
    for (int q = 0; q < nsb; ++q) {
      const double* vs = sb + q * SE + cg * PP;   // V[sigma] of my PP columns
      const double* tq = tab + q * 3 * PP * PP;
      double vc[PP], dxr[HALF][PP], cacc[PP];
#pragma unroll
      for (int c = 0; c < PP; ++c) {
        vc[c] = vs[c];
        cacc[c] = 0.0;
      }
      if (!DXS) {
#pragma unroll
        for (int r = 0; r < HALF; ++r)
#pragma unroll
          for (int c = 0; c < PP; ++c) dxr[r][c] = tq[(ih * HALF + r) * PP + c];
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int rg = (s >> 1) + 4 * k, i2 = rg % PP, i3 = rg / PP;
        const double yz = tq[PP * PP + i2 * PP + j2] + tq[2 * PP * PP + i3 * PP + j3];
        double wt[HALF], ra[HALF];
#pragma unroll
        for (int r = 0; r < HALF; ++r) {
          wt[r] = vt[rg * PP + ih * HALF + r];
          ra[r] = racc[(k * HALF + r) * NT + t];
        }
#pragma unroll
        for (int r = 0; r < HALF; ++r)
#pragma unroll
          for (int c = 0; c < PP; ++c) {
            const double dx = DXS ? tq[(ih * HALF + r) * PP + c] : dxr[r][c];
            const double kv = kernel_shape<KIND>(dx + yz, nid);
            ra[r] = fma(kv, vc[c], ra[r]);
            cacc[c] = fma(kv, wt[r], cacc[c]);
          }
#pragma unroll
        for (int r = 0; r < HALF; ++r) racc[(k * HALF + r) * NT + t] = ra[r];
      }
      // column sums over the 8 slices (lanes xor 4, 2, 1): after the xor-4
      // step a lane keeps the half of the columns selected by its bit 2
      constexpr int H2 = PP / 2;
      const bool hi = (s & 4) != 0;
      double keep[H2];
#pragma unroll
      for (int c = 0; c < H2; ++c) {
        const double send = hi ? cacc[c] : cacc[H2 + c];
        const double mine = hi ? cacc[H2 + c] : cacc[c];
        keep[c] = mine + __shfl_xor_sync(0xffffffffu, send, 4);
      }
#pragma unroll
      for (int c = 0; c < H2; ++c) {
        keep[c] += __shfl_xor_sync(0xffffffffu, keep[c], 2);
        keep[c] += __shfl_xor_sync(0xffffffffu, keep[c], 1);
      }
      const int r3 = s & 3;
      if (r3 < H2) {
        const int sigma = ucols[e0 + b * SB + q];
        double v = keep[0];
#pragma unroll
        for (int c = 1; c < H2; ++c)
          if (c == r3) v = keep[c];
        const int j1 = (hi ? H2 : 0) + r3;
        atomicAdd(OUT + (int64_t)sigma * ostride + cg * PP + j1, coef * v);
      }
    }
    __syncthreads();   // buffer b & 1 and tab are rewritten next iteration
  }
  // row sums: reduce over the 4 column groups of the warp (lanes xor 8, 16),
  // then one RED per row from the lanes of column group 0 mod 4
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int rg = (s >> 1) + 4 * k;
#pragma unroll
    for (int r = 0; r < HALF; ++r) {
      double v = racc[(k * HALF + r) * NT + t];
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      if ((cg & 3) == 0) atomicAdd(OUT + (int64_t)tau * ostride + rg * PP + ih * HALF + r, coef * v);
    }
  }
}

// V[leaf][j] = w_j u[leaf][j] (near-field source vector, both directions)
__global__ void near_weight_kernel(int sL, int L, const double* __restrict__ widths, const double* __restrict__ ub,
                                   int K_pad, double* __restrict__ V, int64_t nleaf) {
  const int P = sL * sL * sL;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nleaf * P;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t leaf = e / P;
    const int j = (int)(e % P);
    int c[3];
    morton_decode(leaf, 3, L, c);
    const int j1 = j % sL, j2 = (j / sL) % sL, j3 = j / (sL * sL);
    const double w = widths[c[0] * sL + j1] * widths[c[1] * sL + j2] * widths[c[2] * sL + j3];
    V[e] = w * ub[leaf * K_pad + j];
  }
}

bool regen_sym_supported(int d, int pp) { return d == 3 && (pp == 4 || pp == 6); }

template <int PP, int KIND, int SB, int MINB, bool DXS = false>
static void sym_k(KernelParams kp, int level, const double* ax, const int* order, int64_t nrows,
                  const int64_t* uptr, const int* ucols, const double* V, int64_t vstride, double* OUT,
                  int64_t ostride, double coef, cudaStream_t st) {
  constexpr int P = PP * PP * PP;
  const size_t smem =
      sizeof(double) * (2 * SB * (P + 3 * PP) + SB * 3 * PP * PP + P + 3 * PP + (size_t)(P / 8) * PP * PP * 8);
  cudaFuncSetAttribute(regen_sym_kernel<PP, KIND, SB, MINB, DXS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  regen_sym_kernel<PP, KIND, SB, MINB, DXS><<<(unsigned)nrows, PP * PP * 8, smem, st>>>(kp, level, ax, order, uptr, ucols, V,
                                                                         vstride, OUT, ostride, coef);
}

template <int PP>
static void sym_p(KernelParams kp, int level, const double* ax, const int* order, int64_t nrows,
                  const int64_t* uptr, const int* ucols, const double* V, int64_t vstride, double* OUT,
                  int64_t ostride, cudaStream_t st) {
  const double coef = kernel_coef(kp);
  // 8 sources per stage, two CTAs per SM (measured: 3 CTAs per SM with the
  // x-differences in shared memory, or 4-source stages, are 1-8% slower)
  if (kp.kind == 0)
    sym_k<PP, 0, 8, 2>(kp, level, ax, order, nrows, uptr, ucols, V, vstride, OUT, ostride, coef, st);
  else
    sym_k<PP, 2, 8, 2>(kp, level, ax, order, nrows, uptr, ucols, V, vstride, OUT, ostride, coef, st);
}

void launch_regen_sym(const KernelParams& kp, int pp, int level, const double* ax, const int* order, int64_t nrows,
                      const int64_t* uptr, const int* ucols, const double* V, int64_t vstride, double* OUT,
                      int64_t ostride, cudaStream_t st) {
  if (nrows <= 0) return;
  if (pp == 4)
    sym_p<4>(kp, level, ax, order, nrows, uptr, ucols, V, vstride, OUT, ostride, st);
  else
    sym_p<6>(kp, level, ax, order, nrows, uptr, ucols, V, vstride, OUT, ostride, st);
}

void launch_near_weight(int sL, int L, const double* widths, const double* ub, int K_pad, double* V, int64_t nleaf,
                        cudaStream_t st) {
  const int64_t total = nleaf * sL * sL * sL;
  if (total <= 0) return;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  near_weight_kernel<<<grid, 256, 0, st>>>(sL, L, widths, ub, K_pad, V, nleaf);
}

}  // namespace htlr
