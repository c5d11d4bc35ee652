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
#include "htlr_mbarrier.cuh"

namespace htlr {

template <int PP, int KIND, int NS, int MINB>
__global__ void __launch_bounds__(PP * PP * 8 + 32, MINB)
    regen_sym_kernel(KernelParams kp, int level, const double* __restrict__ ax, const int* __restrict__ order,
                     int64_t t0, const int64_t* __restrict__ uptr, const int* __restrict__ ucols,
                     const double* __restrict__ V, int64_t vstride, double* __restrict__ OUT, int64_t ostride,
                     double coef) {
  constexpr int P = PP * PP * PP, HALF = PP / 2, U = PP * PP / 4;
  constexpr int NCT = PP * PP * 8, NCW = NCT / 32;   // consumer threads / warps
  constexpr int SE = P + 3 * PP;                     // staged doubles per source: V then 3 x PP coordinates
  constexpr int TE = 3 * PP * PP;                    // squared axis differences per source
  extern __shared__ __align__(16) double sm[];
  double* stage = sm;                      // NS x SE      (bulk copies)
  double* tab = stage + NS * SE;           // NS x TE      (producer warp)
  double* vt = tab + NS * TE;              // P            V[tau]
  double* xt = vt + P;                     // 3 x PP       tau coordinates
  double* racc = xt + 3 * PP;              // U x HALF x NCT row sums (thread-minor)
  uint64_t* full = reinterpret_cast<uint64_t*>(racc + U * HALF * NCT);
  uint64_t* ready = full + NS;
  uint64_t* empty = ready + NS;
  int* sig = reinterpret_cast<int*>(empty + NS);
  const double nid = -1.0 / kp.denom;
  const int row = order[blockIdx.x];   // own row (longest lists first)
  const int64_t tau = t0 + row;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int64_t e0 = uptr[row];
  const int ns = (int)(uptr[row + 1] - e0);

  if (t == 0) {
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&ready[q], 1);
      mbar_init(&empty[q], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
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
  if (t < NCT)
    for (int k = 0; k < U * HALF; ++k) racc[k * NCT + t] = 0.0;
  __syncthreads();

  if (warp == NCW) {
    // ---------------------------------------------------------- producer
    // bulk-copies source q + NS - 1 while the consumers work on earlier
    // ones; squares the axis differences of source q once it has landed
    auto issue = [&](int q) {
      const int slot = q % NS;
      if (q >= NS) mbar_wait(&empty[slot], (unsigned)(((q / NS) - 1) & 1));
      if (lane == 0) {
        const int sigma = ucols[e0 + q];
        int sc[3];
        morton_decode(sigma, 3, level, sc);
        sig[slot] = sigma;
        double* dst = stage + slot * SE;
        mbar_arrive_expect_tx(&full[slot], (unsigned)(SE * 8));
        bulk_g2s(dst, V + (int64_t)sigma * vstride, P * 8, &full[slot]);
        for (int a = 0; a < 3; ++a) bulk_g2s(dst + P + a * PP, ax + (int64_t)sc[a] * PP, PP * 8, &full[slot]);
      }
      __syncwarp();
    };
    for (int q = 0; q < ns && q < NS - 1; ++q) issue(q);
    for (int q = 0; q < ns; ++q) {
      const int slot = q % NS;
      mbar_wait(&full[slot], (unsigned)((q / NS) & 1));
      const double* eta = stage + slot * SE + P;
      double* tq = tab + slot * TE;
      for (int e = lane; e < TE; e += 32) {
        const int a = e / (PP * PP), i = (e / PP) % PP, j = e % PP;
        const double df = __dadd_rn(xt[a * PP + i], -eta[a * PP + j]);
        tq[e] = __dmul_rn(df, df);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[slot]);
      if (q + NS - 1 < ns) issue(q + NS - 1);
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int cg = t >> 3, s = t & 7;
  const int j2 = cg % PP, j3 = cg / PP, ih = s & 1;
  for (int q = 0; q < ns; ++q) {
    const int slot = q % NS;
    mbar_wait(&ready[slot], (unsigned)((q / NS) & 1));
    const double* vs = stage + slot * SE + cg * PP;   // V[sigma] of my PP columns
    const double* tq = tab + slot * TE;
    double vc[PP], dxr[HALF][PP], cacc[PP];
#pragma unroll
    for (int c = 0; c < PP; ++c) {
      vc[c] = vs[c];
      cacc[c] = 0.0;
    }
#pragma unroll
    for (int r = 0; r < HALF; ++r)
#pragma unroll
      for (int c = 0; c < PP; ++c) dxr[r][c] = tq[(ih * HALF + r) * PP + c];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int rg = (s >> 1) + 4 * k, i2 = rg % PP, i3 = rg / PP;
      const double yz = tq[PP * PP + i2 * PP + j2] + tq[2 * PP * PP + i3 * PP + j3];
      double wt[HALF], ra[HALF];
#pragma unroll
      for (int r = 0; r < HALF; ++r) {
        wt[r] = vt[rg * PP + ih * HALF + r];
        ra[r] = racc[(k * HALF + r) * NCT + t];
      }
#pragma unroll
      for (int r = 0; r < HALF; ++r)
#pragma unroll
        for (int c = 0; c < PP; ++c) {
          const double kv = kernel_shape<KIND>(dxr[r][c] + yz, nid);
          ra[r] = fma(kv, vc[c], ra[r]);
          cacc[c] = fma(kv, wt[r], cacc[c]);
        }
#pragma unroll
      for (int r = 0; r < HALF; ++r) racc[(k * HALF + r) * NCT + t] = ra[r];
    }
    const int sigma = sig[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
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
      double v = keep[0];
#pragma unroll
      for (int c = 1; c < H2; ++c)
        if (c == r3) v = keep[c];
      const int j1 = (hi ? H2 : 0) + r3;
      atomicAdd(OUT + (int64_t)sigma * ostride + cg * PP + j1, coef * v);
    }
  }
  // row sums: reduce over the 4 column groups of the warp (lanes xor 8, 16),
  // then one RED per row from the lanes of column group 0 mod 4
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int rg = (s >> 1) + 4 * k;
#pragma unroll
    for (int r = 0; r < HALF; ++r) {
      double v = racc[(k * HALF + r) * NCT + t];
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

template <int PP, int KIND, int NS, int MINB>
static void sym_k(KernelParams kp, int level, const double* ax, const int* order, int64_t nrows, int64_t t0,
                  const int64_t* uptr, const int* ucols, const double* V, int64_t vstride, double* OUT,
                  int64_t ostride, double coef, cudaStream_t st) {
  constexpr int P = PP * PP * PP, NCT = PP * PP * 8;
  const size_t smem = sizeof(double) * ((size_t)NS * (P + 3 * PP + 3 * PP * PP) + P + 3 * PP +
                                        (size_t)(PP * PP / 4) * (PP / 2) * NCT) +
                      3 * NS * sizeof(uint64_t) + NS * sizeof(int);
  cudaFuncSetAttribute(regen_sym_kernel<PP, KIND, NS, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  regen_sym_kernel<PP, KIND, NS, MINB><<<(unsigned)nrows, NCT + 32, smem, st>>>(kp, level, ax, order, t0, uptr, ucols,
                                                                          V, vstride, OUT, ostride, coef);
}

template <int PP>
static void sym_p(KernelParams kp, int level, const double* ax, const int* order, int64_t nrows, int64_t t0,
                  const int64_t* uptr, const int* ucols, const double* V, int64_t vstride, double* OUT,
                  int64_t ostride, cudaStream_t st) {
  const double coef = kernel_coef(kp);
  // 12-source ring, two CTAs per SM (the Gaussian's exp needs the
  // registers of one)
  if (kp.kind == 0)
    sym_k<PP, 0, 12, 1>(kp, level, ax, order, nrows, t0, uptr, ucols, V, vstride, OUT, ostride, coef, st);
  else
    sym_k<PP, 2, 12, 2>(kp, level, ax, order, nrows, t0, uptr, ucols, V, vstride, OUT, ostride, coef, st);
}

void launch_regen_sym(const KernelParams& kp, int pp, int level, const double* ax, const int* order, int64_t nrows,
                      int64_t t0, const int64_t* uptr, const int* ucols, const double* V, int64_t vstride, double* OUT,
                      int64_t ostride, cudaStream_t st) {
  if (nrows <= 0) return;
  if (pp == 4)
    sym_p<4>(kp, level, ax, order, nrows, t0, uptr, ucols, V, vstride, OUT, ostride, st);
  else
    sym_p<6>(kp, level, ax, order, nrows, t0, uptr, ucols, V, vstride, OUT, ostride, st);
}

void launch_near_weight(int sL, int L, const double* widths, const double* ub, int K_pad, double* V, int64_t nleaf,
                        cudaStream_t st) {
  const int64_t total = nleaf * sL * sL * sL;
  if (total <= 0) return;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  near_weight_kernel<<<grid, 256, 0, st>>>(sL, L, widths, ub, K_pad, V, nleaf);
}

}  // namespace htlr
