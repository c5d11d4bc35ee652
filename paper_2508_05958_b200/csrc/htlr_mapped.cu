// Mapped quasi-uniform tensor grid (BASELINE config 5) on sm_100a.
//
// The reference has only UniformGrid (grids.py:18-43); its algorithm is
// applied to the mapped geometry (oracle/htlr_oracle.py, MappedGeometry):
// points x_i = phi((i+1/2)/n), cells [phi(i/n), phi((i+1)/n)], Nystrom weight
// w_i = product of cell widths.  Nothing is translation invariant, and the
// per-block cores (806 GB for config 5) do not fit one GPU, so:
//   * factors are per (level, interval): Chebyshev nodes of the mapped
//     interval (chebyshev.py:31-38) and the raw Lagrange factor at the mapped
//     points (chebyshev.py:52-66); the source side carries the cell widths.
//     Using the raw (non-orthonormal) factors instead of Q with R folded into
//     the core (blocks.py:146-163) is the same operator;
//   * cores are regenerated inside the contraction: each CTA owns one target
//     cluster and, for every source of its list, evaluates k(xi_t, eta_s) on
//     the fly and accumulates H_t += sum_s k(xi_t, eta_s) W_s (kernel
//     sampling fused with the core contraction; fp64 CUDA-core bound);
//   * near blocks K_ij w_j are regenerated the same way; the diagonal is a
//     per-point integral of k(x_i, .) over its rectangular, off-centre cell
//     (kernels.py:222-249 generalised to 2^d rectangular corner boxes).
#include <algorithm>

#include "htlr_kernels.h"

namespace htlr {

// ---------------------------------------------------------------------------
// per (level, interval) Chebyshev nodes and raw Lagrange factors
// ---------------------------------------------------------------------------
__device__ __forceinline__ double cheb_node_m(double lo, double hi, int t1, int p) {
  double arg = __ddiv_rn(__dmul_rn((double)(2 * t1 - 1), 3.141592653589793), (double)(2 * p));
  return __dadd_rn(__dmul_rn(__dmul_rn(0.5, __dadd_rn(hi, -lo)), cos(arg)), __dmul_rn(0.5, __dadd_rn(hi, lo)));
}

__global__ void mapped_factor_kernel(const MappedFactorJob* __restrict__ jobs, int njobs,
                                     const double* __restrict__ bounds,
                                     const double* __restrict__ coords, const double* __restrict__ widths, int p) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  int acc = 0, ji = -1, j = 0;
  for (int q = 0; q < njobs; ++q) {
    if (gid < acc + jobs[q].nint) {
      ji = q;
      j = gid - acc;
      break;
    }
    acc += jobs[q].nint;
  }
  if (ji < 0) return;
  const MappedFactorJob jb = jobs[ji];
  const int s = jb.side;
  const double lo = bounds[j * s], hi = bounds[(j + 1) * s];
  double nodes[kMaxRank];
  for (int t = 0; t < p; ++t) {
    nodes[t] = cheb_node_m(lo, hi, t + 1, p);
    jb.nodes[j * p + t] = nodes[t];
  }
  for (int i = 0; i < s; ++i) {
    const double x = coords[j * s + i];
    const double w = widths[j * s + i];
    for (int t = 0; t < p; ++t) {
      double prod = 1.0;
      bool first = true;
      for (int q = 0; q < p; ++q) {
        if (q == t) continue;
        double f = __ddiv_rn(__dadd_rn(x, -nodes[q]), __dadd_rn(nodes[t], -nodes[q]));
        prod = first ? f : __dmul_rn(prod, f);
        first = false;
      }
      jb.L[((int64_t)j * s + i) * p + t] = prod;
      jb.WL[((int64_t)j * s + i) * p + t] = w * prod;
    }
  }
}

// ---------------------------------------------------------------------------
// per-point cell integral of k(x_i, .) (the Nystrom diagonal)
// ---------------------------------------------------------------------------
template <int KIND, int Q>
__global__ void mapped_diag_kernel(KernelParams kp, int d, int n, int q_rt, const double* __restrict__ gx_g,
                                   const double* __restrict__ gw_g, const double* __restrict__ bounds,
                                   const double* __restrict__ coords, double* __restrict__ out, int64_t npts) {
  // one warp per point: 2^d corner boxes x d Duffy pyramids (warp-uniform
  // loops) x q^d Gauss points of the radially graded rule (lanes), shuffle
  // reduction; k = coef * shape(r^2) with the division-free shapes of the
  // regeneration kernels.  Q = q as a constant turns the Gauss-index splits
  // into multiplies (0: runtime q).
  const int q = Q ? Q : q_rt;
  __shared__ double gx[64], gw[64];
  for (int i = threadIdx.x; i < q; i += blockDim.x) {
    gx[i] = gx_g[i];
    gw[i] = gw_g[i];
  }
  __syncthreads();
  const double nid = -1.0 / kp.denom;
  const double coef = kernel_coef(kp);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int qd = (d == 2) ? q * q : q * q * q;
  const int ncorner = 1 << d;
  for (int64_t pt = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); pt < npts; pt += warps) {
    int idx[3] = {(int)(pt % n), (int)((pt / n) % n), d == 3 ? (int)(pt / ((int64_t)n * n)) : 0};
    double lo_e[3] = {0, 0, 0}, hi_e[3] = {0, 0, 0};
    for (int a = 0; a < d; ++a) {
      const double x = coords[idx[a]];
      lo_e[a] = x - bounds[idx[a]];
      hi_e[a] = bounds[idx[a] + 1] - x;
    }
    double acc = 0.0;
    for (int corner = 0; corner < ncorner; ++corner) {
      double ext[3] = {0, 0, 0}, vol = 1.0;
      for (int a = 0; a < d; ++a) {
        ext[a] = ((corner >> (d - 1 - a)) & 1) ? hi_e[a] : lo_e[a];
        vol = vol * ext[a];
      }
      for (int axis = 0; axis < d; ++axis) {
        for (int pidx = lane; pidx < qd; pidx += 32) {
          const int ii[3] = {pidx % q, (pidx / q) % q, pidx / (q * q)};
          const double tt = gx[ii[axis]];
          const double t = tt * tt * tt;
          double w = 1.0, r2 = 0.0;
          for (int a = 0; a < d; ++a) {
            const double c = (a == axis) ? ext[a] * t : ext[a] * t * gx[ii[a]];
            r2 = __dadd_rn(r2, __dmul_rn(c, c));
            w = w * ((a == axis) ? 3.0 * (tt * tt) * gw[ii[a]] : gw[ii[a]]);
          }
          const double jac = vol * ((d == 2) ? t : t * t);
          acc += kernel_shape<KIND>(r2, nid) * (jac * w);
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) out[pt] = coef * acc;
  }
}

// ---------------------------------------------------------------------------
// admissible blocks: kernel sampling fused with the core contraction
//   H[tau][r][t] = sum_{sigma in list(tau)} sum_s k(xi_t, eta_s) W[sigma][r][s]
// one CTA per target cluster; thread = target node multi-index t (F-order).
// r^2 is assembled from per-dimension squared differences, in numpy's order
// ((dx^2 + dy^2) + dz^2).  PP = p as a compile-time constant keeps the
// innermost x-differences in registers (0: generic, slower).
// ---------------------------------------------------------------------------
template <int RB, int PP, int KIND>
__global__ void regen_adm_kernel(KernelParams kp, int d, int p_rt, int level, const double* __restrict__ nodes,
                                 const int64_t* __restrict__ rowptr, const int* __restrict__ cols, int64_t t0,
                                 const double* __restrict__ W, int K_pad, double* __restrict__ H, int R, int r0) {
  // SB sources are staged per barrier pair (fewer barriers, more loads in
  // flight); their W vectors arrive pre-scaled by the kernel constant
  constexpr int SB = RB >= 16 ? 1 : 4;
  extern __shared__ double sm[];
  const double nid = -1.0 / kp.denom;
  const int p = PP ? PP : p_rt;
  const int P = (d == 2) ? p * p : p * p * p;
  double* sW = sm;                            // SB x RB x P
  double* sEta = sW + SB * RB * P;            // SB x 3 x kMaxRank
  double* sYZ = sEta + SB * 3 * kMaxRank;     // per thread: dy^2[p], dz^2[p]
  const int64_t row = blockIdx.x;
  const int64_t tau = t0 + row;
  int tc[3];
  morton_decode(tau, d, level, tc);
  const int t = threadIdx.x;
  const bool act = t < P;
  const int t1 = t % p, t2 = (t / p) % p, t3 = t / (p * p);
  const double xi0 = act ? nodes[tc[0] * p + t1] : 0.0;
  const double xi1 = act ? nodes[tc[1] * p + t2] : 0.0;
  const double xi2 = (act && d == 3) ? nodes[tc[2] * p + t3] : 0.0;
  double* myYZ = sYZ + (int64_t)t * 2 * p;
  double acc[RB];
#pragma unroll
  for (int q = 0; q < RB; ++q) acc[q] = 0.0;
  const int nrb = min(RB, R - r0);
  const double coef = kernel_coef(kp);
  const int64_t e_end = rowptr[row + 1];
  for (int64_t e0 = rowptr[row]; e0 < e_end; e0 += SB) {
    const int nsb = (int)min((int64_t)SB, e_end - e0);
    __syncthreads();
    for (int i = threadIdx.x; i < nsb * d * p; i += blockDim.x) {
      const int b = i / (d * p), rem = i % (d * p), a = rem / p, k = rem % p;
      const int sigma = cols[e0 + b];
      int sc[3];
      morton_decode(sigma, d, level, sc);
      sEta[(b * 3 + a) * kMaxRank + k] = nodes[sc[a] * p + k];
    }
    for (int i = threadIdx.x; i < nsb * nrb * P; i += blockDim.x) {
      const int b = i / (nrb * P), rem = i % (nrb * P), q = rem / P, sidx = rem % P;
      const int sigma = cols[e0 + b];
      sW[(b * RB + q) * P + sidx] = coef * W[((int64_t)sigma * R + r0 + q) * K_pad + sidx];
    }
    __syncthreads();
    if (!act) continue;
    for (int b = 0; b < nsb; ++b) {
      const double* eta = sEta + b * 3 * kMaxRank;
      const double* wb = sW + b * RB * P;
      double dx2[PP ? PP : kMaxRank];
#pragma unroll
      for (int s = 0; s < (PP ? PP : kMaxRank); ++s) {
        if (s < p) {
          const double a = __dadd_rn(xi0, -eta[s]);
          dx2[s] = __dmul_rn(a, a);
        }
      }
      for (int s = 0; s < p; ++s) {
        const double bb = __dadd_rn(xi1, -eta[kMaxRank + s]);
        myYZ[s] = __dmul_rn(bb, bb);
        if (d == 3) {
          const double c = __dadd_rn(xi2, -eta[2 * kMaxRank + s]);
          myYZ[p + s] = __dmul_rn(c, c);
        }
      }
      const int n3 = (d == 3) ? p : 1;
      for (int s3 = 0; s3 < n3; ++s3) {
        const double z2 = (d == 3) ? myYZ[p + s3] : 0.0;
        for (int s2 = 0; s2 < p; ++s2) {
          const double yz = myYZ[s2] + z2;
          const double* w = wb + (s2 + p * s3) * p;
#pragma unroll
          for (int s1 = 0; s1 < (PP ? PP : kMaxRank); ++s1) {
            if (s1 < p) {
              const double kv = kernel_shape<KIND>(dx2[s1] + yz, nid);
#pragma unroll
              for (int q = 0; q < RB; ++q)
                if (q < nrb) acc[q] += kv * w[q * P + s1];
            }
          }
        }
      }
    }
  }
  if (act)
    for (int q = 0; q < nrb; ++q) H[(tau * R + r0 + q) * (int64_t)P + t] = acc[q];
}

// ---------------------------------------------------------------------------
// inadmissible blocks: Y[tau][r][i] = sum_sigma sum_j k(x_i, y_j) w_j u_j,
// the coincident pair skipped (its value is the per-point cell integral,
// added by the downward kernel); thread = target point i.
// ---------------------------------------------------------------------------
template <int RB, int SS, int KIND>
__global__ void regen_near_kernel(KernelParams kp, int d, int sL_rt, int L, const double* __restrict__ coords,
                                  const double* __restrict__ widths, const int64_t* __restrict__ rowptr,
                                  const int* __restrict__ cols, int64_t t0, const double* __restrict__ ub, int K_pad,
                                  double* __restrict__ Y, int R, int r0) {
  constexpr int SB = RB >= 16 ? 1 : 4;
  extern __shared__ double sm[];
  const double nid = -1.0 / kp.denom;
  const int sL = SS ? SS : sL_rt;
  const int P = (d == 2) ? sL * sL : sL * sL * sL;
  double* sV = sm;                   // SB x RB x P   (c w_j u_j)
  double* sY = sV + SB * RB * P;     // SB x 3 x 16   (source coordinates)
  double* sYZ = sY + SB * 3 * 16;    // per thread dy^2[sL], dz^2[sL]
  const int64_t row = blockIdx.x;
  const int64_t tau = t0 + row;
  int tc[3];
  morton_decode(tau, d, L, tc);
  const int i = threadIdx.x;
  const bool act = i < P;
  const int i1 = i % sL, i2 = (i / sL) % sL, i3 = i / (sL * sL);
  const double x0 = act ? coords[tc[0] * sL + i1] : 0.0;
  const double x1 = act ? coords[tc[1] * sL + i2] : 0.0;
  const double x2 = (act && d == 3) ? coords[tc[2] * sL + i3] : 0.0;
  double* myYZ = sYZ + (int64_t)i * 2 * sL;
  double acc[RB];
#pragma unroll
  for (int q = 0; q < RB; ++q) acc[q] = 0.0;
  const int nrb = min(RB, R - r0);
  const double coef = kernel_coef(kp);
  const int64_t e_end = rowptr[row + 1];
  for (int64_t e0 = rowptr[row]; e0 < e_end; e0 += SB) {
    const int nsb = (int)min((int64_t)SB, e_end - e0);
    __syncthreads();
    for (int k = threadIdx.x; k < nsb * d * sL; k += blockDim.x) {
      const int b = k / (d * sL), rem = k % (d * sL), a = rem / sL, j = rem % sL;
      int sc[3];
      morton_decode(cols[e0 + b], d, L, sc);
      sY[(b * 3 + a) * 16 + j] = coords[sc[a] * sL + j];
    }
    for (int k = threadIdx.x; k < nsb * nrb * P; k += blockDim.x) {
      const int b = k / (nrb * P), rem = k % (nrb * P), q = rem / P, j = rem % P;
      const int sigma = cols[e0 + b];
      int sc[3];
      morton_decode(sigma, d, L, sc);
      const int j1 = j % sL, j2 = (j / sL) % sL, j3 = j / (sL * sL);
      double w = widths[sc[0] * sL + j1] * widths[sc[1] * sL + j2];
      if (d == 3) w = w * widths[sc[2] * sL + j3];
      sV[(b * RB + q) * P + j] = coef * (w * ub[((int64_t)sigma * R + r0 + q) * K_pad + j]);
    }
    __syncthreads();
    if (!act) continue;
    for (int b = 0; b < nsb; ++b) {
      const bool self = cols[e0 + b] == tau;
      const double* yb = sY + b * 3 * 16;
      const double* vb = sV + b * RB * P;
      double dx2[SS ? SS : 16];
#pragma unroll
      for (int s = 0; s < (SS ? SS : 16); ++s) {
        if (s < sL) {
          const double a = __dadd_rn(x0, -yb[s]);
          dx2[s] = __dmul_rn(a, a);
        }
      }
      for (int s = 0; s < sL; ++s) {
        const double bb = __dadd_rn(x1, -yb[16 + s]);
        myYZ[s] = __dmul_rn(bb, bb);
        if (d == 3) {
          const double c = __dadd_rn(x2, -yb[32 + s]);
          myYZ[sL + s] = __dmul_rn(c, c);
        }
      }
      const int n3 = (d == 3) ? sL : 1;
      for (int j3 = 0; j3 < n3; ++j3) {
        const double z2 = (d == 3) ? myYZ[sL + j3] : 0.0;
        for (int j2 = 0; j2 < sL; ++j2) {
          const double yz = myYZ[j2] + z2;
          const int jb = (j2 + sL * j3) * sL;
          const double* v = vb + jb;
#pragma unroll
          for (int j1 = 0; j1 < (SS ? SS : 16); ++j1) {
            if (j1 < sL) {
              if (self && jb + j1 == i) continue;
              const double kv = kernel_shape<KIND>(dx2[j1] + yz, nid);
#pragma unroll
              for (int q = 0; q < RB; ++q)
                if (q < nrb) acc[q] += kv * v[q * P + j1];
            }
          }
        }
      }
    }
  }
  if (act)
    for (int q = 0; q < nrb; ++q) Y[(tau * R + r0 + q) * (int64_t)P + i] = acc[q];
}

// one block of the regenerated operator, materialised for export (parity)
__global__ void mapped_core_export_kernel(KernelParams kp, int d, int p, const double* __restrict__ nt,
                                          const double* __restrict__ ns, double* __restrict__ out) {
  const int P = (d == 2) ? p * p : p * p * p;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)P * P;
       e += (int64_t)gridDim.x * blockDim.x) {
    int ti = (int)(e % P), si = (int)(e / P);
    double x[3], y[3];
    for (int a = 0; a < d; ++a) {
      x[a] = nt[a * p + ti % p];
      y[a] = ns[a * p + si % p];
      ti /= p;
      si /= p;
    }
    out[e] = kernel_from_r2(kp, r2_of(d, x, y));
  }
}

__global__ void mapped_near_export_kernel(KernelParams kp, int d, int sL, const double* __restrict__ xt,
                                          const double* __restrict__ ys, const double* __restrict__ ws, int self,
                                          double* __restrict__ out) {
  const int P = (d == 2) ? sL * sL : sL * sL * sL;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)P * P;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / P), j = (int)(e % P);
    if (self && i == j) {
      out[e] = 0.0;
      continue;
    }
    double x[3], y[3];
    int ii = i, jj = j;
    double w = 1.0;
    for (int a = 0; a < d; ++a) {
      x[a] = xt[a * sL + ii % sL];
      y[a] = ys[a * sL + jj % sL];
      w = w * ws[a * sL + jj % sL];
      ii /= sL;
      jj /= sL;
    }
    out[e] = kernel_from_r2(kp, r2_of(d, x, y)) * w;
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
void launch_mapped_factors(const MappedFactorJob* jobs, int njobs, int total_intervals, const double* bounds,
                           const double* coords, const double* widths, int p, cudaStream_t st) {
  if (total_intervals <= 0) return;
  mapped_factor_kernel<<<(total_intervals + 63) / 64, 64, 0, st>>>(jobs, njobs, bounds, coords, widths, p);
}

// 3-D fast path (q = Q): the point-independent factors of every (pyramid
// axis, Gauss point) pair -- the graded coordinate factors f_a and the weight
// t^2 * prod(w) -- are tabulated once per CTA in shared memory, so an
// evaluation is r^2 = sum (ext_a f_a)^2, one shape evaluation and one FMA.
template <int KIND, int Q>
__global__ void __launch_bounds__(256) mapped_diag3_kernel(KernelParams kp, int n, const double* __restrict__ gx_g,
                                                          const double* __restrict__ gw_g,
                                                          const double* __restrict__ bounds,
                                                          const double* __restrict__ coords,
                                                          double* __restrict__ out, int64_t npts) {
  constexpr int QD = Q * Q * Q;
  extern __shared__ double tab[];   // [axis][pidx] x {f0, f1, f2, wt}
  for (int e = threadIdx.x; e < 3 * QD; e += blockDim.x) {
    const int axis = e / QD, pidx = e % QD;
    const int ii[3] = {pidx % Q, (pidx / Q) % Q, pidx / (Q * Q)};
    const double tt = gx_g[ii[axis]];
    const double t = tt * tt * tt;
    double w = 1.0;
    for (int a = 0; a < 3; ++a) {
      tab[e * 4 + a] = (a == axis) ? t : t * gx_g[ii[a]];
      w = w * ((a == axis) ? 3.0 * (tt * tt) * gw_g[ii[a]] : gw_g[ii[a]]);
    }
    tab[e * 4 + 3] = (t * t) * w;
  }
  __syncthreads();
  const double nid = -1.0 / kp.denom;
  const double coef = kernel_coef(kp);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t pt = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); pt < npts; pt += warps) {
    const int idx[3] = {(int)(pt % n), (int)((pt / n) % n), (int)(pt / ((int64_t)n * n))};
    double lo_e[3], hi_e[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double x = coords[idx[a]];
      lo_e[a] = x - bounds[idx[a]];
      hi_e[a] = bounds[idx[a] + 1] - x;
    }
    double acc = 0.0;
#pragma unroll 1
    for (int corner = 0; corner < 8; ++corner) {
      const double e0 = (corner & 4) ? hi_e[0] : lo_e[0];
      const double e1 = (corner & 2) ? hi_e[1] : lo_e[1];
      const double e2 = (corner & 1) ? hi_e[2] : lo_e[2];
      const double vol = (e0 * e1) * e2;
      for (int e = lane; e < 3 * QD; e += 32) {
        const double2 f01 = *reinterpret_cast<const double2*>(tab + e * 4);
        const double2 f2w = *reinterpret_cast<const double2*>(tab + e * 4 + 2);
        const double c0 = e0 * f01.x, c1 = e1 * f01.y, c2 = e2 * f2w.x;
        double r2 = __dmul_rn(c0, c0);
        r2 = __dadd_rn(r2, __dmul_rn(c1, c1));
        r2 = __dadd_rn(r2, __dmul_rn(c2, c2));
        acc = fma(kernel_shape<KIND>(r2, nid), vol * f2w.y, acc);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) out[pt] = coef * acc;
  }
}

template <int KIND>
static void mapped_diag_k(const KernelParams& kp, int d, int n, int q, const double* gx, const double* gw,
                          const double* bounds, const double* coords, double* out, int64_t npts, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((npts + 7) / 8, 148 * 16);
  if (q == 10 && d == 3) {
    const size_t smem = sizeof(double) * 4 * 3 * 1000;
    cudaFuncSetAttribute(mapped_diag3_kernel<KIND, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mapped_diag3_kernel<KIND, 10><<<std::min(grid, 148 * 2), 256, smem, st>>>(kp, n, gx, gw, bounds, coords, out,
                                                                             npts);
  } else if (q == 10)
    mapped_diag_kernel<KIND, 10><<<grid, 256, 0, st>>>(kp, d, n, q, gx, gw, bounds, coords, out, npts);
  else
    mapped_diag_kernel<KIND, 0><<<grid, 256, 0, st>>>(kp, d, n, q, gx, gw, bounds, coords, out, npts);
}

void launch_mapped_diag(const KernelParams& kp, int d, int n, int q, const double* gx, const double* gw,
                        const double* bounds, const double* coords, double* out, int64_t npts, cudaStream_t st) {
  if (kp.kind == 0)
    mapped_diag_k<0>(kp, d, n, q, gx, gw, bounds, coords, out, npts, st);
  else if (kp.kind == 1)
    mapped_diag_k<1>(kp, d, n, q, gx, gw, bounds, coords, out, npts, st);
  else
    mapped_diag_k<2>(kp, d, n, q, gx, gw, bounds, coords, out, npts, st);
}

static int regen_threads(int P) { return ((P + 31) / 32) * 32; }

template <int RB, int PP, int KIND>
static void adm_k(const KernelParams& kp, int d, int p, int level, const double* nodes, const int64_t* rowptr,
                  const int* cols, int64_t t0, int64_t nt, const double* W, int K_pad, double* H, int R, int r0,
                  cudaStream_t st) {
  const int P = (d == 2) ? p * p : p * p * p;
  const int thr = regen_threads(P);
  const size_t SB = RB >= 16 ? 1 : 4;
  size_t smem = sizeof(double) * (SB * RB * P + SB * 3 * kMaxRank + (size_t)thr * 2 * p);
  cudaFuncSetAttribute(regen_adm_kernel<RB, PP, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  regen_adm_kernel<RB, PP, KIND><<<(unsigned)nt, thr, smem, st>>>(kp, d, p, level, nodes, rowptr, cols, t0, W, K_pad,
                                                                 H, R, r0);
}

template <int RB, int PP>
static void adm_t(const KernelParams& kp, int d, int p, int level, const double* nodes, const int64_t* rowptr,
                  const int* cols, int64_t t0, int64_t nt, const double* W, int K_pad, double* H, int R, int r0,
                  cudaStream_t st) {
  if (kp.kind == 0)
    adm_k<RB, PP, 0>(kp, d, p, level, nodes, rowptr, cols, t0, nt, W, K_pad, H, R, r0, st);
  else if (kp.kind == 1)
    adm_k<RB, PP, 1>(kp, d, p, level, nodes, rowptr, cols, t0, nt, W, K_pad, H, R, r0, st);
  else
    adm_k<RB, PP, 2>(kp, d, p, level, nodes, rowptr, cols, t0, nt, W, K_pad, H, R, r0, st);
}

template <int RB>
static void adm_p(const KernelParams& kp, int d, int p, int level, const double* nodes, const int64_t* rowptr,
                  const int* cols, int64_t t0, int64_t nt, const double* W, int K_pad, double* H, int R, int r0,
                  cudaStream_t st) {
  switch (p) {
    case 4: adm_t<RB, 4>(kp, d, p, level, nodes, rowptr, cols, t0, nt, W, K_pad, H, R, r0, st); break;
    case 6: adm_t<RB, 6>(kp, d, p, level, nodes, rowptr, cols, t0, nt, W, K_pad, H, R, r0, st); break;
    case 8: adm_t<RB, 8>(kp, d, p, level, nodes, rowptr, cols, t0, nt, W, K_pad, H, R, r0, st); break;
    default: adm_t<RB, 0>(kp, d, p, level, nodes, rowptr, cols, t0, nt, W, K_pad, H, R, r0, st); break;
  }
}

void launch_regen_adm(const KernelParams& kp, int d, int p, int level, const double* nodes, const int64_t* rowptr,
                      const int* cols, int64_t t0, int64_t nt, const double* W, int K_pad, double* H, int R,
                      cudaStream_t st) {
  if (nt <= 0) return;
  for (int r0 = 0; r0 < R;) {
    const int left = R - r0;
    if (left >= 16) {
      adm_p<16>(kp, d, p, level, nodes, rowptr, cols, t0, nt, W, K_pad, H, R, r0, st);
      r0 += 16;
    } else if (left >= 4) {
      adm_p<4>(kp, d, p, level, nodes, rowptr, cols, t0, nt, W, K_pad, H, R, r0, st);
      r0 += 4;
    } else {
      adm_p<1>(kp, d, p, level, nodes, rowptr, cols, t0, nt, W, K_pad, H, R, r0, st);
      r0 += 1;
    }
  }
}

template <int RB, int SS, int KIND>
static void near_k(const KernelParams& kp, int d, int sL, int L, const double* coords, const double* widths,
                   const int64_t* rowptr, const int* cols, int64_t t0, int64_t nt, const double* ub, int K_pad,
                   double* Y, int R, int r0, cudaStream_t st) {
  const int P = (d == 2) ? sL * sL : sL * sL * sL;
  const int thr = regen_threads(P);
  const size_t SB = RB >= 16 ? 1 : 4;
  size_t smem = sizeof(double) * (SB * RB * P + SB * 3 * 16 + (size_t)thr * 2 * sL);
  cudaFuncSetAttribute(regen_near_kernel<RB, SS, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  regen_near_kernel<RB, SS, KIND><<<(unsigned)nt, thr, smem, st>>>(kp, d, sL, L, coords, widths, rowptr, cols, t0,
                                                                  ub, K_pad, Y, R, r0);
}

template <int RB, int SS>
static void near_t(const KernelParams& kp, int d, int sL, int L, const double* coords, const double* widths,
                   const int64_t* rowptr, const int* cols, int64_t t0, int64_t nt, const double* ub, int K_pad,
                   double* Y, int R, int r0, cudaStream_t st) {
  if (kp.kind == 0)
    near_k<RB, SS, 0>(kp, d, sL, L, coords, widths, rowptr, cols, t0, nt, ub, K_pad, Y, R, r0, st);
  else if (kp.kind == 1)
    near_k<RB, SS, 1>(kp, d, sL, L, coords, widths, rowptr, cols, t0, nt, ub, K_pad, Y, R, r0, st);
  else
    near_k<RB, SS, 2>(kp, d, sL, L, coords, widths, rowptr, cols, t0, nt, ub, K_pad, Y, R, r0, st);
}

template <int RB>
static void near_s(const KernelParams& kp, int d, int sL, int L, const double* coords, const double* widths,
                   const int64_t* rowptr, const int* cols, int64_t t0, int64_t nt, const double* ub, int K_pad,
                   double* Y, int R, int r0, cudaStream_t st) {
  switch (sL) {
    case 4: near_t<RB, 4>(kp, d, sL, L, coords, widths, rowptr, cols, t0, nt, ub, K_pad, Y, R, r0, st); break;
    case 6: near_t<RB, 6>(kp, d, sL, L, coords, widths, rowptr, cols, t0, nt, ub, K_pad, Y, R, r0, st); break;
    case 8: near_t<RB, 8>(kp, d, sL, L, coords, widths, rowptr, cols, t0, nt, ub, K_pad, Y, R, r0, st); break;
    default: near_t<RB, 0>(kp, d, sL, L, coords, widths, rowptr, cols, t0, nt, ub, K_pad, Y, R, r0, st); break;
  }
}

void launch_regen_near(const KernelParams& kp, int d, int sL, int L, const double* coords, const double* widths,
                       const int64_t* rowptr, const int* cols, int64_t t0, int64_t nt, const double* ub, int K_pad,
                       double* Y, int R, cudaStream_t st) {
  if (nt <= 0) return;
  for (int r0 = 0; r0 < R;) {
    const int left = R - r0;
    if (left >= 16) {
      near_s<16>(kp, d, sL, L, coords, widths, rowptr, cols, t0, nt, ub, K_pad, Y, R, r0, st);
      r0 += 16;
    } else if (left >= 4) {
      near_s<4>(kp, d, sL, L, coords, widths, rowptr, cols, t0, nt, ub, K_pad, Y, R, r0, st);
      r0 += 4;
    } else {
      near_s<1>(kp, d, sL, L, coords, widths, rowptr, cols, t0, nt, ub, K_pad, Y, R, r0, st);
      r0 += 1;
    }
  }
}

void launch_mapped_core_export(const KernelParams& kp, int d, int p, const double* nt, const double* ns, double* out,
                               cudaStream_t st) {
  mapped_core_export_kernel<<<256, 256, 0, st>>>(kp, d, p, nt, ns, out);
}

void launch_mapped_near_export(const KernelParams& kp, int d, int sL, const double* xt, const double* ys,
                               const double* ws, int self, double* out, cudaStream_t st) {
  mapped_near_export_kernel<<<256, 256, 0, st>>>(kp, d, sL, xt, ys, ws, self, out);
}

}  // namespace htlr
