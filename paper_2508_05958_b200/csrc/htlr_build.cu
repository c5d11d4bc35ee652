// Construction kernels of the B200 HTLR plan (sm_100a).
//
//   diag_kernel        diagonal cell average      kernels.py:195-265
//   factor_qr_kernel   Lagrange factor + thin Householder QR per level
//                                                  chebyshev.py:31-66, tensor.py:107-115,
//                                                  blocks.py:146-162
//   core_sample_kernel Chebyshev kernel sampling, h^d fold
//                                                  chebyshev.py:69-85, blocks.py:163
//   core_mode_kernel   one mode product of the R (or raw square) factor
//                                                  blocks.py:146-163, tensor.py:35-52
//   core_tile_kernel   store the core pre-tiled for the m16n8k8 GEMM
//   near_block_kernel  unique inadmissible blocks a_i 1[i=j] + K_ij h^d
//                                                  blocks.py:190-227, kernels.py:120-149
//
// On a uniform grid every admissible block's factors depend only on the box
// side and its core only on (level, offset) (translation-invariant kernels),
// so the plan builds one factor pair per level and one core per unique
// (level, offset) from a representative leaf of the reference's list.
#include "htlr_device.cuh"
#include "htlr_kernels.h"

namespace htlr {

// ---------------------------------------------------------------------------
// diagonal cell average
// ---------------------------------------------------------------------------
__global__ void diag_kernel(KernelParams kp, int d, double h, int q, const double* __restrict__ gx,
                            const double* __restrict__ gw, int singular, double* __restrict__ out) {
  __shared__ double red[256];
  double acc = 0.0;
  const int qd = (d == 2) ? q * q : q * q * q;
  if (!singular) {
    // kernels.py:210-219: tensor GL rule over [-h/2, h/2]^d, weights h*gw
    for (int idx = threadIdx.x; idx < qd; idx += blockDim.x) {
      int i0 = idx % q, i1 = (idx / q) % q, i2 = idx / (q * q);
      int ii[3] = {i0, i1, i2};
      double pt[3] = {0, 0, 0}, zero[3] = {0, 0, 0};
      double w = 1.0;
      for (int a = 0; a < d; ++a) {
        pt[a] = __dadd_rn(-h / 2, __dmul_rn(h, gx[ii[a]]));
        w = w * __dmul_rn(h, gw[ii[a]]);
      }
      acc += kernel_from_r2(kp, r2_of(d, zero, pt)) * w;
    }
  } else {
    // kernels.py:222-249: 2^d corner sub-cells x d Duffy pyramids, radial
    // coordinate t^3 along `axis`, Jacobian s^d t^(d-1)
    const double s = h / 2.0;
    const double sd = (d == 2) ? s * s : s * s * s;
    const int ncorner = 1 << d;
    const int total = ncorner * d * qd;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      int pidx = idx % qd;
      int axis = (idx / qd) % d;
      int corner = idx / (qd * d);
      int ii[3] = {pidx % q, (pidx / q) % q, pidx / (q * q)};
      double tt = gx[ii[axis]];
      double t = tt * tt * tt;
      double w = 1.0;
      double pt[3] = {0, 0, 0}, zero[3] = {0, 0, 0};
      for (int a = 0; a < d; ++a) {
        double sign = ((corner >> (d - 1 - a)) & 1) ? 1.0 : -1.0;
        double z = (a == axis) ? s * t : s * t * gx[ii[a]];
        pt[a] = sign * z;
        double wa = (a == axis) ? 3.0 * (tt * tt) * gw[ii[a]] : gw[ii[a]];
        w = w * wa;
      }
      double jac = sd * ((d == 2) ? t : t * t);
      acc += kernel_from_r2(kp, r2_of(d, zero, pt)) * (jac * w);
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double hd = (d == 2) ? h * h : h * h * h;
    out[0] = red[0] / hd;
  }
}

// ---------------------------------------------------------------------------
// Per-level Lagrange factor of the representative box [0, s) and its thin
// Householder QR with LAPACK's dlarfg sign convention (dgeqr2 + dorg2r), so
// Q matches numpy.linalg.qr column signs.  s == p: R := raw factor, Q := I
// (blocks.py:155-158).  One thread per level (s x p is at most 64 x 16).
// ---------------------------------------------------------------------------
__global__ void factor_qr_kernel(int nlev, const FactorJob* __restrict__ jobs, double h, int p) {
  int li = blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= nlev) return;
  FactorJob jb = jobs[li];
  const int s = jb.side;
  double* A = jb.work;   // s x p scratch, column-major (A[i + s*j])
  double lo = 0.0, hi = (double)s * h;
  double nodes[kMaxRank];
  for (int t = 0; t < p; ++t) nodes[t] = cheb_node(lo, hi, t + 1, p);
  // chebyshev.py:58-65: product over j != t in ascending j
  for (int i = 0; i < s; ++i) {
    double x = __dmul_rn(__dadd_rn((double)i, 0.5), h);
    for (int t = 0; t < p; ++t) {
      double prod = 1.0;
      bool first = true;
      for (int j = 0; j < p; ++j) {
        if (j == t) continue;
        double fct = __ddiv_rn(__dadd_rn(x, -nodes[j]), __dadd_rn(nodes[t], -nodes[j]));
        prod = first ? fct : __dmul_rn(prod, fct);
        first = false;
      }
      A[i + s * t] = prod;
    }
  }
  if (s == p) {
    for (int i = 0; i < p; ++i)
      for (int j = 0; j < p; ++j) {
        jb.R[i * p + j] = A[i + s * j];
        jb.Q[i * p + j] = (i == j) ? 1.0 : 0.0;
      }
    return;
  }
  double tau[kMaxRank];
  // dgeqr2
  for (int i = 0; i < p; ++i) {
    double alpha = A[i + s * i];
    double xnorm2 = 0.0;
    for (int k = i + 1; k < s; ++k) xnorm2 += A[k + s * i] * A[k + s * i];
    double xnorm = sqrt(xnorm2);
    if (xnorm == 0.0) {
      tau[i] = 0.0;
    } else {
      double beta = -copysign(sqrt(alpha * alpha + xnorm * xnorm), alpha);
      tau[i] = (beta - alpha) / beta;
      double scal = 1.0 / (alpha - beta);
      for (int k = i + 1; k < s; ++k) A[k + s * i] *= scal;
      A[i + s * i] = beta;
    }
    // apply H_i = I - tau v v^T (v = [1; A[i+1:, i]]) to A[i:, i+1:]
    for (int j = i + 1; j < p; ++j) {
      double w = A[i + s * j];
      for (int k = i + 1; k < s; ++k) w += A[k + s * i] * A[k + s * j];
      w *= tau[i];
      A[i + s * j] -= w;
      for (int k = i + 1; k < s; ++k) A[k + s * j] -= w * A[k + s * i];
    }
  }
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) jb.R[i * p + j] = (j >= i) ? A[i + s * j] : 0.0;
  // dorg2r: Q (s x p) from the reflectors, last to first
  double* Qc = jb.work2;   // s x p column-major
  for (int j = 0; j < p; ++j)
    for (int k = 0; k < s; ++k) Qc[k + s * j] = (k == j) ? 1.0 : 0.0;
  for (int i = p - 1; i >= 0; --i) {
    for (int j = i; j < p; ++j) {
      double w = Qc[i + s * j];
      for (int k = i + 1; k < s; ++k) w += A[k + s * i] * Qc[k + s * j];
      w *= tau[i];
      Qc[i + s * j] -= w;
      for (int k = i + 1; k < s; ++k) Qc[k + s * j] -= w * A[k + s * i];
    }
  }
  for (int k = 0; k < s; ++k)
    for (int j = 0; j < p; ++j) jb.Q[k * p + j] = Qc[k + s * j];
}

// ---------------------------------------------------------------------------
// Kernel sampling on tensor Chebyshev grids: core[t + P*s] = h^d k(xi_t, eta_s),
// target multi-index t (F-order) first, source s last (chebyshev.py:79-85).
// grid: (entry chunks, cores in batch)
// ---------------------------------------------------------------------------
__global__ void core_sample_kernel(const CoreJob* __restrict__ jobs, int d, int p, double h, double hd,
                                   KernelParams kp, double* __restrict__ out) {
  const CoreJob jb = jobs[blockIdx.y];
  __shared__ double nt[3][kMaxRank], ns[3][kMaxRank];
  if (threadIdx.x < d * p) {
    int a = threadIdx.x / p, t = threadIdx.x % p;
    double tlo = (double)jb.tlo[a] * h, thi = (double)(jb.tlo[a] + jb.side) * h;
    double slo = (double)jb.slo[a] * h, shi = (double)(jb.slo[a] + jb.side) * h;
    nt[a][t] = cheb_node(tlo, thi, t + 1, p);
    ns[a][t] = cheb_node(slo, shi, t + 1, p);
  }
  __syncthreads();
  const int P = (d == 2) ? p * p : p * p * p;
  const int64_t PP = (int64_t)P * P;
  double* dst = out + (int64_t)blockIdx.y * PP;
  for (int64_t lin = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lin < PP;
       lin += (int64_t)gridDim.x * blockDim.x) {
    int ti = (int)(lin % P), si = (int)(lin / P);
    double x[3], y[3];
    for (int a = 0; a < d; ++a) {
      x[a] = nt[a][ti % p];
      y[a] = ns[a][si % p];
      ti /= p;
      si /= p;
    }
    dst[lin] = hd * kernel_from_r2(kp, r2_of(d, x, y));
  }
}

// One mode product out = in x_mode M (tensor.py:35-52) over a batch of cores;
// M is the core's level factor (R, or the raw factor for square levels).
// mode is 0-based over the 2d modes; stride = p^mode.
__global__ void core_mode_kernel(const CoreJob* __restrict__ jobs, int p, int64_t PP, int64_t stride,
                                 const double* __restrict__ in, double* __restrict__ out) {
  const CoreJob jb = jobs[blockIdx.y];
  const double* M = jb.R;
  const double* src = in + (int64_t)blockIdx.y * PP;
  double* dst = out + (int64_t)blockIdx.y * PP;
  for (int64_t lin = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lin < PP;
       lin += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)((lin / stride) % p);
    int64_t base = lin - (int64_t)i * stride;
    double acc = 0.0;
    for (int j = 0; j < p; ++j) acc += M[i * p + j] * src[base + (int64_t)j * stride];
    dst[lin] = acc;
  }
}

// Store a finished core (P x P, element (m, k) at m + P*k) pre-tiled into the
// level's GEMM table, zero padding rows to M_pad and columns to K_pad.
__global__ void core_tile_kernel(const CoreJob* __restrict__ jobs, int P, const double* __restrict__ in,
                                 int MT, int M_pad, int K_pad) {
  const CoreJob jb = jobs[blockIdx.y];
  const double* src = in + (int64_t)blockIdx.y * P * P;
  const int64_t tot = (int64_t)M_pad * K_pad;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    int m = (int)(e % M_pad), k = (int)(e / M_pad);
    double v = (m < P && k < P) ? src[m + (int64_t)P * k] : 0.0;
    jb.dst[tiled_offset(m, k, MT, K_pad)] = v;
  }
}

// ---------------------------------------------------------------------------
// Unique inadmissible blocks (one per leaf-level offset): K_ij h^d with the
// tau == sigma diagonal replaced by the cell average (blocks.py:213-226,
// kernels.py:139-149); a(x_i) is added in the matvec epilogue.
// ---------------------------------------------------------------------------
__global__ void near_block_kernel(const NearJob* __restrict__ jobs, int d, int s, double h, double hd,
                                  KernelParams kp, const double* __restrict__ diag, int MT, int M_pad,
                                  int K_pad) {
  const NearJob jb = jobs[blockIdx.y];
  const int P = (d == 2) ? s * s : s * s * s;
  const int64_t tot = (int64_t)M_pad * K_pad;
  const double dval = diag[0];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    int m = (int)(e % M_pad), k = (int)(e / M_pad);
    double v = 0.0;
    if (m < P && k < P) {
      if (jb.self && m == k) {
        v = dval * hd;
      } else {
        double x[3], y[3];
        int mi = m, ki = k;
        for (int a = 0; a < d; ++a) {
          x[a] = __dmul_rn(__dadd_rn((double)(jb.tlo[a] + mi % s), 0.5), h);
          y[a] = __dmul_rn(__dadd_rn((double)(jb.slo[a] + ki % s), 0.5), h);
          mi /= s;
          ki /= s;
        }
        v = kernel_from_r2(kp, r2_of(d, x, y)) * hd;
      }
    }
    jb.dst[tiled_offset(m, k, MT, K_pad)] = v;
  }
}

// ---------------------------------------------------------------------------
// Toeplitz generators of the near blocks (3-D, leaf side 8, dyadic h): block
// delta has A[i][j] = G[(j - i) + 7 per axis], exactly (the coordinates
// (c + 1/2) h are exact, so r^2 only depends on the index difference).  G is
// read back from the tiled block itself, so the generated operand equals the
// stored one bit for bit.
// ---------------------------------------------------------------------------
__global__ void near_gen_kernel(const double* __restrict__ table, int64_t mat_stride, int nmats, int MT, int K_pad,
                                double* __restrict__ gen) {
  const int total = kGenSide * kGenSide * kGenSide;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)nmats * total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(e / total), u = (int)(e % total);
    const int uu[3] = {u % kGenSide, (u / kGenSide) % kGenSide, u / (kGenSide * kGenSide)};
    int row = 0, col = 0, mul = 1;
    for (int a = 0; a < 3; ++a) {
      const int i = uu[a] <= 7 ? 7 - uu[a] : 0, j = uu[a] <= 7 ? 0 : uu[a] - 7;
      row += i * mul;
      col += j * mul;
      mul *= 8;
    }
    gen[(int64_t)m * kGenStride + u] = table[(int64_t)m * mat_stride + tiled_offset(row, col, MT, K_pad)];
  }
}

void launch_near_gen(const double* table, int64_t mat_stride, int nmats, int MT, int K_pad, double* gen,
                     cudaStream_t st) {
  if (nmats <= 0) return;
  near_gen_kernel<<<148 * 4, 256, 0, st>>>(table, mat_stride, nmats, MT, K_pad, gen);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
void launch_diag(const KernelParams& kp, int d, double h, int q, const double* gx, const double* gw,
                 int singular, double* out, cudaStream_t st) {
  diag_kernel<<<1, 256, 0, st>>>(kp, d, h, q, gx, gw, singular, out);
}

void launch_factor_qr(int nlev, const FactorJob* jobs, double h, int p, cudaStream_t st) {
  factor_qr_kernel<<<1, 32, 0, st>>>(nlev, jobs, h, p);
}

void launch_core_batch(const CoreJob* jobs, int nbatch, int d, int p, double h, double hd,
                       const KernelParams& kp, double* buf0, double* buf1, int MT, int M_pad, int K_pad,
                       cudaStream_t st) {
  const int P = (d == 2) ? p * p : p * p * p;
  const int64_t PP = (int64_t)P * P;
  int chunks = (int)((PP + 255) / 256);
  if (chunks > 1024) chunks = 1024;
  dim3 grid(chunks, nbatch);
  core_sample_kernel<<<grid, 256, 0, st>>>(jobs, d, p, h, hd, kp, buf0);
  // blocks.py:146-163 order: (u_1, mode 1), (v_1, mode d+1), (u_2, 2), (v_2, d+2), ...
  double* in = buf0;
  double* out = buf1;
  for (int a = 0; a < d; ++a) {
    for (int side = 0; side < 2; ++side) {
      int mode = side == 0 ? a : d + a;
      int64_t stride = 1;
      for (int j = 0; j < mode; ++j) stride *= p;
      core_mode_kernel<<<grid, 256, 0, st>>>(jobs, p, PP, stride, in, out);
      double* tmp = in;
      in = out;
      out = tmp;
    }
  }
  int64_t tot = (int64_t)M_pad * K_pad;
  int tchunks = (int)((tot + 255) / 256);
  if (tchunks > 1024) tchunks = 1024;
  core_tile_kernel<<<dim3(tchunks, nbatch), 256, 0, st>>>(jobs, P, in, MT, M_pad, K_pad);
}

void launch_near_blocks(const NearJob* jobs, int njobs, int d, int s, double h, double hd,
                        const KernelParams& kp, const double* diag, int MT, int M_pad, int K_pad,
                        cudaStream_t st) {
  int64_t tot = (int64_t)M_pad * K_pad;
  int chunks = (int)((tot + 255) / 256);
  if (chunks > 1024) chunks = 1024;
  near_block_kernel<<<dim3(chunks, njobs), 256, 0, st>>>(jobs, d, s, h, hd, kp, diag, MT, M_pad, K_pad);
}

}  // namespace htlr
