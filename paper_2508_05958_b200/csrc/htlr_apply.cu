// Matvec kernels of the B200 HTLR plan (sm_100a).
//
// The reference applies every leaf independently (operators.py:138-161,
// blocks.py:230-259): W = V^T-mode products of u_sigma, H = core . W,
// f_tau += U-mode products of H.  Factors depend only on a box, so the same
// algebra is regrouped exactly into
//   permute_in   u (F-order) -> leaf-box-major ub         (operators.py:144-148)
//   upward       W_l[c] = (V^T x V^T x V^T) u_c per cluster (blocks.py:239-247)
//   gemm         H_l[t] += G_l[o(t,s)] W_l[s] over the admissible list, and
//                Y[t]   += D[o(t,s)] ub[s] over the near list, as batched
//                fp64 tensor-core GEMMs (mma.sync m16n8k8 -> DMMA) with
//                gathered B columns                  (blocks.py:248-250, operators.py:150)
//   downward     f = Y + a u + sum_l (U x U x U) H_l[anc] per leaf box, written
//                back in F-order                     (blocks.py:251-259, operators.py:153-156)
#include <algorithm>
#include <cstdlib>

#include "htlr_kernels.h"

namespace htlr {

// Physical -> logical index of a box vector stored with a z-plane pitch
// (zpitch == 0: natural layout).  Pitched layout (separable passes): plane z
// of `plane` doubles starts at z * zpitch, so one bulk copy of the box lands
// in shared memory with bank-conflict-free mode-z fragments.  Returns a value
// >= nplanes * plane for padding positions.
__device__ __forceinline__ int unpitch(int kp, int plane, int nplanes, int zpitch) {
  if (!zpitch) return kp;
  const int pl = kp / zpitch, off = kp - pl * zpitch;
  return (off < plane && pl < nplanes) ? pl * plane + off : nplanes * plane;
}

// ---------------------------------------------------------------------------
// permute: ub[(b*R + r)*K_pad + k] = u[(global point of (b, k))*R + r]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void permute_body(const double* __restrict__ u, double* __restrict__ ub, int d, int n,
                                             int s, int bits, int R, int K_pad, int64_t b0, int64_t nb,
                                             const ZeroList& zero, int64_t blk, int64_t nblk, int zpitch = 0,
                                             int zlo = 0, int zhi = 0) {
  if (blk >= nb) {
    // the extra CTAs zero the accumulators of the coming GEMM passes
    const int64_t stride = (nblk - nb) * blockDim.x;
    const int64_t first = (blk - nb) * blockDim.x + threadIdx.x;
    for (int q = 0; q < zero.cnt; ++q) {
      double* z = zero.p[q];
      for (int64_t e = first; e < zero.n[q]; e += stride) z[e] = 0.0;
    }
    return;
  }
  const int64_t b = b0 + blk;   // leaf box, Morton id
  int bc[3];
  morton_decode(b, d, bits, bc);
  if (zhi > 0 && (bc[2] < zlo || bc[2] >= zhi)) return;
  const int P = (d == 2) ? s * s : s * s * s;
  for (int idx = threadIdx.x; idx < R * K_pad; idx += blockDim.x) {
    int r = idx % R, kp = idx / R;
    const int k = (d == 3) ? unpitch(kp, s * s, s, zpitch) : kp;
    double v = 0.0;
    if (k < P) {
      int x = k % s, y = (k / s) % s, z = k / (s * s);
      int64_t g = (int64_t)(bc[0] * s + x) + (int64_t)n * (bc[1] * s + y);
      if (d == 3) g += (int64_t)n * n * (bc[2] * s + z);
      v = u[g * R + r];
    }
    ub[((int64_t)b * R + r) * K_pad + kp] = v;
  }
}

__global__ void permute_in_kernel(const double* __restrict__ u, double* __restrict__ ub, int d, int n,
                                  int s, int bits, int R, int K_pad, int64_t b0, int64_t nb, ZeroList zero,
                                  int zpitch) {
  permute_body(u, ub, d, n, s, bits, R, K_pad, b0, nb, zero, blockIdx.x, gridDim.x, zpitch);
}

void launch_permute_in(const double* u, double* ub, int d, int n, int s, int R, int K_pad, int64_t b0,
                       int64_t nb, cudaStream_t st, const ZeroList* zero, int zpitch) {
  int bits = 0;
  while ((s << bits) < n) ++bits;
  ZeroList z;
  int64_t words = 0;
  if (zero) {
    z = *zero;
    for (int q = 0; q < z.cnt; ++q) words += z.n[q];
  }
  const int64_t zblocks = std::min<int64_t>((words + 2047) / 2048, 4 * 148);
  if (nb > 0 || zblocks > 0)
    permute_in_kernel<<<(unsigned)(nb + zblocks), 256, 0, st>>>(u, ub, d, n, s, bits, R, K_pad, b0, nb, z, zpitch);
}

// ---------------------------------------------------------------------------
// upward pass: one CTA per (cluster, rhs); the three mode products run as
// three whole-box phases (every global load of the box is issued in phase 1,
// so the CTA pays one memory latency, not one per slab):
//   T1[a1, y, z] = sum_x Qx[x][a1] u[x, y, z]
//   T2[a1, a2, z] = sum_y Qy[y][a2] T1[a1, y, z]
//   W[a1, a2, a3] = sum_z Qz[z][a3] T2[a1, a2, z]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void upward_body(const double* __restrict__ u, double* __restrict__ W, int d, int n,
                                            int s, int p, int bits, int R, int K_pad, const double* __restrict__ Q,
                                            int64_t qstride, int64_t c, int r, double* sm, int zpitch = 0) {
  double* sQ = sm;                          // d x s*p (factor of each dimension)
  double* T1 = sQ + d * s * p;              // p*s*s (3-D) / p*s (2-D)
  double* T2 = T1 + p * s * (d == 3 ? s : 1);   // p*p*s (3-D)
  int cc[3];
  morton_decode(c, d, bits, cc);
  for (int i = threadIdx.x; i < d * s * p; i += blockDim.x) {
    const int a = i / (s * p);
    sQ[i] = Q[(qstride ? cc[a] * qstride : 0) + i % (s * p)];
  }
  const double* sQx = sQ;
  const double* sQy = sQ + s * p;
  const double* sQz = sQ + 2 * s * p;
  const int P = (d == 2) ? p * p : p * p * p;
  const int nz = (d == 3) ? s : 1;
  __syncthreads();
  for (int i = threadIdx.x; i < p * s * nz; i += blockDim.x) {
    const int a1 = i % p, y = (i / p) % s, z = i / (p * s);
    int64_t g = (int64_t)cc[0] * s + (int64_t)n * (cc[1] * s + y);
    if (d == 3) g += (int64_t)n * n * (cc[2] * s + z);
    double v = 0.0;
    for (int x = 0; x < s; ++x) v += sQx[x * p + a1] * u[(g + x) * R + r];
    T1[i] = v;
  }
  __syncthreads();
  double* dst = W + ((int64_t)c * R + r) * K_pad;
  if (d == 2) {
    for (int i = threadIdx.x; i < K_pad; i += blockDim.x) {
      double v = 0.0;
      if (i < P) {
        const int a1 = i % p, a2 = i / p;
        for (int y = 0; y < s; ++y) v += sQy[y * p + a2] * T1[a1 + p * y];
      }
      dst[i] = v;
    }
    return;
  }
  for (int i = threadIdx.x; i < p * p * s; i += blockDim.x) {
    const int a1 = i % p, a2 = (i / p) % p, z = i / (p * p);
    const double* t1 = T1 + a1 + p * s * z;
    double v = 0.0;
    for (int y = 0; y < s; ++y) v += sQy[y * p + a2] * t1[p * y];
    T2[i] = v;
  }
  __syncthreads();
  for (int ip = threadIdx.x; ip < K_pad; ip += blockDim.x) {
    const int i = unpitch(ip, p * p, p, zpitch);
    double v = 0.0;
    if (i < P) {
      const int a12 = i % (p * p), a3 = i / (p * p);
      for (int z = 0; z < s; ++z) v += sQz[z * p + a3] * T2[a12 + p * p * z];
    }
    dst[ip] = v;
  }
}

// Split variant for levels with few clusters (3-D): CTA (cluster, rhs, slab)
// runs the three mode products on its side / nslab z-planes only, writes the
// partial W (the mode-3 sum over its planes), and the last of the nslab CTAs
// of the cluster (arrival counter, gpu-scope fences) sums the partials into W
// and resets the counter.
__device__ __forceinline__ void upward_split_body(const double* __restrict__ u, double* __restrict__ W, int n, int s,
                                                  int p, int bits, int R, int K_pad, const double* __restrict__ Q,
                                                  int64_t qstride, int64_t c, int64_t c0, int r, int slab, int nslab,
                                                  double* __restrict__ scratch, int* __restrict__ counters,
                                                  double* sm, int zpitch = 0) {
  const int zs = s / nslab, z0 = slab * zs;
  double* sQ = sm;                 // 3 x s*p
  double* T1 = sQ + 3 * s * p;     // p*s*zs
  double* T2 = T1 + p * s * zs;    // p*p*zs
  __shared__ int last;
  int cc[3];
  morton_decode(c, 3, bits, cc);
  for (int i = threadIdx.x; i < 3 * s * p; i += blockDim.x) {
    const int a = i / (s * p);
    sQ[i] = Q[(qstride ? cc[a] * qstride : 0) + i % (s * p)];
  }
  const double* sQx = sQ;
  const double* sQy = sQ + s * p;
  const double* sQz = sQ + 2 * s * p;
  const int P = p * p * p;
  __syncthreads();
  for (int i = threadIdx.x; i < p * s * zs; i += blockDim.x) {
    const int a1 = i % p, y = (i / p) % s, z = z0 + i / (p * s);
    const int64_t g = (int64_t)cc[0] * s + (int64_t)n * (cc[1] * s + y) + (int64_t)n * n * (cc[2] * s + z);
    double v = 0.0;
    for (int x = 0; x < s; ++x) v += sQx[x * p + a1] * u[(g + x) * R + r];
    T1[i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < p * p * zs; i += blockDim.x) {
    const int a1 = i % p, a2 = (i / p) % p, z = i / (p * p);
    const double* t1 = T1 + a1 + p * s * z;
    double v = 0.0;
    for (int y = 0; y < s; ++y) v += sQy[y * p + a2] * t1[p * y];
    T2[i] = v;
  }
  __syncthreads();
  const int64_t cr = (c - c0) * R + r;
  double* part = scratch + (cr * nslab + slab) * P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    const int a12 = i % (p * p), a3 = i / (p * p);
    double v = 0.0;
    for (int z = 0; z < zs; ++z) v += sQz[(z0 + z) * p + a3] * T2[a12 + p * p * z];
    part[i] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counters + cr, 1) == nslab - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double* p0 = scratch + cr * nslab * P;
  double* dst = W + ((int64_t)c * R + r) * K_pad;
  for (int ip = threadIdx.x; ip < K_pad; ip += blockDim.x) {
    const int i = unpitch(ip, p * p, p, zpitch);
    double v = 0.0;
    if (i < P)
      for (int q = 0; q < nslab; ++q) v += __ldcg(p0 + q * P + i);
    dst[ip] = v;
  }
  if (threadIdx.x == 0) counters[cr] = 0;
}

size_t upward_split_smem_words(int side, int p, int nslab) {
  const int zs = side / nslab;
  return (size_t)3 * side * p + (size_t)p * side * zs + (size_t)p * p * zs;
}

int upward_nslab(int d, int side, int64_t nc, int R) {
  if (d != 3) return 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int ns = 1;
  while (nc * R * ns < 2 * sms && side % (2 * ns) == 0 && side / (2 * ns) >= 4) ns *= 2;
  return ns;
}

__global__ void upward_split_kernel(const double* __restrict__ u, double* __restrict__ W, int n, int s, int p,
                                    int bits, int R, int K_pad, const double* __restrict__ Q, int64_t qstride,
                                    int64_t c0, int nslab, double* __restrict__ scratch, int* __restrict__ counters,
                                    int zpitch) {
  extern __shared__ double sm[];
  upward_split_body(u, W, n, s, p, bits, R, K_pad, Q, qstride, c0 + blockIdx.x / nslab, c0, blockIdx.y,
                    (int)(blockIdx.x % nslab), nslab, scratch, counters, sm, zpitch);
}

__global__ void upward_kernel(const double* __restrict__ u, double* __restrict__ W, int d, int n, int s,
                              int p, int bits, int R, int K_pad, const double* __restrict__ Q, int64_t qstride,
                              int64_t c0, int zpitch) {
  extern __shared__ double sm[];
  upward_body(u, W, d, n, s, p, bits, R, K_pad, Q, qstride, c0 + blockIdx.x, blockIdx.y, sm, zpitch);
}

// ---------------------------------------------------------------------------
// prologue of an unsharded matvec in one launch: the permute CTAs, the CTAs
// zeroing the accumulators, and the upward CTAs of every compressed level
// (all three only read u), instead of 1 + levels launches and memset nodes
// ---------------------------------------------------------------------------
__global__ void prologue_kernel(PrologueParams pp) {
  extern __shared__ double sm[];
  const int64_t b = blockIdx.x;
  if (b < pp.nb_perm + pp.nb_zero) {
    permute_body(pp.u, pp.ub, pp.d, pp.n, pp.sL, pp.bits_L, pp.R, pp.K_pad_leaf, pp.b0, pp.nb_perm, pp.zero, b,
                 pp.nb_perm + pp.nb_zero, pp.zpitch_leaf, pp.zlo, pp.zhi);
    return;
  }
  int64_t rest = b - pp.nb_perm - pp.nb_zero;
  for (int li = 0; li < pp.nlev; ++li) {
    const UpLevel& lv = pp.lev[li];
    const int ns = lv.nslab > 1 ? lv.nslab : 1;
    const int64_t cnt = lv.nc * pp.R * ns;
    if (rest < cnt) {
      if (pp.zhi > 0) {   // cluster filter: its last leaf-box z index in [zlo, zhi)
        int cc[3];
        morton_decode(lv.c0 + rest / ((int64_t)pp.R * ns), 3, lv.bits, cc);
        const int span = 1 << (pp.bits_L - lv.bits);
        const int zl = cc[2] * span + span - 1;
        if (zl < pp.zlo || zl >= pp.zhi) return;
      }
      if (ns > 1) {
        const int64_t cr = rest / ns;
        upward_split_body(pp.u, lv.W, pp.n, lv.side, pp.p, lv.bits, pp.R, lv.K_pad, lv.Q, lv.qstride,
                          lv.c0 + cr / pp.R, lv.c0, (int)(cr % pp.R), (int)(rest % ns), ns, lv.scratch, lv.counters,
                          sm, lv.zpitch);
        return;
      }
      upward_body(pp.u, lv.W, pp.d, pp.n, lv.side, pp.p, lv.bits, pp.R, lv.K_pad, lv.Q, lv.qstride,
                  lv.c0 + rest / pp.R, (int)(rest % pp.R), sm, lv.zpitch);
      return;
    }
    rest -= cnt;
  }
}

// large boxes (whole-box phases above ~200 KB of shared memory): mode 1 and 2
// per z-slab, the mode-3 product accumulated slab by slab
__global__ void upward_slab_kernel(const double* __restrict__ u, double* __restrict__ W, int d, int n, int s,
                              int p, int bits, int R, int K_pad, const double* __restrict__ Q, int64_t qstride,
                              int64_t c0, int zpitch) {
  extern __shared__ double sm[];
  double* sQ = sm;             // d x s*p (factor of each dimension)
  double* T1 = sQ + d * s * p; // p*s
  double* T2 = T1 + p * s;     // p*p
  double* acc = T2 + p * p;    // p^d
  const int64_t c = c0 + blockIdx.x;   // cluster, Morton id
  const int r = blockIdx.y;
  int cc[3];
  morton_decode(c, d, bits, cc);
  for (int i = threadIdx.x; i < d * s * p; i += blockDim.x) {
    const int a = i / (s * p);
    sQ[i] = Q[(qstride ? cc[a] * qstride : 0) + i % (s * p)];
  }
  const double* sQx = sQ;
  const double* sQy = sQ + s * p;
  const double* sQz = sQ + 2 * s * p;
  const int P = (d == 2) ? p * p : p * p * p;
  for (int i = threadIdx.x; i < P; i += blockDim.x) acc[i] = 0.0;
  __syncthreads();
  const int nz = (d == 3) ? s : 1;
  for (int z = 0; z < nz; ++z) {
    // T1[a1 + p*y] = sum_x Q[x][a1] u[x, y, z]
    for (int i = threadIdx.x; i < p * s; i += blockDim.x) {
      int a1 = i % p, y = i / p;
      int64_t g = (int64_t)cc[0] * s + (int64_t)n * (cc[1] * s + y);
      if (d == 3) g += (int64_t)n * n * (cc[2] * s + z);
      double v = 0.0;
      for (int x = 0; x < s; ++x) v += sQx[x * p + a1] * u[(g + x) * R + r];
      T1[i] = v;
    }
    __syncthreads();
    if (d == 2) {
      for (int i = threadIdx.x; i < p * p; i += blockDim.x) {
        int a1 = i % p, a2 = i / p;
        double v = 0.0;
        for (int y = 0; y < s; ++y) v += sQy[y * p + a2] * T1[a1 + p * y];
        acc[i] = v;
      }
      __syncthreads();
    } else {
      for (int i = threadIdx.x; i < p * p; i += blockDim.x) {
        int a1 = i % p, a2 = i / p;
        double v = 0.0;
        for (int y = 0; y < s; ++y) v += sQy[y * p + a2] * T1[a1 + p * y];
        T2[i] = v;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        int a12 = i % (p * p), a3 = i / (p * p);
        acc[i] += sQz[z * p + a3] * T2[a12];
      }
      __syncthreads();
    }
  }
  double* dst = W + ((int64_t)c * R + r) * K_pad;
  for (int ip = threadIdx.x; ip < K_pad; ip += blockDim.x) {
    const int i = d == 3 ? unpitch(ip, p * p, p, zpitch) : ip;
    dst[ip] = i < P ? acc[i] : 0.0;
  }
}

size_t upward_smem_words(int d, int side, int p) {
  return (size_t)d * side * p + (size_t)p * side * (d == 3 ? side : 1) + (d == 3 ? (size_t)p * p * side : 0);
}

void launch_prologue(const PrologueParams& pp_in, cudaStream_t st) {
  PrologueParams pp = pp_in;
  int64_t words = 0;
  for (int q = 0; q < pp.zero.cnt; ++q) words += pp.zero.n[q];
  pp.nb_zero = std::min<int64_t>((words + 2047) / 2048, 4 * 148);
  int bits = 0;
  while ((pp.sL << bits) < pp.n) ++bits;
  pp.bits_L = bits;
  size_t smem_words = 0;
  int64_t blocks = pp.nb_perm + pp.nb_zero;
  for (int li = 0; li < pp.nlev; ++li) {
    const UpLevel& lv = pp.lev[li];
    const int ns = lv.nslab > 1 ? lv.nslab : 1;
    smem_words = std::max(smem_words, ns > 1 ? upward_split_smem_words(lv.side, pp.p, ns)
                                             : upward_smem_words(pp.d, lv.side, pp.p));
    blocks += lv.nc * pp.R * ns;
  }
  const size_t smem = smem_words * sizeof(double);
  if (smem > 48 * 1024) cudaFuncSetAttribute(prologue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (blocks > 0) prologue_kernel<<<(unsigned)blocks, 256, smem, st>>>(pp);
}

void launch_upward(const double* u, double* W, int d, int n, int side, int p, int level, int R,
                   int K_pad, const double* Q, int64_t qstride, int64_t c0, int64_t nc, cudaStream_t st,
                   int nslab, double* scratch, int* counters, int zpitch) {
  const size_t smem = sizeof(double) * upward_smem_words(d, side, p);
  if (nc <= 0) return;
  if (nslab > 1 && d == 3) {
    const size_t sm2 = sizeof(double) * upward_split_smem_words(side, p, nslab);
    if (sm2 > 48 * 1024)
      cudaFuncSetAttribute(upward_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    upward_split_kernel<<<dim3((unsigned)(nc * nslab), R), 256, sm2, st>>>(u, W, n, side, p, level, R, K_pad, Q,
                                                                          qstride, c0, nslab, scratch, counters,
                                                                          zpitch);
    return;
  }
  static int force_slab = -1;   // HTLR_UPWARD_SLAB=1: slab kernel for every box (tests)
  if (force_slab < 0) {
    const char* e = std::getenv("HTLR_UPWARD_SLAB");
    force_slab = (e && e[0] == '1') ? 1 : 0;
  }
  if (smem <= 200 * 1024 && !force_slab) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(upward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    upward_kernel<<<dim3((unsigned)nc, R), 256, smem, st>>>(u, W, d, n, side, p, level, R, K_pad, Q, qstride, c0,
                                                            zpitch);
    return;
  }
  const int P = (d == 2) ? p * p : p * p * p;
  const size_t smem2 = sizeof(double) * (size_t)(d * side * p + p * side + p * p + P);
  if (smem2 > 48 * 1024)
    cudaFuncSetAttribute(upward_slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  upward_slab_kernel<<<dim3((unsigned)nc, R), 256, smem2, st>>>(u, W, d, n, side, p, level, R, K_pad, Q, qstride,
                                                                c0, zpitch);
}

// ---------------------------------------------------------------------------
// gathered fp64 tensor-core GEMM: the kernels are in htlr_gemm.cu
// (gemm_persistent_kernel, gemm_thin_kernel); here the tile choice and the
// dispatch.
// ---------------------------------------------------------------------------
// Tile layout per matrix size: "thin" (MT = -M_pad, whole matrix per item,
// m8n8k4 chains) when 8-row padding of P is a supported instantiation, else
// 128- (or 64-) row tiles of m16n8k8 fragments.
int gemm_mt_for(int P_out) {
  const int m8 = (P_out + 7) / 8;
  if (gemm_use_persistent() && thin_m8_supported(m8) && P_out != 64) return -8 * m8;
  return P_out <= 64 ? 64 : 128;
}
int gemm_wide_wn() { return 3; }   // 12 consumer warps: measured +1.3% over 8 (cfg4 leaf pass)
int gemm_nt(int MT) { return (MT == 128 && gemm_use_persistent()) ? 32 * gemm_wide_wn() : 64; }

void launch_gemm(int MT, int NT, const double* A, int64_t mat_stride, const double* B, double* C,
                 const GemmTask* tasks, int ntasks, const int2* pairs, int R, int Rc, int K_pad,
                 int M_valid, int ldc, int RT, cudaStream_t st, const double* gen) {
  if (MT < 0) {
    launch_gemm_thin(-MT, NT, A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, st);
    return;
  }
  launch_gemm_persistent(MT, NT, A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, RT, st, gen);
}

// ---------------------------------------------------------------------------
// fused downward pass + epilogue: one CTA per (leaf box, rhs)
//   facc = sum_l (U_l[sub] x U_l[sub] x U_l[sub]) H_l[ancestor]
//   f    = facc + Y + a u      (scattered back to F-order)
// ---------------------------------------------------------------------------
__global__ void downward_kernel(const double* __restrict__ u, double* __restrict__ f,
                                const double* __restrict__ Y, int ldy, const double* __restrict__ avec,
                                double aconst, const double* __restrict__ dvec, int d, int n, int sL, int L, int R,
                                int p, DownParams dp, int64_t b0) {
  extern __shared__ double sm[];
  const int PL = (d == 2) ? sL * sL : sL * sL * sL;
  const int P = (d == 2) ? p * p : p * p * p;
  double* facc = sm;                 // PL
  double* Hs = facc + PL;            // P
  double* E1 = Hs + P;               // sL * p^(d-1)
  double* E2 = E1 + sL * ((d == 2) ? p : p * p);   // sL^2 * p (3-D only)
  double* Us = E2 + ((d == 3) ? sL * sL * p : 0);  // d * sL * p
  const int64_t b = b0 + blockIdx.x;   // leaf box, Morton id
  const int r = blockIdx.y;
  // blockIdx.z: range of slabs of the last axis (small grids split a box
  // over several CTAs; the cheap E1/E2 stages are recomputed by each)
  const int slab = (d == 2) ? sL : sL * sL;
  const int i_lo = (int)((int64_t)blockIdx.z * sL / gridDim.z) * slab;
  const int i_hi = (int)((int64_t)(blockIdx.z + 1) * sL / gridDim.z) * slab;
  int bc[3];
  morton_decode(b, d, L, bc);
  for (int i = i_lo + threadIdx.x; i < i_hi; i += blockDim.x) facc[i] = 0.0;
  for (int li = 0; li < dp.nlev; ++li) {
    const DownLevel lv = dp.lev[li];
    const int shift = L - lv.level;
    int off[3];
    for (int a = 0; a < 3; ++a) off[a] = (bc[a] & ((1 << shift) - 1)) * sL;
    const int64_t anc = b >> (d * shift);   // Morton parent chain
    __syncthreads();
    const double* Hsrc = lv.H + (anc * R + r) * (int64_t)lv.P;
    for (int i = threadIdx.x; i < P; i += blockDim.x) Hs[i] = Hsrc[i];
    if (lv.K) {
      // H-matrix baseline: dense factor row of each point of this leaf box
      // inside its level-l ancestor box (F-order), times H
      __syncthreads();
      const int sl = lv.side;
      for (int i = i_lo + threadIdx.x; i < i_hi; i += blockDim.x) {
        const int x = i % sL, y = (i / sL) % sL, z = i / (sL * sL);
        int64_t row = (off[0] + x) + (int64_t)sl * (off[1] + y);
        if (d == 3) row += (int64_t)sl * sl * (off[2] + z);
        const double* kr = lv.K + row * P;
        double v = 0.0;
        for (int a = 0; a < P; ++a) v += kr[a] * Hs[a];
        facc[i] += v;
      }
      continue;
    }
    for (int i = threadIdx.x; i < d * sL * p; i += blockDim.x) {
      int a = i / (sL * p), rem = i % (sL * p);
      int x = rem / p, col = rem % p;
      const int64_t base = lv.qstride ? (int64_t)(bc[a] >> shift) * lv.qstride : 0;
      Us[i] = lv.Q[base + (off[a] + x) * p + col];
    }
    __syncthreads();
    const double* U1 = Us;
    const double* U2 = Us + sL * p;
    const double* U3 = Us + 2 * sL * p;
    if (d == 2) {
      // E1[x + sL*a2] = sum_a1 U1[x][a1] H[a1 + p*a2]
      for (int i = threadIdx.x; i < sL * p; i += blockDim.x) {
        int x = i % sL, a2 = i / sL;
        double v = 0.0;
        for (int a1 = 0; a1 < p; ++a1) v += U1[x * p + a1] * Hs[a1 + p * a2];
        E1[i] = v;
      }
      __syncthreads();
      for (int i = i_lo + threadIdx.x; i < i_hi; i += blockDim.x) {
        int x = i % sL, y = i / sL;
        double v = 0.0;
        for (int a2 = 0; a2 < p; ++a2) v += U2[y * p + a2] * E1[x + sL * a2];
        facc[i] += v;
      }
    } else {
      for (int i = threadIdx.x; i < sL * p * p; i += blockDim.x) {
        int x = i % sL, a23 = i / sL;
        double v = 0.0;
        for (int a1 = 0; a1 < p; ++a1) v += U1[x * p + a1] * Hs[a1 + p * a23];
        E1[i] = v;   // E1[x + sL*(a2 + p*a3)]
      }
      __syncthreads();
      for (int i = threadIdx.x; i < sL * sL * p; i += blockDim.x) {
        int x = i % sL, y = (i / sL) % sL, a3 = i / (sL * sL);
        double v = 0.0;
        for (int a2 = 0; a2 < p; ++a2) v += U2[y * p + a2] * E1[x + sL * (a2 + p * a3)];
        E2[i] = v;   // E2[x + sL*(y + sL*a3)]
      }
      __syncthreads();
      for (int i = i_lo + threadIdx.x; i < i_hi; i += blockDim.x) {
        int xy = i % (sL * sL), z = i / (sL * sL);
        double v = 0.0;
        for (int a3 = 0; a3 < p; ++a3) v += U3[z * p + a3] * E2[xy + sL * sL * a3];
        facc[i] += v;
      }
    }
  }
  __syncthreads();
  const double* Yb = Y ? Y + ((int64_t)b * R + r) * ldy : nullptr;
  for (int i = i_lo + threadIdx.x; i < i_hi; i += blockDim.x) {
    int x = i % sL, y = (i / sL) % sL, z = i / (sL * sL);
    int64_t gidx = (int64_t)(bc[0] * sL + x) + (int64_t)n * (bc[1] * sL + y);
    if (d == 3) gidx += (int64_t)n * n * (bc[2] * sL + z);
    double uv = u[gidx * R + r];
    double a = avec ? avec[gidx] : aconst;
    if (dvec) a = dvec[gidx] + a;   // mapped grid: per-point cell integral
    double v = facc[i];
    if (Yb) v += Yb[i];
    f[gidx * R + r] = v + a * uv;
  }
}

void launch_downward(const double* u, double* f, const double* Y, int ldy, const double* a_vec,
                     double a_const, const double* dvec, int d, int n, int sL, int L, int R, int p,
                     const DownParams& dp, int64_t b0, int64_t nb, cudaStream_t st) {
  int P = (d == 2) ? p * p : p * p * p;
  int PL = (d == 2) ? sL * sL : sL * sL * sL;
  size_t words = PL + P + sL * ((d == 2) ? p : p * p) + ((d == 3) ? sL * sL * p : 0) + d * sL * p;
  size_t smem = words * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(downward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (nb <= 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ctas = nb * R;
  const int zs = ctas >= 2 * sms ? 1 : (int)std::min<int64_t>(sL, (2 * sms + ctas - 1) / ctas);
  downward_kernel<<<dim3((unsigned)nb, R, zs), 256, smem, st>>>(u, f, Y, ldy, a_vec, a_const, dvec, d, n, sL, L, R,
                                                               p, dp, b0);
}

}  // namespace htlr
