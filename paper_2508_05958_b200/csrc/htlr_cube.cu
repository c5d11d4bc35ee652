// Upward and downward passes of separable plans (p = leaf side = 8, 3-D,
// uniform grid) over *cubes*: the level-(L-1) boxes, 16^3 points = the 8
// sibling leaf boxes of one parent (sm_100a).
//
// Upward (blocks.py:239-247, the reference's per-block contraction
// u_box -> (Q_z (x) Q_y (x) Q_x)^T u over a cluster's points, regrouped): a
// CTA contracts its cube with the level-(L-1) factor Q_c (16 x 8 per axis)
// in three mode products -- z and x on the fp64 tensor pipe, y on DFMA -- and
// stores W_{L-1}[cube] (one CTA owns every entry: no atomics).  A coarser
// level l contracts the same points with Q_l, whose rows over the cube are
// degree-7 polynomials like Q_c's columns, so Q_l[cube rows] = Q_c M_l with
// M_l = Q_c^T Q_l[cube rows] (8 x 8 per axis and sub-position, checked at
// construction to ~1e-15) and
//   W_l[anc] += (M_l (x) M_l (x) M_l)^T W_{L-1}[cube]
// (three 8 x 8 mode products and one fp64 RED per entry).  The permute (u in
// F-order -> the pitched leaf boxes ub the leaf pass reads) is fused in.
//
// Downward (blocks.py:251-258 + operators.py:153-156, the mirror):
//   H_eff = H_{L-1}[cube] + sum_l (M_l (x) M_l (x) M_l) H_l[anc_l],
//   f = (Q_c (x) Q_c (x) Q_c) H_eff + Y + a u     over the cube's points.
//
// Work split: warp w owns the cube's point rows y = 2w, 2w + 1.  Per row the
// 16 x 16 (x, z) slab is the B operand of mode z straight from registers
// (loaded from global, no staging); its C fragment is reused as the B operand
// of mode x with a permuted k order; mode y crosses warps (a shared-memory
// sum of the 8 warps' partial W in the upward pass; H_eff in shared memory,
// read by every warp, in the downward pass).
//
// Fragment layouts (mma.m8n8k4.row.col.f64): A: lane holds A[g][q]; B: lane
// holds B[q][g]; C: lane holds C[g][2q + j], g = lane / 4, q = lane % 4.
#include "htlr_device.cuh"
#include "htlr_kernels.h"

namespace htlr {

namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

constexpr int kCubeThreads = 256;
constexpr int kHP = 72;   // H_eff c-plane pitch (= 8 mod 16: double2 reads of (a, a + 1) conflict free)

// T = (M_x (x) M_y (x) M_z)^T S  (TR = true) or (M_x (x) M_y (x) M_z) S
// (TR = false) for one 8^3 tensor at a + 8 b + 64 c, mode by mode through two
// shared scratch tensors; every thread handles entries tid, tid + 256.
// Returns the result in t2 (entries e = tid, tid + 256 in out[0..1]).
template <bool TR>
__device__ __forceinline__ void transfer3(const double* __restrict__ M, const double* __restrict__ S, double* t1,
                                          double* t2, double (&out)[2]) {
  auto m = [&](int axis, int from, int to) {   // factor entry coupling index 'from' (source) -> 'to'
    const double* Ma = M + axis * 64;
    return TR ? Ma[from * 8 + to] : Ma[to * 8 + from];
  };
  const int tid = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 2; ++k) {   // mode x
    const int e = tid + kCubeThreads * k, a = e & 7, rest = e & ~7;
    double v = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) v = fma(m(0, s, a), S[rest + s], v);
    t1[e] = v;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 2; ++k) {   // mode y
    const int e = tid + kCubeThreads * k, b = (e >> 3) & 7, rest = e & ~56;
    double v = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) v = fma(m(1, s, b), t1[rest + 8 * s], v);
    t2[e] = v;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 2; ++k) {   // mode z
    const int e = tid + kCubeThreads * k, c = e >> 6, rest = e & 63;
    double v = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) v = fma(m(2, s, c), t2[rest + 64 * s], v);
    out[k] = v;
  }
}

// stage the M tables of the coarser levels at the cube's sub-positions:
// ms[li][axis][64]
__device__ __forceinline__ void stage_transfers(const CubeLevels& cl, const int* cc, int L, double* ms) {
  for (int li = 0; li < cl.ncoarse; ++li) {
    const int span = L - 1 - cl.lev[li].level;   // cube levels below the ancestor
    for (int e = threadIdx.x; e < 3 * 64; e += kCubeThreads) {
      const int a = e >> 6, s = cc[a] & ((1 << span) - 1);
      ms[li * 192 + e] = __ldg(cl.lev[li].M + s * 64 + (e & 63));
    }
  }
}

__global__ void __launch_bounds__(kCubeThreads, 4)
    upward_cube_kernel(CubeLevels cl, int L, int R, int64_t nb, const double* __restrict__ u,
                       double* __restrict__ ub_out, int ldub, int zpub, int n, int zlo, int zhi) {
  extern __shared__ __align__(16) double smc[];
  double* qs = smc;                      // Q_c [16][8]
  double* ms = qs + 128;                 // [coarse level][axis][8 x 8]
  double* red = ms + kMaxCubeCoarse * 192;   // [warp][b][lane][2], then W_{L-1} / transfer scratch
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  const int r = blockIdx.y;
  const int64_t bb = 8 * (int64_t)blockIdx.x;   // first leaf box (Morton) of the cube
  if (bb >= nb) return;
  int c0[3];
  morton_decode(bb, 3, L, c0);                  // even leaf-box coordinates
  if (c0[2] < zlo || c0[2] >= zhi) return;      // z-slab shards / host-pipeline slabs: whole cubes
  const int cc[3] = {c0[0] >> 1, c0[1] >> 1, c0[2] >> 1};
  const int64_t n2 = (int64_t)n * n;
  // this warp's rows y0, y0 + 1 of the cube: B fragments of mode z, (x = 8 h
  // + g, z = 4 ks + q), loaded before anything else
  double v[2][2][4];
  {
    const int64_t base = (int64_t)(8 * c0[0] + g) + (int64_t)n * (8 * c0[1] + 2 * w) + n2 * (8 * c0[2] + q);
#pragma unroll
    for (int yy = 0; yy < 2; ++yy)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          v[yy][h][ks] = __ldg(u + (base + 8 * h + (int64_t)n * yy + n2 * 4 * ks) * R + r);
  }
  if (threadIdx.x < 128 && cl.Qc) qs[threadIdx.x] = __ldg(cl.Qc + threadIdx.x);
  stage_transfers(cl, cc, L, ms);
  // the permute: every loaded point to its pitched leaf box in ub (skipped
  // when the leaf pass reads u itself)
#pragma unroll
  for (int yy = 0; yy < 2 && ub_out; ++yy) {
    const int y = 2 * w + yy;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int z = 4 * ks + q;
        const int64_t box = bb + ((h << 2) | ((y >> 3) << 1) | (z >> 3));
        ub_out[(box * R + r) * ldub + g + 8 * (y & 7) + zpub * (z & 7)] = v[yy][h][ks];
      }
  }
  if (!cl.Qc) return;   // no compressed level: the permute only
  __syncthreads();
  // mode z: Z[c][x] = sum_z Qc[z][c] u[x][z]  (A[m = c][k = z], per x half h)
  double zc[2][2][2];
#pragma unroll
  for (int yy = 0; yy < 2; ++yy)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      zc[yy][h][0] = zc[yy][h][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) dmma(zc[yy][h][0], zc[yy][h][1], qs[(4 * ks + q) * 8 + g], v[yy][h][ks]);
    }
  // mode x: E[a][c] = sum_x Qc[x][a] Z[c][x]  (Z's C fragment as B: k = x = 8 h + 2 q + j)
  double e[2][2];
#pragma unroll
  for (int yy = 0; yy < 2; ++yy) {
    e[yy][0] = e[yy][1] = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma(e[yy][0], e[yy][1], qs[(8 * h + 2 * q + j) * 8 + g], zc[yy][h][j]);
  }
  // mode y (DFMA): P[a][b][c] = sum_{y in the warp} Qc[y][b] E_y[a][c]
  double2* red2 = reinterpret_cast<double2*>(red);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const double m0 = qs[(2 * w) * 8 + b], m1 = qs[(2 * w + 1) * 8 + b];
    red2[(w * 8 + b) * 32 + lane] = make_double2(fma(m1, e[1][0], m0 * e[0][0]), fma(m1, e[1][1], m0 * e[0][1]));
  }
  __syncthreads();
  // W_{L-1}[a][b][c] = sum over the 8 warps; entry (b, lane', j) -> a = lane' / 4, c = 2 (lane' % 4) + j
  double wv[2];
  int widx[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int ent = threadIdx.x + kCubeThreads * k, b = ent >> 6, ln = (ent >> 1) & 31, j = ent & 1;
    double s = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) s += red[ww * 512 + ent];
    wv[k] = s;
    widx[k] = (ln >> 2) + 8 * b + 64 * (2 * (ln & 3) + j);
  }
  __syncthreads();   // red is reused below
  double* wc = red;          // W_{L-1} at a + 8 b + 64 c
  double* t1 = red + 512;
  double* t2 = red + 1024;
  {
    const int64_t cube = bb >> 3;
    double* W = cl.Wc + (cube * R + r) * (int64_t)cl.K_pad_c;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int a = widx[k] & 7, b = (widx[k] >> 3) & 7, c = widx[k] >> 6;
      W[a + 8 * b + cl.zpitch_c * c] = wv[k];
      wc[widx[k]] = wv[k];
    }
  }
  for (int li = 0; li < cl.ncoarse; ++li) {
    __syncthreads();
    double t[2];
    transfer3<true>(ms + li * 192, wc, t1, t2, t);
    const CubeLevel lv = cl.lev[li];
    const int64_t anc = bb >> (3 * (L - lv.level));
    double* W = lv.W + (anc * R + r) * (int64_t)lv.K_pad;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int ent = threadIdx.x + kCubeThreads * k, a = ent & 7, b = (ent >> 3) & 7, c = ent >> 6;
      atomicAdd(W + a + 8 * b + lv.zpitch * c, t[k]);
    }
  }
}

__global__ void __launch_bounds__(kCubeThreads, 4)
    downward_cube_kernel(CubeLevels cl, int L, int R, int64_t b0, int64_t nb, const double* __restrict__ u,
                         double* __restrict__ f, const double* __restrict__ Y, const double* __restrict__ avec,
                         double aconst, int n, int zlo, int zhi, int red) {
  extern __shared__ __align__(16) double smc[];
  double* qs = smc;                      // Q_c [16][8]
  double* ms = qs + 128;                 // [coarse level][axis][8 x 8]
  double* hs = ms + kMaxCubeCoarse * 192;    // staged H: [level][512]
  double* he = hs + (kMaxCubeCoarse + 1) * 512;   // H_eff at a + 8 b + kHP c
  double* t1 = he + 8 * kHP;
  double* t2 = t1 + 512;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  const int r = blockIdx.y;
  const int64_t bb = b0 + 8 * (int64_t)blockIdx.x;
  if (bb >= b0 + nb) return;
  int c0[3];
  morton_decode(bb, 3, L, c0);
  if (c0[2] < zlo || c0[2] >= zhi) return;
  const int cc[3] = {c0[0] >> 1, c0[1] >> 1, c0[2] >> 1};
  const int64_t n2 = (int64_t)n * n;
  const bool has_h = cl.Qc != nullptr;
  if (has_h) {
    if (threadIdx.x < 128) qs[threadIdx.x] = __ldg(cl.Qc + threadIdx.x);
    stage_transfers(cl, cc, L, ms);
    // H_{L-1}[cube] and every coarser level's H at the ancestor, 16 B copies in flight together
    for (int li = 0; li <= cl.ncoarse; ++li) {
      const double* src = li == 0 ? cl.Hc + ((bb >> 3) * R + r) * 512
                                  : cl.lev[li - 1].H + ((bb >> (3 * (L - cl.lev[li - 1].level))) * R + r) * 512;
      const unsigned d = (unsigned)__cvta_generic_to_shared(hs + li * 512 + 2 * threadIdx.x);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + 2 * threadIdx.x) : "memory");
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    double acc[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) acc[k] = hs[threadIdx.x + kCubeThreads * k];
    for (int li = 0; li < cl.ncoarse; ++li) {
      double t[2];
      transfer3<false>(ms + li * 192, hs + (li + 1) * 512, t1, t2, t);
      acc[0] += t[0];
      acc[1] += t[1];
      __syncthreads();   // t1 / t2 reused by the next level
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int ent = threadIdx.x + kCubeThreads * k;
      he[(ent & 63) + kHP * (ent >> 6)] = acc[k];
    }
    __syncthreads();
  }
#pragma unroll 1
  for (int yy = 0; yy < 2; ++yy) {
    const int y = 2 * w + yy;
    double fz[2][2][2];   // [hz][h][j]: (z = 8 hz + g, x = 8 h + 2 q + j)
#pragma unroll
    for (int hz = 0; hz < 2; ++hz)
#pragma unroll
      for (int h = 0; h < 2; ++h) fz[hz][h][0] = fz[hz][h][1] = 0.0;
    if (has_h) {
      // mode y (DFMA): G[c = g][a = 2 q + j] = sum_b Qc[y][b] H_eff[a][b][c]
      double gv[2] = {0.0, 0.0};
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const double m = qs[y * 8 + b];
        const double2 hv = *reinterpret_cast<const double2*>(he + 2 * q + 8 * b + kHP * g);
        gv[0] = fma(m, hv.x, gv[0]);
        gv[1] = fma(m, hv.y, gv[1]);
      }
      // mode x: E[x][c] = sum_a Qc[x][a] G[a][c]  (G as B: k = a = 2 q + j, n = c = g)
      double ex[2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        ex[h][0] = ex[h][1] = 0.0;
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(ex[h][0], ex[h][1], qs[(8 * h + g) * 8 + 2 * q + j], gv[j]);
      }
      // mode z: F[z][x] = sum_c Qc[z][c] E[x][c]  (E as B: k = c = 2 q + j, n = x = g)
#pragma unroll
      for (int hz = 0; hz < 2; ++hz)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma(fz[hz][h][0], fz[hz][h][1], qs[(8 * hz + g) * 8 + 2 * q + j], ex[h][j]);
    }
    // epilogue: f = F + Y + a u at (x = 8 h + 2 q + j, y, z = 8 hz + g)
#pragma unroll
    for (int hz = 0; hz < 2; ++hz)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t box = bb + ((h << 2) | ((y >> 3) << 1) | hz);
        const int64_t gi = (int64_t)(8 * c0[0] + 8 * h + 2 * q) + (int64_t)n * (8 * c0[1] + y) +
                           n2 * (8 * c0[2] + 8 * hz + g);
        double o[2] = {fz[hz][h][0], fz[hz][h][1]};
        if (Y) {
          const double* yb = Y + (box * R + r) * 512 + 2 * q + 8 * (y & 7) + 64 * g;
          o[0] += __ldg(yb);
          o[1] += __ldg(yb + 1);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const double a = avec ? __ldg(avec + gi + j) : aconst;
          if (a != 0.0) o[j] = fma(a, __ldg(u + (gi + j) * R + r), o[j]);
        }
        if (red) {   // f is summed: the leaf pass adds its share itself (band_plane_kernel, fred)
          atomicAdd(f + gi * R + r, o[0]);
          atomicAdd(f + (gi + 1) * R + r, o[1]);
        } else if (R == 1) {
          *reinterpret_cast<double2*>(f + gi) = make_double2(o[0], o[1]);
        } else {
          f[gi * R + r] = o[0];
          f[(gi + 1) * R + r] = o[1];
        }
      }
  }
}

}  // namespace

bool cube_supported(int d, int p, int sL, int L) { return d == 3 && p == kSepP && sL == kSepP && L >= 1; }

void launch_upward_cube(const CubeLevels& cl, int L, int R, int64_t nb, cudaStream_t st, const double* u,
                        double* ub_out, int ldub, int zpub, int n, int zlo, int zhi) {
  if (nb <= 0) return;
  const size_t smem = (size_t)(128 + kMaxCubeCoarse * 192 + 4096) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(upward_cube_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  upward_cube_kernel<<<dim3((unsigned)((nb + 7) / 8), R), kCubeThreads, smem, st>>>(cl, L, R, nb, u, ub_out, ldub,
                                                                                    zpub, n, zlo, zhi);
}

void launch_downward_cube(const CubeLevels& cl, int L, int R, int64_t b0, int64_t nb, cudaStream_t st,
                          const double* u, double* f, const double* Y, const double* a_vec, double a_const, int n,
                          int zlo, int zhi, bool red) {
  if (nb <= 0) return;
  const size_t smem =
      (size_t)(128 + kMaxCubeCoarse * 192 + (kMaxCubeCoarse + 1) * 512 + 8 * kHP + 1024) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(downward_cube_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  downward_cube_kernel<<<dim3((unsigned)((nb + 7) / 8), R), kCubeThreads, smem, st>>>(cl, L, R, b0, nb, u, f, Y,
                                                                                      a_vec, a_const, n, zlo, zhi,
                                                                                      red ? 1 : 0);
}

}  // namespace htlr
