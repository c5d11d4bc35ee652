// Separable-core formulation of the HTLR coupling and near-field passes
// (sm_100a), for tensor-product kernels on uniform grids (the Gaussian,
// kernels.py:90-92: exp(-|x-y|^2 / (2 s^2)) = prod_a exp(-(x_a-y_a)^2 / (2 s^2))).
//
// The reference's admissible block (blocks.py:126-164) is
//   (U_1 x U_2 x U_3) . core . (V_1 x V_2 x V_3)^T,
//   core = multi_mode_apply(h^d G, [R_u1, R_v1, R_u2, R_v2, ...]),
//   G[t, s] = k(xi_t, eta_s) on the tensor Chebyshev grids (chebyshev.py:69-85).
// For a tensor-product kernel G = G_1 (x) G_2 (x) G_3 with 1-D samples
// G_a[t, s] = g(xi_t^a - eta_s^a), and every mode product acts on one factor,
// so the core is exactly the Kronecker product of three p x p matrices
//   C_a(o_a) = h R G_a(o_a) R^T
// (R = the level's QR factor, or the raw Lagrange factor when side == p,
// blocks.py:155-162), each depending only on the per-axis box offset o_a on a
// uniform grid.  Likewise the near block (blocks.py:190-227) is
// (x)_a E(o_a), E[i, j] = h g(x_i - y_j), except for the tau == sigma
// diagonal, which the reference replaces by the cell average (kernels.py:
// 120-149): a rank-one-per-entry correction (corr * u_tau) added by the item
// that owns the self pair.  So every (target, source) pair of a pass applies
//   Y_tau += (C(o_z) (x) C(o_y) (x) C(o_x)) X_sigma      (F-order vectors)
// -- three 8 x 8 mode products (3 * 8^4 MAC) instead of one 512 x 512 GEMV
// (8^6 MAC): the same operator, 85x fewer flops.
//
// sep_apply_kernel: one warp per work item = (target, run of its pairs, rhs).
// Pairs of a target are sorted by (kind, o_x, o_y, o_z); the mode-z product
// runs per pair on the fp64 tensor pipe (mma.m8n8k4, 16 DMMA), accumulating
// Z over a run of equal (kind, o_x, o_y) ("group"); at a group boundary the
// mode-x product (16 DMMA, the C fragment of mode z is reused as the B
// operand with a permuted k order, no shuffles) and the mode-y product
// (128 DFMA per lane) fold Z into the target's accumulator Y (registers).  The
// item ends with an fp64 RED of Y into the pass's accumulator (H_l or the
// leaf-level Y), which the matvec prologue zeroed.
//
// Fragment layouts (mma.m8n8k4.row.col.f64): A: lane holds A[lane/4][lane%4];
// B: lane holds B[lane%4][lane/4]; C: lane holds C[lane/4][2(lane%4) + j].
//   X (source tensor X[a,b,c] at a + 8b + 64c): B operand of tile t = b,
//     k-step ks: X[a = lane/4, b = t, c = 4 ks + lane%4]
//   Z_t[k', a] (C fragment)      = sum_c Mz[k', c] X[a, t, c]
//   T_t[i, k'] (C fragment)      = sum_a Mx[i, a] Z_t[k', a]
//   Y[i, j, k'] (lane: i = lane/4, k' = 2(lane%4) + jj)
//                               += sum_t My[j, t] T_t[i, k']
#include "htlr_device.cuh"
#include "htlr_kernels.h"
#include "htlr_mbarrier.cuh"

#include <algorithm>
#include <cstdlib>

namespace htlr {

namespace {

// not volatile: pure register op, so the compiler may interleave independent
// accumulator chains
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// 1-D factor of the Gaussian: g(delta) = exp(-delta^2 / (2 s^2))
__device__ __forceinline__ double gauss1d(double delta, double denom) {
  return exp(-__dmul_rn(delta, delta) / denom);
}

// One table slot per (kind, per-axis offset): the 8 x 8 matrix M in the three
// fragment orders the apply kernel reads, plus row-major for export.
__global__ void sep_tables_kernel(const SepJob* __restrict__ jobs, int p, int sL, double h, KernelParams kp,
                                  const double* __restrict__ diag, double hd, double* __restrict__ corr_out) {
  const SepJob jb = jobs[blockIdx.x];
  __shared__ double G[kSepP * kSepP], T[kSepP * kSepP], M[kSepP * kSepP];
  const int tid = threadIdx.x;   // 64 threads: one entry each
  const int i = tid / kSepP, j = tid % kSepP;
  if (jb.kind == 1) {
    // near block factor (blocks.py:225-226): x_i = (t0 sL + i + 1/2) h, y_j likewise
    const double x = __dmul_rn(__dadd_rn((double)(jb.t0 * sL + i), 0.5), h);
    const double y = __dmul_rn(__dadd_rn((double)((jb.t0 + jb.o) * sL + j), 0.5), h);
    M[tid] = __dmul_rn(h, gauss1d(__dadd_rn(x, -y), kp.denom));
  } else {
    // Chebyshev nodes of the target box [t0 s h, (t0+1) s h) and the source box
    const double tlo = (double)(jb.t0 * jb.side) * h, thi = (double)((jb.t0 + 1) * jb.side) * h;
    const double slo = (double)((jb.t0 + jb.o) * jb.side) * h, shi = (double)((jb.t0 + jb.o + 1) * jb.side) * h;
    const double xi = cheb_node(tlo, thi, i + 1, p), eta = cheb_node(slo, shi, j + 1, p);
    G[tid] = __dmul_rn(h, gauss1d(__dadd_rn(xi, -eta), kp.denom));
    __syncthreads();
    // T = R G (target mode), M = T R^T (source mode); R row-major p x p
    double acc = 0.0;
    for (int k = 0; k < p; ++k) acc += jb.R[i * p + k] * G[k * kSepP + j];
    T[tid] = acc;
    __syncthreads();
    acc = 0.0;
    for (int k = 0; k < p; ++k) acc += T[i * kSepP + k] * jb.R[j * p + k];
    M[tid] = acc;
  }
  __syncthreads();
  double* dst = jb.dst;
  // [0, 64): mode-z A fragments, [ks][lane] = M[lane/4][4 ks + lane%4]
  // [64, 128): mode-x A fragments, [ks][lane] = M[lane/4][2 (lane%4) + ks]
  // [128, 192): mode-y scalars, [t][j] = scale * M[j][t]
  // [192, 256): M row-major (unscaled; block export)
  {
    const int ks = tid / 32, lane = tid % 32;
    dst[tid] = M[(lane >> 2) * kSepP + 4 * ks + (lane & 3)];
    dst[64 + tid] = M[(lane >> 2) * kSepP + 2 * (lane & 3) + ks];
    dst[128 + tid] = kp.scale * M[j * kSepP + i];   // tid = t * 8 + j with t = i
    dst[192 + tid] = M[tid];
  }
  if (jb.kind == 1 && jb.o == 0 && tid == 0 && corr_out) {
    // self block diagonal: reference value hd * cell average, Kronecker value
    // scale * E(0)[0][0]^3 (the product the apply kernel forms)
    const double e = M[0];
    corr_out[0] = hd * diag[0] - (kp.scale * e) * e * e;
  }
}

// Group flush shared by both apply kernels: Y += My(o_y) . (Mx(o_x) . Z).
__device__ __forceinline__ void sep_flush(const double* __restrict__ tab, int g, int NO, int lane,
                                          double (&z)[kSepP][2], double (&y)[kSepP][2]) {
  const int kind = g >> 8, ox = (g >> 4) & 15, oy = g & 15;
  const double* ax = tab + (kind * NO + ox) * kSepSlotSmem + 64;
  const double b0 = ax[lane], b1 = ax[32 + lane];
  const double* my = tab + (kind * NO + oy) * kSepSlotSmem + 128;
  // mode x for every t (k-step 0 of all tiles, then k-step 1: dependent DMMAs
  // 8 apart), then mode y
  double tt[kSepP][2];
#pragma unroll
  for (int t = 0; t < kSepP; ++t) tt[t][0] = tt[t][1] = 0.0;
#pragma unroll
  for (int t = 0; t < kSepP; ++t) dmma(tt[t][0], tt[t][1], b0, z[t][0]);
#pragma unroll
  for (int t = 0; t < kSepP; ++t) dmma(tt[t][0], tt[t][1], b1, z[t][1]);
#pragma unroll
  for (int t = 0; t < kSepP; ++t) {
    const double2* mv = reinterpret_cast<const double2*>(my + t * kSepP);
#pragma unroll
    for (int jp = 0; jp < kSepP / 2; ++jp) {
      const double2 m = mv[jp];
      y[2 * jp][0] = fma(m.x, tt[t][0], y[2 * jp][0]);
      y[2 * jp][1] = fma(m.x, tt[t][1], y[2 * jp][1]);
      y[2 * jp + 1][0] = fma(m.y, tt[t][0], y[2 * jp + 1][0]);
      y[2 * jp + 1][1] = fma(m.y, tt[t][1], y[2 * jp + 1][1]);
    }
    z[t][0] = z[t][1] = 0.0;
  }
}

template <bool kSelfCorr>
__device__ __forceinline__ void sep_item(const double* __restrict__ tab, const SepItem& it, const int2* __restrict__ pr,
                                         const double* __restrict__ B, int ldb, double* __restrict__ C, int ldc, int R,
                                         int r, double corr, int NO, int lane, int zp) {
  double y[kSepP][2];
#pragma unroll
  for (int j = 0; j < kSepP; ++j) y[j][0] = y[j][1] = 0.0;
  double z[kSepP][2];
#pragma unroll
  for (int t = 0; t < kSepP; ++t) z[t][0] = z[t][1] = 0.0;
  const int boff = (lane >> 2) + zp * (lane & 3);
  auto load = [&](double (&x)[kSepP][2], int src) {
    const double* s = B + ((int64_t)src * R + r) * ldb + boff;
#pragma unroll
    for (int t = 0; t < kSepP; ++t) {
      x[t][0] = __ldg(s + 8 * t);
      x[t][1] = __ldg(s + 8 * t + 4 * zp);
    }
  };
  int2 cur = pr[0];
  double xb[kSepP][2];
  load(xb, cur.x);
  for (int q = 0; q < it.count; ++q) {
    const bool more = q + 1 < it.count;
    const int2 nxt = more ? pr[q + 1] : cur;
    double xn[kSepP][2];
    if (more) load(xn, nxt.x);
    // mode z (per pair): Z_t += Mz(o_z) X_t
    {
      const int code = cur.y;
      const double* az = tab + ((code >> 12) * NO + (code & 15)) * kSepSlotSmem;
      const double a0 = az[lane], a1 = az[32 + lane];
#pragma unroll
      for (int t = 0; t < kSepP; ++t) dmma(z[t][0], z[t][1], a0, xb[t][0]);
#pragma unroll
      for (int t = 0; t < kSepP; ++t) dmma(z[t][0], z[t][1], a1, xb[t][1]);
    }
    const int g = cur.y >> 4;
    if (!more || (nxt.y >> 4) != g) {
      sep_flush(tab, g, NO, lane, z, y);
    }
    if (more) {
#pragma unroll
      for (int t = 0; t < kSepP; ++t) {
        xb[t][0] = xn[t][0];
        xb[t][1] = xn[t][1];
      }
      cur = nxt;
    }
  }
  const int yoff = (lane >> 2) + 128 * (lane & 3);   // i + 64 k', k' = 2 (lane % 4) + jj
  if (kSelfCorr) {
    const double* s = B + ((int64_t)it.tgt * R + r) * ldb + (lane >> 2) + 2 * zp * (lane & 3);
#pragma unroll
    for (int j = 0; j < kSepP; ++j) {
      y[j][0] = fma(corr, __ldg(s + 8 * j), y[j][0]);
      y[j][1] = fma(corr, __ldg(s + 8 * j + zp), y[j][1]);
    }
  }
  double* o = C + ((int64_t)it.tgt * R + r) * ldc + yoff;
#pragma unroll
  for (int j = 0; j < kSepP; ++j) {
    atomicAdd(o + 8 * j, y[j][0]);
    atomicAdd(o + 8 * j + 64, y[j][1]);
  }
}

__global__ void __launch_bounds__(kSepWarps * 32)
    sep_apply_kernel(const double* __restrict__ tables, int nslots, int NO, const SepItem* __restrict__ items,
                     int nitems, const int2* __restrict__ pairs, const double* __restrict__ B, int ldb,
                     double* __restrict__ C, int ldc, int R, const double* __restrict__ corr_ptr, int zp) {
  extern __shared__ double tab[];
  for (int e = threadIdx.x; e < nslots * kSepSlotSmem; e += blockDim.x)
    tab[e] = tables[(e / kSepSlotSmem) * kSepSlot + e % kSepSlotSmem];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * kSepWarps + (threadIdx.x >> 5);
  if (item >= nitems) return;
  const SepItem it = items[item];
  const int r = blockIdx.y;
  if (it.flags & 1)
    sep_item<true>(tab, it, pairs + it.begin, B, ldb, C, ldc, R, r, corr_ptr[0], NO, lane, zp);
  else
    sep_item<false>(tab, it, pairs + it.begin, B, ldb, C, ldc, R, r, 0.0, NO, lane, zp);
}

// Cooperative pass, persistent: CTA i walks the parts i, i + grid, ... (a
// part = a parent cluster and a run of the source columns of its 8 children;
// parts sorted longest first).  NG groups of 8 consumer warps (warp w applies
// the blocks of child target tgt0 + w % 8; group w / 8 takes every NG-th
// column of the CTA's column sequence) and a producer warp that bulk-copies
// every source box of a column once, as 8 z-planes at a 68-double pitch (so
// the mode-z B fragments -- lanes a = lane/4, c = 4 ks + lane%4 -- hit 32
// distinct banks), into a ring of NS = sep_ring_slots(NG) column slots (full /
// empty mbarriers); the ring runs across part boundaries, so the next part's
// columns load while the current one finishes.  A column has fixed (o_x, o_y)
// for every warp, so a warp flushes its Z accumulator when the block kind
// changes along the column and at its end (one flush for the far columns, at
// most three where near blocks sit between admissible ones).  At the end of a
// part each group adds its partial Y into C (fp64 RED).
template <int NG>
__global__ void __launch_bounds__((8 * NG + 1) * 32, 1)
    sep_block_kernel(const double* __restrict__ tables, int nslots, int NO, const SepBlock* __restrict__ blocks,
                     int nblocks, const SepCol* __restrict__ cols, const double* __restrict__ B, int ldb,
                     double* __restrict__ C, int ldc, int R, const double* __restrict__ corr_ptr, int zp) {
  constexpr int NS = sep_ring_slots(NG), SLOT = kSepColMax * kSepBoxSmem, NCW = 8 * NG;
  extern __shared__ __align__(16) double sm[];
  double* tab = sm;
  double* ring = tab + nslots * kSepSlotSmem;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * SLOT);
  uint64_t* empty = full + NS;
  const int r = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int e = threadIdx.x; e < nslots * kSepSlotSmem; e += blockDim.x)
    tab[e] = tables[(e / kSepSlotSmem) * kSepSlot + e % kSepSlotSmem];
  __syncthreads();
  if (warp == NCW) {
    // ------------------------------------------------------------ producer
    int gc = 0;   // column index in this CTA's sequence (ring position)
    for (int part = blockIdx.x; part < nblocks; part += gridDim.x) {
      const SepBlock bk = blocks[part];
      const SepCol* cl = cols + bk.col_begin;
      for (int c = 0; c < bk.col_count; ++c, ++gc) {
        const int slot = gc % NS;
        if (gc >= NS) mbar_wait(&empty[slot], (unsigned)(((gc / NS) - 1) & 1));
        const int n = cl[c].n;
        double* dst = ring + slot * SLOT;
        if (zp == kSepZPitch) {
          // boxes stored pitched: one bulk copy per box
          if (lane == 0) mbar_arrive_expect_tx(&full[slot], (unsigned)(n * kSepBoxSmem * 8));
          __syncwarp();
          if (lane < n)
            bulk_g2s(dst + lane * kSepBoxSmem, B + ((int64_t)cl[c].src[lane] * R + r) * ldb, kSepBoxSmem * 8,
                     &full[slot]);
        } else {
          // natural layout: 8 plane copies per box into the padded slots
          if (lane == 0) mbar_arrive_expect_tx(&full[slot], (unsigned)(n * 512 * 8));
          __syncwarp();
          for (int e = lane; e < n * 8; e += 32) {
            const int k = e >> 3, pl = e & 7;
            bulk_g2s(dst + k * kSepBoxSmem + pl * 68, B + ((int64_t)cl[c].src[k] * R + r) * ldb + pl * 64, 64 * 8,
                     &full[slot]);
          }
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------- consumers
  const int tw = warp & 7, grp = warp >> 3;
  const int xoff = (lane >> 2) + 68 * (lane & 3);
  const int yoff = (lane >> 2) + 128 * (lane & 3);
  double y[kSepP][2], z[kSepP][2];
#pragma unroll
  for (int j = 0; j < kSepP; ++j) y[j][0] = y[j][1] = z[j][0] = z[j][1] = 0.0;
  int gc0 = 0;   // first ring position of the current part
  for (int part = blockIdx.x; part < nblocks; part += gridDim.x) {
    const SepBlock bk = blocks[part];
    const SepCol* cl = cols + bk.col_begin;
    // this group's first column of the part
    int c = ((grp - gc0) % NG + NG) % NG;
    const bool mine = c < bk.col_count;
    for (; c < bk.col_count; c += NG) {
      const int gc = gc0 + c;
      const int slot = gc % NS;
      const int n = cl[c].n;
      // the column's pair codes of this warp's target, one per lane
      const int mycode = lane < n ? (int)cl[c].code[lane][tw] : 0xFFFF;
      mbar_wait(&full[slot], (unsigned)((gc / NS) & 1));
      const double* xs = ring + slot * SLOT + xoff;
      int g = -1;
      for (int k = 0; k < n; ++k) {
        const int code = __shfl_sync(0xffffffffu, mycode, k);
        if (code == 0xFFFF) continue;
        if ((code >> 4) != g) {   // kind change inside the column (o_x, o_y fixed)
          if (g >= 0) sep_flush(tab, g, NO, lane, z, y);
          g = code >> 4;
        }
        double xv[kSepP][2];
#pragma unroll
        for (int t = 0; t < kSepP; ++t) {
          xv[t][0] = xs[k * kSepBoxSmem + 8 * t];
          xv[t][1] = xs[k * kSepBoxSmem + 8 * t + 272];
        }
        const double* az = tab + ((code >> 12) * NO + (code & 15)) * kSepSlotSmem;
        const double a0 = az[lane], a1 = az[32 + lane];
#pragma unroll
        for (int t = 0; t < kSepP; ++t) dmma(z[t][0], z[t][1], a0, xv[t][0]);
#pragma unroll
        for (int t = 0; t < kSepP; ++t) dmma(z[t][0], z[t][1], a1, xv[t][1]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (g >= 0) sep_flush(tab, g, NO, lane, z, y);
    }
    // the group that owns the part's column 0 adds the self-block correction
    const int tgt = bk.tgt0 + tw;
    const bool corr = (gc0 % NG) == grp && ((bk.corr_mask >> tw) & 1);
    if (corr) {
      const double cv = corr_ptr[0];
      const double* s = B + ((int64_t)tgt * R + r) * ldb + (lane >> 2) + 2 * zp * (lane & 3);
#pragma unroll
      for (int j = 0; j < kSepP; ++j) {
        y[j][0] = fma(cv, __ldg(s + 8 * j), y[j][0]);
        y[j][1] = fma(cv, __ldg(s + 8 * j + zp), y[j][1]);
      }
    }
    if (mine || corr) {
      double* o = C + ((int64_t)tgt * R + r) * ldc + yoff;
#pragma unroll
      for (int j = 0; j < kSepP; ++j) {
        atomicAdd(o + 8 * j, y[j][0]);
        atomicAdd(o + 8 * j + 64, y[j][1]);
        y[j][0] = y[j][1] = 0.0;
      }
    }
    gc0 += bk.col_count;
  }
}

// Banded leaf pass (strong admissibility, eta = 1, uniform grid): at the leaf
// level every (target, source) pair is a child pair of an inadmissible parent
// pair, so the offsets o = sigma - tau a target tau meets form product sets:
// per axis o_a = 2 po_a + c'_a - c_a (po = parent offset in {-2..2}^3 minus the
// 8 corners {+-2}^3, c / c' = child positions).  Per axis, with c = tau's
// coordinate parity:
//   all children of the parents:  R10 = {-4-c, ..., 5-c}   (minus the corner
//                                  parents' children: A4 = {-4-c,-3-c,4-c,5-c})
//   leaf near field:               R5  = {-2, ..., 2}        (minus {+-2}^3)
// so, with K_S = sum_{o in S} M(o) shift(o) along one axis (M = the level's
// admissible factor C or the near factor E, htlr_sep.cu header),
//   Y = C10^3 - C4^3 - C5^3 + C2^3 + E5^3 - E2^3   (+ the self-block diagonal
//       correction), X^3 = X_x X_y X_z.
// Every term is a Kronecker product of three block-banded 1-D operators, so
// the pass is three line sweeps (z, then y, then x) over lines of leaf boxes;
// the same blocks as the reference's list (every pair's C(o_x) C(o_y) C(o_z) or
// E(...)), summed in a different order.  The plan checks the leaf lists
// against this structure before it enables the banded pass.
//
// sep_band_kernel<A, MODE>: one CTA per (line of nb boxes along axis A, rhs);
// the line is staged in shared memory as [box][k = coordinate along A][n =
// the other two, pitch 68] (B fragments bank-conflict free), warp w computes
// boxes q = w, w + 16, ...: out[m][n] = sum_{b in S(q)} M(b - q)[m][k]
// X_b[k][n] as 16 DMMA m8n8k4 per (q, b).  MODE 0: in = ub, out = the six
// term buffers; MODE 1: term buffers in place; MODE 2: Y += scale * sum_t
// sign_t term_t + corr * ub.
__device__ __forceinline__ int band_count(int t) { return t == 0 ? 10 : (t == 1 || t == 3 || t == 5) ? ((t == 1) ? 4 : 2) : 5; }
__device__ __forceinline__ int band_off(int t, int c, int i) {
  switch (t) {
    case 0: return -4 - c + i;
    case 1: return i < 2 ? -4 - c + i : 2 - c + i;   // -4-c, -3-c, 4-c, 5-c
    case 3:
    case 5: return i ? 2 : -2;
    default: return i - 2;                           // 2, 4: -2..2
  }
}

constexpr int kBandTerms = 6;
constexpr int kBandWarps = 16;

// element e = x + 8 y + 64 z of a box -> (k, n) for a sweep along axis A
template <int A>
__device__ __forceinline__ int band_kn(int x, int y, int z) {
  if (A == 2) return z * kSepZPitch + x + 8 * y;
  if (A == 1) return y * kSepZPitch + x + 8 * z;
  return x * kSepZPitch + y + 8 * z;
}
// output (m, n) -> natural element index
template <int A>
__device__ __forceinline__ int band_elem(int m, int n) {
  if (A == 2) return n + 64 * m;
  if (A == 1) return (n & 7) + 8 * m + 64 * (n >> 3);
  return m + 8 * n;
}

template <int A, int MODE>
__global__ void __launch_bounds__(kBandWarps * 32, 2)
    sep_band_kernel(const double* __restrict__ tables, int NO, int L, int R, const double* __restrict__ ub,
                    int ldub, int zpub, double* __restrict__ ws, int64_t term_stride, double* __restrict__ Y,
                    const double* __restrict__ corr_ptr, double scale, int nterms, BandRegion rg) {
  extern __shared__ __align__(16) double sm[];
  const int nb = 1 << L;
  double* tab = sm;                          // [kind][offset] A fragments (64 doubles)
  double* line = sm + 2 * NO * 64;           // [box][8][68]
  const int r = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int OR = (NO - 1) / 2;
  int lc[3];
  {
    const int l = blockIdx.x;
    const int a1 = A == 0 ? 1 : 0, a2 = A == 2 ? 1 : 2;
    lc[a1] = l % nb;
    lc[a2] = l / nb;
    lc[A] = 0;
    // sharded plans: only the lines within 5 boxes of the own region matter
    if (MODE == 0 && (lc[a1] < rg.lo[a1] - 5 || lc[a1] >= rg.hi[a1] + 5 || lc[a2] < rg.lo[a2] - 5 ||
                      lc[a2] >= rg.hi[a2] + 5))
      return;
  }
  for (int e = threadIdx.x; e < 2 * NO * 64; e += blockDim.x) tab[e] = tables[(e >> 6) * kSepSlot + (e & 63)];
  __shared__ int64_t bids[16];
  if (threadIdx.x < nb) {
    int c[3] = {lc[0], lc[1], lc[2]};
    c[A] = threadIdx.x;
    bids[threadIdx.x] = morton_encode(c, 3, L);
  }
  __syncthreads();
  auto box_id = [&](int q) { return bids[q]; };
  auto stage = [&](const double* src, int64_t stride_box, int zp) {
    for (int e = threadIdx.x; e < nb * 512; e += blockDim.x) {
      const int q = e >> 9, i = e & 511;
      const int x = i & 7, y = (i >> 3) & 7, z = i >> 6;
      line[q * kSepBoxSmem + band_kn<A>(x, y, z)] = src[(box_id(q) * R + r) * stride_box + x + 8 * y + zp * z];
    }
  };
  // one term's band product for box q into acc
  auto apply = [&](int t, int q, double (&acc)[kSepP][2], double sg) {
    const int kind = t >= 4 ? 1 : 0, c = q & 1, cnt = band_count(t);
    const double* xs = line + (lane & 3) * kSepZPitch + (lane >> 2);
    for (int i = 0; i < cnt; ++i) {
      const int o = band_off(t, c, i), b = q + o;
      if (b < 0 || b >= nb) continue;
      const double* az = tab + (kind * NO + o + OR) * 64;
      const double a0 = sg * az[lane], a1 = sg * az[32 + lane];
      const double* xb = xs + b * kSepBoxSmem;
      double xv[kSepP][2];
#pragma unroll
      for (int t8 = 0; t8 < kSepP; ++t8) {
        xv[t8][0] = xb[8 * t8];
        xv[t8][1] = xb[8 * t8 + 4 * kSepZPitch];
      }
#pragma unroll
      for (int t8 = 0; t8 < kSepP; ++t8) dmma(acc[t8][0], acc[t8][1], a0, xv[t8][0]);
#pragma unroll
      for (int t8 = 0; t8 < kSepP; ++t8) dmma(acc[t8][0], acc[t8][1], a1, xv[t8][1]);
    }
  };
  const int m = lane >> 2, n0 = 2 * (lane & 3);
  if (MODE == 0) {
    if (A == 2 && zpub == kSepZPitch && ldub == kSepBoxSmem) {
      // pitched boxes are already in the z-sweep's staging layout: 16-byte
      // asynchronous copies of the whole box
      for (int e = threadIdx.x; e < nb * (kSepBoxSmem / 2); e += blockDim.x) {
        const int q = e / (kSepBoxSmem / 2), i = 2 * (e % (kSepBoxSmem / 2));
        const double* g = ub + (box_id(q) * R + r) * (int64_t)ldub + i;
        const unsigned d = (unsigned)__cvta_generic_to_shared(line + q * kSepBoxSmem + i);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(g) : "memory");
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
    } else {
      stage(ub, ldub, zpub);
    }
    __syncthreads();
    for (int q = rg.lo[A] + warp; q < rg.hi[A]; q += kBandWarps) {
      const int64_t ob = (box_id(q) * R + r) * 512;
      for (int t = 0; t < nterms; ++t) {
        double acc[kSepP][2];
#pragma unroll
        for (int t8 = 0; t8 < kSepP; ++t8) acc[t8][0] = acc[t8][1] = 0.0;
        apply(t, q, acc, 1.0);
        double* o = ws + t * term_stride + ob;
#pragma unroll
        for (int t8 = 0; t8 < kSepP; ++t8) {
          if (A == 2) {   // n, n + 1 adjacent in memory
            *reinterpret_cast<double2*>(o + band_elem<A>(m, 8 * t8 + n0)) = make_double2(acc[t8][0], acc[t8][1]);
          } else {
            o[band_elem<A>(m, 8 * t8 + n0)] = acc[t8][0];
            o[band_elem<A>(m, 8 * t8 + n0 + 1)] = acc[t8][1];
          }
        }
      }
    }
    return;
  }
  double ya[(MODE == 2) ? 1 : 1][kSepP][2];
  // MODE 2 keeps one accumulator per warp box; nb <= 16 boxes per line -> one box per warp
  for (int q0 = 0; q0 < nb; q0 += kBandWarps) {
    const int q = q0 + warp;
#pragma unroll
    for (int t8 = 0; t8 < kSepP; ++t8) ya[0][t8][0] = ya[0][t8][1] = 0.0;
    for (int t = 0; t < nterms; ++t) {
      __syncthreads();   // previous term's readers are done with the line
      stage(ws + t * term_stride, 512, 64);
      __syncthreads();
      if (q >= nb) continue;
      if (MODE == 1) {
        double acc[kSepP][2];
#pragma unroll
        for (int t8 = 0; t8 < kSepP; ++t8) acc[t8][0] = acc[t8][1] = 0.0;
        apply(t, q, acc, 1.0);
        double* o = ws + t * term_stride + (box_id(q) * R + r) * 512;
#pragma unroll
        for (int t8 = 0; t8 < kSepP; ++t8) {
          o[band_elem<A>(m, 8 * t8 + n0)] = acc[t8][0];
          o[band_elem<A>(m, 8 * t8 + n0 + 1)] = acc[t8][1];
        }
      } else {
        // the term's sign folded into the A fragments: accumulate in place
        apply(t, q, ya[0], (t == 1 || t == 2 || t == 5) ? -1.0 : 1.0);
      }
    }
    if (MODE == 2 && q < nb) {
      const int64_t bid = box_id(q);
      double* o = Y + (bid * R + r) * 512;
      const double* us = ub + (bid * R + r) * ldub;
      const double cv = corr_ptr ? corr_ptr[0] : 0.0;
#pragma unroll
      for (int t8 = 0; t8 < kSepP; ++t8)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int e = band_elem<A>(m, 8 * t8 + n0 + jj);
          const int x = e & 7, y = (e >> 3) & 7, z = e >> 6;
          o[e] = corr_ptr ? fma(scale, ya[0][t8][jj], cv * __ldg(us + x + 8 * y + zpub * z)) : scale * ya[0][t8][jj];
        }
    }
  }
}

// sweeps y and x fused (sep_band_xy_kernel<NB>): the mode-y and mode-x
// products mix only x and y, so one CTA per (z-point plane, rhs) stages the
// plane of a term (NB^2 box cells of 8 x 8 points, [y][x] at a pitch of
// 8 NB + 4 doubles: B fragments bank-conflict free along both axes), runs the
// y sweep into registers (2 DMMA per (cell, source box)), writes it back in
// place, runs the x sweep into the Y accumulator (term sign folded into the A
// fragments) and moves to the next term; at the end Y += scale * acc +
// corr * u.  NB = 16 at the leaf level of config 4: 128 CTAs of 32 warps, 8
// cells per warp (16 registers per lane for each of the two accumulators).
template <int NB>
__host__ __device__ constexpr int band_xy_warps() { return NB >= 16 ? 32 : kBandWarps; }

template <int NB>
__global__ void __launch_bounds__(band_xy_warps<NB>() * 32, 1)
    sep_band_xy_kernel(const double* __restrict__ tables, int NO, int L, int R, const double* __restrict__ ub,
                       int ldub, int zpub, const double* __restrict__ ws, int64_t term_stride, double* __restrict__ Y,
                       const double* __restrict__ corr_ptr, double scale, int nterms, BandRegion rg) {
  constexpr int NW = band_xy_warps<NB>();
  constexpr int CPW = NB * NB / NW;   // cells per warp (one row / column segment)
  constexpr int SEG = NB / CPW;        // segments per row
  constexpr int PITCH = 8 * NB + 4;
  extern __shared__ __align__(16) double sm[];
  double* tab = sm;
  double* P = sm + 2 * NO * 64;
  __shared__ int64_t bids[NB * NB];
  const int r = blockIdx.y, zl = blockIdx.x & 7, bz = rg.lo[2] + (blockIdx.x >> 3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int OR = (NO - 1) / 2;
  for (int e = threadIdx.x; e < 2 * NO * 64; e += blockDim.x) tab[e] = tables[(e >> 6) * kSepSlot + (e & 63)];
  for (int c = threadIdx.x; c < NB * NB; c += blockDim.x) {
    const int cc[3] = {c % NB, c / NB, bz};
    bids[c] = morton_encode(cc, 3, L);
  }
  double yacc[CPW][2];
#pragma unroll
  for (int i = 0; i < CPW; ++i) yacc[i][0] = yacc[i][1] = 0.0;
  const int kq = lane & 3, nq = lane >> 2;
  for (int t = 0; t < nterms; ++t) {
    __syncthreads();
    {
      // asynchronous 16-byte copies: every load of the plane in flight at once
      const double* src = ws + t * term_stride + 64 * zl;
      for (int e = threadIdx.x; e < NB * NB * 32; e += blockDim.x) {
        const int c = e >> 5, i = 2 * (e & 31);
        const double* g = src + (bids[c] * R + r) * 512 + i;
        const unsigned d = (unsigned)__cvta_generic_to_shared(P + (8 * (c / NB) + (i >> 3)) * PITCH + 8 * (c % NB) + (i & 7));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(g) : "memory");
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
    }
    __syncthreads();
    const int kind = t >= 4 ? 1 : 0, cnt = band_count(t);
    // y sweep: acc[y'][x] = sum_o My(o)[y'][y] T[8 (by + o) + y][8 bx + x];
    // the warp's cells share by (a row segment), so one A fragment per offset
    double acc[CPW][2];
#pragma unroll
    for (int i = 0; i < CPW; ++i) acc[i][0] = acc[i][1] = 0.0;
    {
      const int by = warp / SEG, bx0 = (warp % SEG) * CPW;
      const double* xb0 = P + kq * PITCH + 8 * bx0 + nq;
      // sharded plans: only the rows of the own region, columns within 5 boxes of it
      const bool need = by >= rg.lo[1] && by < rg.hi[1] && bx0 < rg.hi[0] + 5 && bx0 + CPW > rg.lo[0] - 5;
      for (int j = 0; j < (need ? cnt : 0); ++j) {
        const int o = band_off(t, by & 1, j), b = by + o;
        if (b < 0 || b >= NB) continue;
        const double* az = tab + (kind * NO + o + OR) * 64;
        const double a0 = az[lane], a1 = az[32 + lane];
        const double* xb = xb0 + 8 * b * PITCH;
#pragma unroll
        for (int i = 0; i < CPW; ++i) dmma(acc[i][0], acc[i][1], a0, xb[8 * i]);
#pragma unroll
        for (int i = 0; i < CPW; ++i) dmma(acc[i][0], acc[i][1], a1, xb[8 * i + 4 * PITCH]);
      }
      __syncthreads();
      double* wb = P + (8 * by + nq) * PITCH + 8 * bx0 + 2 * kq;
#pragma unroll
      for (int i = 0; i < CPW; ++i) *reinterpret_cast<double2*>(wb + 8 * i) = make_double2(acc[i][0], acc[i][1]);
    }
    __syncthreads();
    // x sweep: yacc[x'][y] += sg * sum_o Mx(o)[x'][x] U[8 by + y][8 (bx + o) + x];
    // the warp's cells share bx (a column segment)
    {
      const double sg = (t == 1 || t == 2 || t == 5) ? -1.0 : 1.0;
      const int bx = warp / SEG, by0 = (warp % SEG) * CPW;
      const double* xb0 = P + (8 * by0 + nq) * PITCH + kq;
      const bool need = bx >= rg.lo[0] && bx < rg.hi[0] && by0 < rg.hi[1] && by0 + CPW > rg.lo[1];
      for (int j = 0; j < (need ? cnt : 0); ++j) {
        const int o = band_off(t, bx & 1, j), b = bx + o;
        if (b < 0 || b >= NB) continue;
        const double* az = tab + (kind * NO + o + OR) * 64;
        const double a0 = sg * az[lane], a1 = sg * az[32 + lane];
        const double* xb = xb0 + 8 * b;
#pragma unroll
        for (int i = 0; i < CPW; ++i) dmma(yacc[i][0], yacc[i][1], a0, xb[8 * i * PITCH]);
#pragma unroll
        for (int i = 0; i < CPW; ++i) dmma(yacc[i][0], yacc[i][1], a1, xb[8 * i * PITCH + 4]);
      }
    }
  }
  // epilogue: lane holds (x' = nq, y = 2 kq + jj) of each cell (bx, by0 + i)
  const double cv = corr_ptr ? corr_ptr[0] : 0.0;
  const int bx = warp / SEG, by0 = (warp % SEG) * CPW;
#pragma unroll
  for (int i = 0; i < CPW; ++i) {
    // sharded plans: only the own cells (the rest saw partial halo data)
    if (bx < rg.lo[0] || bx >= rg.hi[0] || by0 + i < rg.lo[1] || by0 + i >= rg.hi[1]) continue;
    const int64_t bid = bids[(by0 + i) * NB + bx];
    double* o = Y + (bid * R + r) * 512 + 64 * zl + nq + 16 * kq;
    const double* us = ub + (bid * R + r) * ldub + zpub * zl + nq + 16 * kq;
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      double v = scale * yacc[i][jj];
      if (corr_ptr) v = fma(cv, __ldg(us + 8 * jj), v);
      o[8 * jj] = v;   // every entry of the level's accumulator is written here once
    }
  }
}

}  // namespace

// consumer warp groups of the cooperative kernel (two: alternate columns)
int sep_block_groups() { return 2; }

size_t sep_block_smem_bytes(int nslots) {
  const int NS = sep_ring_slots(sep_block_groups());
  return ((size_t)nslots * kSepSlotSmem + (size_t)NS * kSepColMax * kSepBoxSmem) * sizeof(double) +
         2 * NS * sizeof(uint64_t);
}

template <int NG>
static void launch_sep_block_t(const double* tables, int nslots, int NO, const SepBlock* blocks, int nblocks,
                               const SepCol* cols, const double* B, int ldb, double* C, int ldc, int R,
                               const double* corr, int zpitch, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sep_block_kernel<NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = nblocks < sms ? nblocks : sms;   // persistent: one CTA per SM
  sep_block_kernel<NG><<<dim3(grid, R), (8 * NG + 1) * 32, sep_block_smem_bytes(nslots), st>>>(
      tables, nslots, NO, blocks, nblocks, cols, B, ldb, C, ldc, R, corr, zpitch ? zpitch : 64);
}

void launch_sep_block(const double* tables, int nslots, int NO, const SepBlock* blocks, int nblocks, const SepCol* cols,
                      const double* B, int ldb, double* C, int ldc, int R, const double* corr, cudaStream_t st,
                      int zpitch) {
  if (nblocks <= 0) return;
  if (sep_block_groups() == 1)
    launch_sep_block_t<1>(tables, nslots, NO, blocks, nblocks, cols, B, ldb, C, ldc, R, corr, zpitch, st);
  else
    launch_sep_block_t<2>(tables, nslots, NO, blocks, nblocks, cols, B, ldb, C, ldc, R, corr, zpitch, st);
}

void launch_sep_tables(const SepJob* jobs, int njobs, int p, int sL, double h, const KernelParams& kp,
                       const double* diag, double hd, double* corr_out, cudaStream_t st) {
  if (njobs <= 0) return;
  sep_tables_kernel<<<njobs, kSepP * kSepP, 0, st>>>(jobs, p, sL, h, kp, diag, hd, corr_out);
}

size_t sep_smem_bytes(int nslots) { return (size_t)nslots * kSepSlotSmem * sizeof(double); }

void launch_sep_apply(const double* tables, int nslots, int NO, const SepItem* items, int nitems, const int2* pairs,
                      const double* B, int ldb, double* C, int ldc, int R, const double* corr, cudaStream_t st,
                      int zpitch) {
  if (nitems <= 0) return;
  const size_t smem = sep_smem_bytes(nslots);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sep_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr = true;
  }
  dim3 grid((nitems + kSepWarps - 1) / kSepWarps, R);
  sep_apply_kernel<<<grid, kSepWarps * 32, smem, st>>>(tables, nslots, NO, items, nitems, pairs, B, ldb, C, ldc, R,
                                                       corr, zpitch ? zpitch : 64);
}


size_t sep_band_smem_bytes(int NO, int L) {
  return ((size_t)2 * NO * 64 + (size_t)(1 << L) * kSepBoxSmem) * sizeof(double);
}

int64_t sep_band_workspace(int L, int R) { return (int64_t)kBandTerms * ((int64_t)1 << (3 * L)) * R * 512; }


template <int A, int MODE>
static void launch_band_t(const double* tables, int NO, int L, int R, const double* ub, int ldub, int zpub,
                          double* ws, double* Y, const double* corr, double scale, int nterms, cudaStream_t st,
                          const BandRegion& rg) {
  const size_t smem = sep_band_smem_bytes(NO, L);
  const int64_t tstride = ((int64_t)1 << (3 * L)) * R * 512;
  sep_band_kernel<A, MODE><<<dim3(1u << (2 * L), R), kBandWarps * 32, smem, st>>>(tables, NO, L, R, ub, ldub, zpub,
                                                                                   ws, tstride, Y, corr, scale,
                                                                                   nterms, rg);
}

size_t sep_band_xy_smem_bytes(int NO, int L) {
  const int nb = 1 << L;
  return ((size_t)2 * NO * 64 + (size_t)(8 * nb) * (8 * nb + 4)) * sizeof(double);
}


template <int NB>
static void launch_band_xy_t(const double* tables, int NO, int L, int R, const double* ub, int ldub, int zpub,
                             const double* ws, double* Y, const double* corr, double scale, int nterms,
                             cudaStream_t st, const BandRegion& rg) {
  const int64_t tstride = ((int64_t)1 << (3 * L)) * R * 512;
  const int planes = 8 * (rg.hi[2] - rg.lo[2]);
  if (planes <= 0) return;
  sep_band_xy_kernel<NB><<<dim3(planes, R), band_xy_warps<NB>() * 32, sep_band_xy_smem_bytes(NO, L), st>>>(
      tables, NO, L, R, ub, ldub, zpub, ws, tstride, Y, corr, scale, nterms, rg);
}


void launch_sep_band(int sweep, const double* tables, int NO, int L, int R, const double* ub, int ldub, int zpub,
                     double* ws, double* Y, const double* corr, double scale, int nterms, cudaStream_t st,
                     const int* lo, const int* hi) {
  zpub = zpub ? zpub : 64;
  const int nb = 1 << L;
  BandRegion rg;
  for (int a = 0; a < 3; ++a) {
    rg.lo[a] = lo ? lo[a] : 0;
    rg.hi[a] = hi ? hi[a] : nb;
  }
  if (sweep == 0) {
    launch_band_t<2, 0>(tables, NO, L, R, ub, ldub, zpub, ws, Y, corr, scale, nterms, st, rg);
  } else if (sweep == 1) {   // the fused y-x sweep (sweep 2 is a no-op)
    if (L == 4) launch_band_xy_t<16>(tables, NO, L, R, ub, ldub, zpub, ws, Y, corr, scale, nterms, st, rg);
    else if (L == 3) launch_band_xy_t<8>(tables, NO, L, R, ub, ldub, zpub, ws, Y, corr, scale, nterms, st, rg);
    else launch_band_xy_t<4>(tables, NO, L, R, ub, ldub, zpub, ws, Y, corr, scale, nterms, st, rg);
  }
}

cudaError_t sep_band_init() {
  const int smem = 200 * 1024;   // an upper bound (<= 227 KB minus static): occupancy follows each launch
  cudaError_t e = cudaFuncSetAttribute(sep_band_kernel<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(sep_band_xy_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(sep_band_xy_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(sep_band_xy_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  return e;
}

}  // namespace htlr
