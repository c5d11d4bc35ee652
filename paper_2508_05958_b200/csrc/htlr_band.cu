// Banded passes as register-resident line sweeps (sm_100a).
//
// At strong admissibility eta = 1 on a uniform grid the pairs a target box
// meets form product sets (htlr_sep.cu, "Banded leaf pass"), so a separable
// pass is
//   Y = C10^3 - C4^3 - C5^3 + C2^3 + E5^3 - E2^3   (+ self correction),
// X^3 = X_x (x) X_y (x) X_z, every X_S = sum_{o in S} M(o) shift(o) a 1-D
// block-banded operator over the boxes of one axis.  Each term is applied as
// three line sweeps, z first, then y, then x.  The reference's blocks
// (grids.py:268-296, blocks.py:126-259) are all applied, in a different order.
//
// The unit of work is a *line*: 8 points across x one axis of boxes long
// (NB boxes x 8 points x 8 points = 64 NB doubles, 2 NB registers per lane)
// in the m8n8k4 B-fragment layout, lane (g = lane/4, q = lane%4) holding
// points (k = q, n = g) and (k = q + 4, n = g) of every box, k running along
// the sweep axis.  A warp applies a term's band to its line entirely in
// registers: for target box b the sum over the band's source boxes s = b + o
// of A(o) B_s, 2 DMMA per (b, o), the box and offset loops unrolled so every
// register index is static (the band of box b depends only on b's parent
// b >> 1 and the term).  No source box is staged or re-read: each is loaded
// once by the one warp whose line holds it.
//
// band_line_kernel (z sweep): one warp per z line (box column (bx, by), point
// row y): reads the line of ub once and writes all NT terms' z-swept lines
// to the term buffers ([term][box][rhs][512], z-plane pitch 64).
//
// band_plane_kernel (y then x sweep): one CTA per z-point plane; per term,
// warp w loads the y line of box column bx = w from the term buffer (the
// next term's line is loaded while the current x sweep runs), sweeps y in
// registers and writes its C fragments to shared memory cell (by, bx) in
// lane order; after a barrier warp w reads box row by = w from shared memory
// as x-sweep B fragments (the y sweep's C fragment is the x sweep's B
// fragment with the k order permuted, the tables' mode-x A fragments use the
// same permutation) and adds its x sweep to the plane's accumulator in tensor
// memory.  The last term ends in Y = scale * acc + corr * ub (self pairs).
// 128 KB of shared memory (NB = 16): the transposition buffer, no staging.
//
// The first and the last sweep share work between the terms (bcount / boff):
// the six bands are unions of five pieces, so the z sweep runs 15 instead of
// 28 offsets per target box, and the x sweep applies each piece once to a
// running combination of the y-swept terms, 19 instead of 28.
#include "htlr_device.cuh"
#include "htlr_kernels.h"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace htlr {

namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// shared-memory load the compiler may not merge with an earlier one (the
// factor fragments of an offset recur in several terms; keeping them all live
// would cost 32+ registers)
__device__ __forceinline__ double lds(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

__device__ __forceinline__ double2 lds2(const double2* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

// Tensor memory as the plane kernel's Y accumulator (128 KB per plane, which
// the register file cannot hold next to the sweep lines): warp w owns 64
// columns of lane quarter w % 4; a double is two 32-bit columns.
__device__ __forceinline__ void tmem_ld16(uint32_t addr, double (&v)[4][2]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int j = 0; j < 2; ++j) v[c][j] = __hiloint2double((int)r[4 * c + 2 * j + 1], (int)r[4 * c + 2 * j]);
}
__device__ __forceinline__ void tmem_st16(uint32_t addr, const double (&v)[4][2]) {
  uint32_t r[16];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      r[4 * c + 2 * j] = (uint32_t)__double2loint(v[c][j]);
      r[4 * c + 2 * j + 1] = (uint32_t)__double2hiint(v[c][j]);
    }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
      ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ double neg(double v) {
  return __longlong_as_double(__double_as_longlong(v) ^ (long long)0x8000000000000000ull);
}

// band of term T (htlr_sep.cu band_count / band_off): count and the i-th
// per-axis offset for a target of coordinate parity c.  T = 0..5 are the six
// terms (C10, C4, C5, C2, E5, E2); 6..9 are pieces of them, which the first
// and the last sweep of a pass share between terms:
//   6: C{-1, 0, 1}   7: C{3 - 6c} (= C10 minus C4 minus C5)   8: E{-1, 0, 1}
//   9: C4 plus piece 7 (= C10 minus C5)
template <int T>
__host__ __device__ constexpr int bcount() {
  return T == 0 ? 10 : T == 1 ? 4 : (T == 3 || T == 5) ? 2 : (T == 6 || T == 8) ? 3 : T == 7 ? 1 : 5;
}
template <int T>
__host__ __device__ constexpr int boff(int c, int i) {
  return T == 0 ? -4 - c + i
       : T == 1 ? (i < 2 ? -4 - c + i : 2 - c + i)
       : (T == 3 || T == 5) ? (i ? 2 : -2)
       : (T == 6 || T == 8) ? i - 1
       : T == 7 ? 3 - 6 * c
       : T == 9 ? (c ? (i < 3 ? -5 + i : i) : (i < 2 ? -4 + i : 1 + i))
       : i - 2;
}
template <int T>
__host__ __device__ constexpr bool bneg() { return T == 1 || T == 2 || T == 5; }
// factor kind of a term or piece: 0 admissible (C), 1 near (E)
template <int T>
__host__ __device__ constexpr int bkind() { return (T == 4 || T == 5 || T == 8) ? 1 : 0; }

// spread the 4 low bits of v to every third bit (Morton interleave)
__host__ __device__ constexpr int spread3(int v) {
  return (v & 1) | ((v & 2) << 2) | ((v & 4) << 4) | ((v & 8) << 6) | ((v & 16) << 8);
}
// Morton id of box (x, y, z): x the most significant bit of each triple
// (htlr_device.cuh morton_encode with d = 3)
__device__ __forceinline__ int64_t morton3(int x, int y, int z) {
  return (int64_t)((spread3(x) << 2) | (spread3(y) << 1) | spread3(z));
}

// shared-memory copy of a pass's factor tables: per (kind, offset) slot the
// standard A fragments [0, 64) and the mode-x (permuted k) ones [64, 128)
constexpr int kTabSlot = 128;
// TMEM columns of a plane CTA: NB warps x 4 NB columns over 4 lane quarters
// (a power of two >= 32)
__host__ __device__ constexpr int plane_tmem_cols(int NB) { return NB == 16 ? 256 : NB == 8 ? 64 : 32; }
template <int NVAL>
__device__ __forceinline__ void stage_tables(double* __restrict__ dst, const double* __restrict__ tables, int NO) {
  for (int e = threadIdx.x; e < 2 * NO * NVAL; e += blockDim.x)
    dst[(e / NVAL) * kTabSlot + e % NVAL] = __ldg(tables + (e / NVAL) * kSepSlot + e % NVAL);
}

// One term's band over a register line: acc[b] (+)= sum_o A(o) in[b + o].
// SLOT 0: standard A fragments, 64: the mode-x (permuted k) ones.
template <int NB, int T, int SLOT, bool SIGN, int B0 = 0, int B1 = NB, bool CHK = false>
__device__ __forceinline__ void band_regs(const double* __restrict__ tab, int NO, int lane, const double (&in)[NB][2],
                                          double (&acc)[NB][2], int tlo = 0, int thi = NB) {
  constexpr int kind = bkind<T>();
  const int OR = (NO - 1) / 2;
#pragma unroll
  for (int i = 0; i < bcount<T>(); ++i) {
    const double* p0 = tab + (kind * NO + boff<T>(0, i) + OR) * kTabSlot + SLOT;
    const double* p1 = tab + (kind * NO + boff<T>(1, i) + OR) * kTabSlot + SLOT;
    double a00 = lds(p0 + lane), a01 = lds(p0 + 32 + lane);
    double a10 = lds(p1 + lane), a11 = lds(p1 + 32 + lane);
    if (SIGN && bneg<T>()) {
      a00 = neg(a00); a01 = neg(a01); a10 = neg(a10); a11 = neg(a11);
    }
#pragma unroll
    for (int b = B0; b < B1; ++b) {
      const int s = b + boff<T>(b & 1, i);
      if (s >= 0 && s < NB && (!CHK || (b >= tlo && b < thi))) dmma(acc[b][0], acc[b][1], (b & 1) ? a10 : a00, in[s][0]);
    }
#pragma unroll
    for (int b = B0; b < B1; ++b) {
      const int s = b + boff<T>(b & 1, i);
      if (s >= 0 && s < NB && (!CHK || (b >= tlo && b < thi))) dmma(acc[b][0], acc[b][1], (b & 1) ? a11 : a01, in[s][1]);
    }
  }
}

// The same band with the B fragments read from shared memory cells
// (cell s of the warp's row: a double2 per lane, lane order); unsigned (the
// cells carry the terms' signs).
template <int NB, int T, int B0, int B1>
__device__ __forceinline__ void band_smem(const double* __restrict__ tab, int NO, int lane,
                                          const double2* __restrict__ row, double (&acc)[NB][2]) {
  constexpr int kind = bkind<T>();
  const int OR = (NO - 1) / 2;
#pragma unroll
  for (int i = 0; i < bcount<T>(); ++i) {
    const double* p0 = tab + (kind * NO + boff<T>(0, i) + OR) * kTabSlot + 64;
    const double* p1 = tab + (kind * NO + boff<T>(1, i) + OR) * kTabSlot + 64;
    const double a00 = lds(p0 + lane), a01 = lds(p0 + 32 + lane);
    const double a10 = lds(p1 + lane), a11 = lds(p1 + 32 + lane);
#pragma unroll
    for (int b = B0; b < B1; ++b) {
      const int s = b + boff<T>(b & 1, i);
      if (s >= 0 && s < NB) {
        const double2 v = lds2(row + s * 32);
        dmma(acc[b][0], acc[b][1], (b & 1) ? a10 : a00, v.x);
        dmma(acc[b][0], acc[b][1], (b & 1) ? a11 : a01, v.y);
      }
    }
  }
}

template <int NB>
__device__ __forceinline__ void zero(double (&a)[NB][2]) {
#pragma unroll
  for (int b = 0; b < NB; ++b) a[b][0] = a[b][1] = 0.0;
}

// z sweep.  Work unit = half a z line: (box column (bx, by), point row y,
// rhs r, half h) -- the targets [H h, H h + H) (H = NB / 2) and the source
// boxes within 5 of them (13 of 16 at NB = 16).  One CTA per SM; warp gw
// takes units gw, gw + S, gw + 2S, ... (S = grid x warps, even, so a warp
// keeps its half): every SM sub-partition gets the same number of units to
// within one (a single warp with two accumulator chains already saturates
// its sub-partition's DMMA pipe, 1 DMMA.8x8x4 per 16 cycles, dependent
// latency 26 cycles: tools/dmma_latency.cu).
constexpr int kLineWarps = 12;
constexpr int kZWarps = 16;   // z sweep over whole halves (band_line_kernel KIND 0, 1)
template <int NB, int NT, bool R1, int HALF, bool FO = false, bool CHK = false>
__device__ __forceinline__ void line_units(const double* __restrict__ tab, int NO, int R, int ldub, int zpub,
                                           const double* __restrict__ ub, double* __restrict__ ws, int64_t tstride,
                                           int u0, int ustride, int nunits, int usel, int n, int zlo, int zhi,
                                           double2* __restrict__ spill) {
  constexpr int H = NB / 2;
  constexpr int S0 = HALF ? (H - 5 > 0 ? H - 5 : 0) : 0;         // loaded source boxes [S0, S1)
  constexpr int S1 = HALF ? NB : (H + 5 < NB ? H + 5 : NB);
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  // unit -> line: both halves active: u >> 1; one half: u
  auto line_of = [&](int u) { return usel ? u : (u >> 1); };
  auto load = [&](int u, double(&in)[NB][2]) {
    const int line = line_of(u);
    const int y = line & 7, col = (line >> 3) % (NB * NB), r = (line >> 3) / (NB * NB);
    if (FO) {
      // straight from the F-order grid vector: box (bx, by, b), point
      // (x = g, y, z = q (+4)) at (8 bx + g) + n (8 by + y) + n^2 (8 b + q)
      const int64_t n2 = (int64_t)n * n;
      const double* s = ub + ((int64_t)(8 * (col % NB) + g) + (int64_t)n * (8 * (col / NB) + y) + n2 * q) * R + r;
#pragma unroll
      for (int b = S0; b < S1; ++b) {
        in[b][0] = __ldg(s + 8 * b * n2 * R);
        in[b][1] = __ldg(s + (8 * b + 4) * n2 * R);
      }
      return;
    }
    const double* s = ub + (morton3(col % NB, col / NB, 0) * R + r) * ldub + 8 * y + g + zpub * q;
#pragma unroll
    for (int b = S0; b < S1; ++b) {
      const double* sb = s + spread3(b) * (int64_t)R * ldub;
      in[b][0] = __ldg(sb);
      in[b][1] = __ldg(sb + 4 * zpub);
    }
  };
  auto compute = [&](int u, const double(&in)[NB][2]) {
    const int line = line_of(u);
    const int y = line & 7, col = (line >> 3) % (NB * NB), r = (line >> 3) / (NB * NB);
    // lane's C fragment: (z' = g, x = 2q + j) of every target box
    double* const ob = ws + (morton3(col % NB, col / NB, 0) * R + r) * 512 + 64 * g + 8 * y + 2 * q;
    // The six terms' bands are unions of five pieces (B = C{-2, 2}, M =
    // C{-1, 0, 1}, P = C{3 - 6c}, A = C4; EB = E{-2, 2}, EM = E{-1, 0, 1}):
    //   C2 = B, C5 = B + M, C10 = B + M + P + A, C4 = A, E2 = EB, E5 = EB + EM,
    // so one accumulator chain per kind gives every term with 15 instead of 28
    // offsets per target box; B + M + P waits in shared memory while A runs.
    double acc[NB][2];
    auto band = [&](auto tc) {
      band_regs<NB, decltype(tc)::value, 0, false, HALF * H, HALF * H + H, CHK>(tab, NO, lane, in, acc, zlo, zhi);
    };
    auto put = [&](int T) {
      double* o = ob + T * tstride;
#pragma unroll
      for (int b = HALF * H; b < HALF * H + H; ++b)
        if (!CHK || (b >= zlo && b < zhi))
          *reinterpret_cast<double2*>(o + spread3(b) * (int64_t)R * 512) = make_double2(acc[b][0], acc[b][1]);
    };
    // a runtime loop over the phases: the compiler cannot interleave (and keep
    // live) several accumulator chains
#pragma unroll 1
    for (int ph = 0; ph < NT; ++ph) {
      switch (ph) {
        case 0:
          zero(acc);
          band(std::integral_constant<int, 3>{});
          put(3);
          break;
        case 1:
          band(std::integral_constant<int, 6>{});
          put(2);
          break;
        case 2:
          band(std::integral_constant<int, 7>{});
#pragma unroll
          for (int b = 0; b < H; ++b) spill[b * 32] = make_double2(acc[HALF * H + b][0], acc[HALF * H + b][1]);
          break;
        case 3:
          zero(acc);
          band(std::integral_constant<int, 1>{});
          put(1);
#pragma unroll
          for (int b = 0; b < H; ++b) {
            const double2 v = spill[b * 32];
            acc[HALF * H + b][0] += v.x;
            acc[HALF * H + b][1] += v.y;
          }
          put(0);
          break;
        case 4:
          zero(acc);
          band(std::integral_constant<int, 5>{});
          put(5);
          break;
        default:
          band(std::integral_constant<int, 8>{});
          put(4);
          break;
      }
    }
  };
  // one register buffer per warp: the other warps of the sub-partition cover
  // a unit's loads (a second buffer with 12 warps, or 8 and 20 warps, measured
  // the same: the sweep is bound by its 117 MB of loads and stores, 19.5 us
  // without the DMMAs, next to 14 us of DMMA issue)
  double a[NB][2];
  __syncthreads();   // the tables (staged by the caller) are in place
  for (int u = u0; u < nunits; u += ustride) {
    load(u, a);
    compute(u, a);
  }
}

// Pair units (z-slab shards narrower than half a line): unit = (line, own
// sibling pair p): targets 2p, 2p + 1 and the 12 source boxes 2p - 5 ...
// 2p + 6, indexed relative to the pair so every register index is static
// (boxes outside the level are loaded as zeros and contribute nothing).
// Restricting a half-line unit's targets by a runtime test would not save
// the work: predicated-off DMMAs still occupy the tensor pipe.
template <int NB, int T>
__device__ __forceinline__ void band_pair(const double* __restrict__ tab, int NO, int lane, const double (&in)[12][2],
                                          double (&acc)[2][2]) {
  constexpr int kind = bkind<T>();
  const int OR = (NO - 1) / 2;
#pragma unroll
  for (int i = 0; i < bcount<T>(); ++i) {
    constexpr int dummy = 0;
    (void)dummy;
    const double* p0 = tab + (kind * NO + boff<T>(0, i) + OR) * kTabSlot;
    const double* p1 = tab + (kind * NO + boff<T>(1, i) + OR) * kTabSlot;
    const double a00 = lds(p0 + lane), a01 = lds(p0 + 32 + lane);
    const double a10 = lds(p1 + lane), a11 = lds(p1 + 32 + lane);
    const int s0 = boff<T>(0, i) + 5, s1 = boff<T>(1, i) + 6;   // relative source boxes of 2p, 2p + 1
    dmma(acc[0][0], acc[0][1], a00, in[s0][0]);
    dmma(acc[1][0], acc[1][1], a10, in[s1][0]);
    dmma(acc[0][0], acc[0][1], a01, in[s0][1]);
    dmma(acc[1][0], acc[1][1], a11, in[s1][1]);
  }
}

template <int NB, int NT, bool R1>
__device__ __forceinline__ void pair_units(const double* __restrict__ tab, int NO, int R, int ldub, int zpub,
                                           const double* __restrict__ ub, double* __restrict__ ws, int64_t tstride,
                                           int u0, int ustride, int n, int zlo, int zhi) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int npairs = (zhi - zlo) >> 1;
  const int nunits = NB * NB * 8 * R * npairs;
  auto load = [&](int u, double(&in)[12][2]) {
    const int line = u / npairs, p = (zlo >> 1) + u % npairs;
    const int y = line & 7, col = (line >> 3) % (NB * NB), r = (line >> 3) / (NB * NB);
    const int64_t n2 = (int64_t)n * n;
    const double* sf = ub + ((int64_t)(8 * (col % NB) + g) + (int64_t)n * (8 * (col / NB) + y) + n2 * q) * R + r;
    const double* sb = ub + (morton3(col % NB, col / NB, 0) * R + r) * ldub + 8 * y + g + zpub * q;
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const int b = 2 * p - 5 + i;
      if (b < 0 || b >= NB) {
        in[i][0] = in[i][1] = 0.0;
      } else if (n) {
        in[i][0] = __ldg(sf + 8 * b * n2 * R);
        in[i][1] = __ldg(sf + (8 * b + 4) * n2 * R);
      } else {
        const double* s = sb + spread3(b) * (int64_t)R * ldub;
        in[i][0] = __ldg(s);
        in[i][1] = __ldg(s + 4 * zpub);
      }
    }
  };
  auto compute = [&](int u, const double(&in)[12][2]) {
    const int line = u / npairs, p = (zlo >> 1) + u % npairs;
    const int y = line & 7, col = (line >> 3) % (NB * NB), r = (line >> 3) / (NB * NB);
    // boxes 2p, 2p + 1: Morton ids m(bx, by, 0) + spread3(2p) (+ 1)
    double* const ob = ws + ((morton3(col % NB, col / NB, 0) + spread3(2 * p)) * R + r) * 512 + 64 * g + 8 * y + 2 * q;
    auto term = [&](auto tc) {
      constexpr int T = decltype(tc)::value;
      double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      band_pair<NB, T>(tab, NO, lane, in, acc);
      double* o = ob + T * tstride;
      *reinterpret_cast<double2*>(o) = make_double2(acc[0][0], acc[0][1]);
      *reinterpret_cast<double2*>(o + (int64_t)R * 512) = make_double2(acc[1][0], acc[1][1]);
    };
#pragma unroll 1
    for (int t = 0; t < NT; ++t) {
      switch (t) {
        case 0: term(std::integral_constant<int, 0>{}); break;
        case 1: term(std::integral_constant<int, 1>{}); break;
        case 2: term(std::integral_constant<int, 2>{}); break;
        case 3: term(std::integral_constant<int, 3>{}); break;
        case 4: term(std::integral_constant<int, 4>{}); break;
        default: term(std::integral_constant<int, 5>{}); break;
      }
    }
  };
  double a[12][2], b[12][2];
  int u = u0;
  if (u < nunits) load(u, a);
  __syncthreads();
  while (u < nunits) {
    const int un = u + ustride;
    if (un < nunits) load(un, b);
    compute(u, a);
    if (un >= nunits) break;
    const int unn = un + ustride;
    if (unn < nunits) load(unn, a);
    compute(un, b);
    u = unn;
  }
}

// half-line units over the target z range [zlo, zhi), which covers whole
// halves: both (the parity of the even-strided unit picks the half) or one
template <int NB, int NT, bool R1, bool FO>
__device__ __forceinline__ void dispatch_halves(const double* __restrict__ tab, int NO, int R, int ldub, int zpub,
                                                const double* __restrict__ ub, double* __restrict__ ws,
                                                int64_t tstride, int gw, int ustride, int nlines, int n, int zlo,
                                                int zhi, double2* __restrict__ spill) {
  const bool h0 = zlo < NB / 2, h1 = zhi > NB / 2;
  if (h0 && h1) {
    if (gw & 1)
      line_units<NB, NT, R1, 1, FO>(tab, NO, R, ldub, zpub, ub, ws, tstride, gw, ustride, 2 * nlines, 0, n, zlo, zhi, spill);
    else
      line_units<NB, NT, R1, 0, FO>(tab, NO, R, ldub, zpub, ub, ws, tstride, gw, ustride, 2 * nlines, 0, n, zlo, zhi, spill);
  } else if (h1) {
    line_units<NB, NT, R1, 1, FO>(tab, NO, R, ldub, zpub, ub, ws, tstride, gw, ustride, nlines, 1, n, zlo, zhi, spill);
  } else {
    line_units<NB, NT, R1, 0, FO>(tab, NO, R, ldub, zpub, ub, ws, tstride, gw, ustride, nlines, 1, n, zlo, zhi, spill);
  }
}

// src: the level's boxes [box][rhs][ldub] (z pitch zpub), or with n > 0 the
// F-order grid vector u[N][R] of an n^3 grid (the leaf pass reads u itself:
// no permuted copy).  Targets are written for z boxes [zlo, zhi) only (a
// z-slab shard); halves without an own box are skipped.
// KIND 0: the level's boxes, whole halves; 1: the F-order u, whole halves;
// 2: sibling pairs of a narrow z slab.  Separate kernels keep the unsharded
// kernel's code what it was (one kernel with all three bodies measured 33 ->
// 37 us for config 4's z sweep).
template <int NB, int NT, bool R1, int KIND, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) band_line_kernel(const double* __restrict__ tables, int NO,
                                                                      int R_, const double* __restrict__ ub, int ldub,
                                                                      int zpub, double* __restrict__ ws,
                                                                      int64_t tstride, int n, int zlo, int zhi) {
  const int R = R1 ? 1 : R_;   // one rhs: every box offset a compile-time constant
  __shared__ double tab[2 * 15 * kTabSlot];
  extern __shared__ __align__(16) double2 spill_sm[];   // [warp][target box of the half][lane]
  stage_tables<64>(tab, tables, NO);   // the units sync after issuing their first loads
  const int gw = blockIdx.x + gridDim.x * (threadIdx.x >> 5);
  const int ustride = gridDim.x * (blockDim.x >> 5);
  const int nlines = NB * NB * 8 * R;
  if (KIND == 2)
    pair_units<NB, NT, R1>(tab, NO, R, ldub, zpub, ub, ws, tstride, gw, ustride, n, zlo & ~1, (zhi + 1) & ~1);
  else
    dispatch_halves<NB, NT, R1, KIND == 1>(tab, NO, R, ldub, zpub, ub, ws, tstride, gw, ustride, nlines, n, zlo, zhi,
                                           spill_sm + (threadIdx.x >> 5) * (NB / 2) * 32 + (threadIdx.x & 31));
}

// y and x sweeps of one z-point plane (blockIdx.x = 8 bz + zl), warps = NB
template <int NB, int NT, bool R1, bool FRED>
__global__ void __launch_bounds__(NB * 32, 1) band_plane_kernel(const double* __restrict__ tables, int NO, int R_,
                                                                const double* __restrict__ ub, int ldub, int zpub,
                                                                const double* __restrict__ ws, int64_t tstride,
                                                                double* __restrict__ Y,
                                                                const double* __restrict__ corr_ptr, double scale,
                                                                int n, int zlo, double* __restrict__ fred, int nf) {
  constexpr int NQ = NB / 4;   // quarters of a row of cells (4 cells = 16 TMEM columns)
  const int R = R1 ? 1 : R_;
  extern __shared__ __align__(16) double smp[];
  double2* cell = reinterpret_cast<double2*>(smp);   // [by][bx][lane]
  double* tab = smp + NB * NB * 64;
  __shared__ uint32_t tmem_sh;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tmem_sh)),
                 "n"(plane_tmem_cols(NB)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  stage_tables<128>(tab, tables, NO);
  const int zl = blockIdx.x & 7, bz = zlo + (blockIdx.x >> 3), r = blockIdx.y;
  const int g = lane >> 2, q = lane & 3;
  // y line of box column bx = w: element (y = q (+4), x = g) of z plane zl;
  // box (w, b, bz) has Morton id morton3(w, 0, bz) + 2 spread3(b)
  const int64_t yb = (morton3(w, 0, bz) * R + r) * 512 + 64 * zl + 8 * q + g, ystride = (int64_t)R * 512 * 2;
  double in[NB][2];
  auto load = [&](int t) {
    const double* s = ws + t * tstride + yb;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      in[b][0] = __ldg(s + spread3(b) * ystride);
      in[b][1] = __ldg(s + spread3(b) * ystride + 32);
    }
  };
  const double2* row = cell + w * NB * 32 + lane;
  double2* mine = cell + w * 32 + lane;   // column bx = w, row b at + b * NB * 32
  load(0);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tm = tmem_sh + ((uint32_t)(32 * (w & 3)) << 16) + 16 * NQ * (w >> 2);
  // The x sweeps share pieces between the terms (bcount / boff): with the
  // cells S running through  V10, V10 - V5, V10 - V5 + V2, -V4, W5, W5 - W2
  // (V_t, W_t the y-swept terms; the y sweep carries the term's sign and adds
  // to the cells it wrote in the phase before),
  //   Y = (C4 + P)_x V10 + M_x (V10 - V5) + B_x (V10 - V5 + V2) + C4_x (-V4)
  //       + EM_x W5 + EB_x (W5 - W2)
  // -- 19 instead of 28 offsets per target cell.
  // phase: term T's y sweep (ADD: onto the cells), then x piece XT of the
  // cells; TN = the next phase's term, whose lines load during the x sweep
  auto term = [&](auto tc, auto xc, auto addc, auto firstc, int TN) {
    constexpr int T = decltype(tc)::value, XT = decltype(xc)::value;
    constexpr bool ADD = decltype(addc)::value, FIRST = decltype(firstc)::value;
    constexpr int H = NB / 2;
    {
      double acc[NB][2];
      if (ADD) {
#pragma unroll
        for (int b = 0; b < H; ++b) {
          const double2 v = mine[b * NB * 32];
          acc[b][0] = v.x, acc[b][1] = v.y;
        }
      } else {
        zero(acc);
      }
      band_regs<NB, T, 0, true, 0, H>(tab, NO, lane, in, acc);
#pragma unroll
      for (int b = 0; b < H; ++b) mine[b * NB * 32] = make_double2(acc[b][0], acc[b][1]);
      if (ADD) {
#pragma unroll
        for (int b = H; b < NB; ++b) {
          const double2 v = mine[b * NB * 32];
          acc[b][0] = v.x, acc[b][1] = v.y;
        }
      }
      band_regs<NB, T, 0, true, H, NB>(tab, NO, lane, in, acc);
#pragma unroll
      for (int b = H; b < NB; ++b) mine[b * NB * 32] = make_double2(acc[b][0], acc[b][1]);
    }
    __syncthreads();
    if (TN >= 0) load(TN);   // in flight during the x sweep
    // x sweep of the warp's row, four cells at a time, added to the TMEM accumulator
    auto quarter = [&](auto qc) {
      constexpr int Q = decltype(qc)::value;
      double acc[NB][2];
      zero(acc);
      band_smem<NB, XT, 4 * Q, 4 * Q + 4>(tab, NO, lane, row, acc);
      double v[4][2];
      if (!FIRST) {
        tmem_ld16(tm + 16 * Q, v);
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c][0] += acc[4 * Q + c][0], v[c][1] += acc[4 * Q + c][1];
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c][0] = acc[4 * Q + c][0], v[c][1] = acc[4 * Q + c][1];
      }
      tmem_st16(tm + 16 * Q, v);
    };
    quarter(std::integral_constant<int, 0>{});
    if (NQ > 1) quarter(std::integral_constant<int, (NQ > 1 ? 1 : 0)>{});
    if (NQ > 2) quarter(std::integral_constant<int, (NQ > 2 ? 2 : 0)>{});
    if (NQ > 3) quarter(std::integral_constant<int, (NQ > 3 ? 3 : 0)>{});
    __syncthreads();
  };
  using TT = std::true_type;
  using FF = std::false_type;
#pragma unroll 1
  for (int ph = 0; ph < NT; ++ph) {
    switch (ph) {
      case 0: term(std::integral_constant<int, 0>{}, std::integral_constant<int, 9>{}, FF{}, TT{}, 2); break;
      case 1: term(std::integral_constant<int, 2>{}, std::integral_constant<int, 6>{}, TT{}, FF{}, 3); break;
      case 2: term(std::integral_constant<int, 3>{}, std::integral_constant<int, 3>{}, TT{}, FF{}, 1); break;
      case 3: term(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{}, FF{}, FF{}, NT > 4 ? 4 : -1); break;
      case 4: term(std::integral_constant<int, 4>{}, std::integral_constant<int, 8>{}, FF{}, FF{}, 5); break;
      default: term(std::integral_constant<int, 5>{}, std::integral_constant<int, 5>{}, TT{}, FF{}, -1); break;
    }
  }
  // lane holds (x' = g, y = 2q + j) of cells (bx = b, by = w)
  const double cv = corr_ptr ? corr_ptr[0] : 0.0;
  const int64_t mw = morton3(0, w, bz) * R + r;
#pragma unroll
  for (int Q = 0; Q < NQ; ++Q) {
    double v[4][2];
    tmem_ld16(tm + 16 * Q, v);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t m = mw + (int64_t)(spread3(4 * Q + c) << 2) * R;
      double* o = Y + m * 512 + 64 * zl + 16 * q + g;
      // the self pair's point: box (4Q + c, w, bz), element (x = g, y = 2q + j, zl)
      const double* us = n ? ub + ((int64_t)(8 * (4 * Q + c) + g) + (int64_t)n * (8 * w + 2 * q) +
                                   (int64_t)n * n * (8 * bz + zl)) * R + r
                           : ub + m * ldub + zpub * zl + 16 * q + g;
      const int64_t ustep = n ? (int64_t)n * R : 8;
      // FRED: the plane's share of f summed straight into the F-order result
      // (the downward pass adds its own with REDs too: no Y round trip and no
      // order between the two); a separate instantiation, so the kernel that
      // stores Y keeps its register allocation
      if constexpr (FRED) {
        double* of = fred + ((int64_t)(8 * (4 * Q + c) + g) + (int64_t)nf * (8 * w + 2 * q) +
                             (int64_t)nf * nf * (8 * bz + zl)) * R + r;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          double val = scale * v[c][j];
          if (corr_ptr) val = fma(cv, __ldg(us + j * ustep), val);
          atomicAdd(of + (int64_t)j * nf * R, val);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          double val = scale * v[c][j];
          if (corr_ptr) val = fma(cv, __ldg(us + j * ustep), val);
          o[8 * j] = val;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_sh), "n"(plane_tmem_cols(NB)));
}

// The y and x sweeps as line kernels (the plane kernel's alternative for
// z-slab shards, whose few planes would occupy few SMs): every unit is a half
// line of one z-point plane, so a slab's sweeps spread over all SMs, and the
// slab's term buffers (1/world of the level's) stay in L2 between them.
//
// band_yline_kernel: unit = (term t, box column bx, z box bz, z point zl,
// half): the y line of z-swept term t (ws, [term][box][rhs][512], element
// 64 zl + 8 y + x) -> y-swept cells in the x sweep's B-fragment order (ws2,
// [term][box][rhs][zl][lane][2]).
template <int NB, int NT, bool R1, int HALF>
__device__ __forceinline__ void yline_units(const double* __restrict__ tab, int NO, int R, const double* __restrict__ ws,
                                            double* __restrict__ ws2, int64_t tstride, int u0, int ustride,
                                            int nunits, int zlo, int nz) {
  constexpr int H = NB / 2;
  constexpr int S0 = HALF ? (H - 5 > 0 ? H - 5 : 0) : 0;
  constexpr int S1 = HALF ? NB : (H + 5 < NB ? H + 5 : NB);
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  // unit u: half = u & 1 (the warp's), then bx, zl, bz, r, t (slowest)
  struct Line {
    int t, bx, bz, zl, r;
  };
  auto decode = [&](int u) {
    int v = u >> 1;
    Line l;
    l.bx = v % NB;
    v /= NB;
    l.zl = v & 7;
    v >>= 3;
    l.bz = zlo + v % nz;
    v /= nz;
    l.r = v % R;
    l.t = v / R;
    return l;
  };
  auto base = [&](const Line& l) {   // box (bx, by = 0, bz): Morton id + 2 spread3(by) per by
    return (morton3(l.bx, 0, l.bz) * R + l.r) * 512;
  };
  auto load = [&](int u, double(&in)[NB][2]) {
    const Line l = decode(u);
    const double* s = ws + l.t * tstride + base(l) + 64 * l.zl + 8 * q + g;
#pragma unroll
    for (int b = S0; b < S1; ++b) {
      const double* sb = s + (int64_t)(2 * spread3(b)) * R * 512;
      in[b][0] = __ldg(sb);
      in[b][1] = __ldg(sb + 32);
    }
  };
  auto compute = [&](int u, const double(&in)[NB][2]) {
    const Line l = decode(u);
    double* o = ws2 + l.t * tstride + base(l) + 64 * l.zl + 2 * lane;
    auto term = [&](auto tc) {
      constexpr int T = decltype(tc)::value;
      double acc[NB][2];
      zero(acc);
      band_regs<NB, T, 0, false, HALF * H, HALF * H + H>(tab, NO, lane, in, acc);
#pragma unroll
      for (int b = HALF * H; b < HALF * H + H; ++b)
        *reinterpret_cast<double2*>(o + (int64_t)(2 * spread3(b)) * R * 512) = make_double2(acc[b][0], acc[b][1]);
    };
    switch (l.t) {
      case 0: term(std::integral_constant<int, 0>{}); break;
      case 1: term(std::integral_constant<int, 1>{}); break;
      case 2: term(std::integral_constant<int, 2>{}); break;
      case 3: term(std::integral_constant<int, 3>{}); break;
      case 4: if (NT > 4) term(std::integral_constant<int, 4>{}); break;
      default: if (NT > 4) term(std::integral_constant<int, 5>{}); break;
    }
  };
  double a[NB][2], b[NB][2];
  int u = u0;
  if (u < nunits) load(u, a);
  __syncthreads();
  while (u < nunits) {
    const int un = u + ustride;
    if (un < nunits) load(un, b);
    compute(u, a);
    if (un >= nunits) break;
    const int unn = un + ustride;
    if (unn < nunits) load(unn, a);
    compute(un, b);
    u = unn;
  }
}

template <int NB, int NT, bool R1>
__global__ void __launch_bounds__(kLineWarps * 32, 1) band_yline_kernel(const double* __restrict__ tables, int NO,
                                                                       int R_, const double* __restrict__ ws,
                                                                       double* __restrict__ ws2, int64_t tstride,
                                                                       int zlo, int nz) {
  const int R = R1 ? 1 : R_;
  __shared__ double tab[2 * 15 * kTabSlot];
  stage_tables<64>(tab, tables, NO);
  const int gw = blockIdx.x + gridDim.x * (threadIdx.x >> 5);
  const int ustride = gridDim.x * (blockDim.x >> 5);
  const int nunits = 2 * NT * R * nz * 8 * NB;
  if (gw & 1)
    yline_units<NB, NT, R1, 1>(tab, NO, R, ws, ws2, tstride, gw, ustride, nunits, zlo, nz);
  else
    yline_units<NB, NT, R1, 0>(tab, NO, R, ws, ws2, tstride, gw, ustride, nunits, zlo, nz);
}

// band_xline_kernel: unit = (box row by, z box bz, z point zl, half): the x
// line of every term's y-swept cells (ws2), the term's sign folded into the
// mode-x A fragments, summed in registers (the next term's line loads while
// the current one computes); Y = scale * sum + corr * u (self pairs).
template <int NB, int NT, bool R1, int HALF>
__device__ __forceinline__ void xline_units(const double* __restrict__ tab, int NO, int R, const double* __restrict__ ws2,
                                            int64_t tstride, double* __restrict__ Y, const double* __restrict__ src,
                                            int ldub, int zpub, int n, const double* __restrict__ corr_ptr,
                                            double scale, int u0, int ustride, int nunits, int zlo, int nz) {
  constexpr int H = NB / 2;
  constexpr int S0 = HALF ? (H - 5 > 0 ? H - 5 : 0) : 0;
  constexpr int S1 = HALF ? NB : (H + 5 < NB ? H + 5 : NB);
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const double cv = corr_ptr ? corr_ptr[0] : 0.0;
  for (int u = u0; u < nunits; u += ustride) {
    int v = u >> 1;
    const int by = v % NB;
    v /= NB;
    const int zl = v & 7;
    v >>= 3;
    const int bz = zlo + v % nz, r = v / nz;
    // cell (bx, by, bz): Morton id morton3(0, by, bz) + 4 spread3(bx)
    const int64_t m0 = morton3(0, by, bz) * R + r;
    const double* s = ws2 + m0 * 512 + 64 * zl + 2 * lane;
    double bufa[NB][2], bufb[NB][2], acc[NB][2];
    zero(acc);
    auto load = [&](int t, double(&in)[NB][2]) {
      const double* st = s + t * tstride;
#pragma unroll
      for (int b = S0; b < S1; ++b) {
        const double2 w2 = __ldg(reinterpret_cast<const double2*>(st + (int64_t)(4 * spread3(b)) * R * 512));
        in[b][0] = w2.x;
        in[b][1] = w2.y;
      }
    };
    // the x pieces shared between the terms (band_plane_kernel): the line S
    // runs through V10, V10 - V5, V10 - V5 + V2, then V4 (negated band), W5,
    // W5 - W2 -- 19 instead of 28 offsets per target cell
    auto axpy = [&](double sgn, double(&s_)[NB][2], const double(&t_)[NB][2]) {
#pragma unroll
      for (int b = S0; b < S1; ++b) s_[b][0] = fma(sgn, t_[b][0], s_[b][0]), s_[b][1] = fma(sgn, t_[b][1], s_[b][1]);
    };
    load(0, bufa);
    load(2, bufb);
    band_regs<NB, 9, 64, false, HALF * H, HALF * H + H>(tab, NO, lane, bufa, acc);
    axpy(-1.0, bufa, bufb);
    load(3, bufb);
    band_regs<NB, 6, 64, false, HALF * H, HALF * H + H>(tab, NO, lane, bufa, acc);
    axpy(1.0, bufa, bufb);
    load(1, bufb);
    band_regs<NB, 3, 64, false, HALF * H, HALF * H + H>(tab, NO, lane, bufa, acc);
    if (NT > 4) load(4, bufa);
    band_regs<NB, 1, 64, true, HALF * H, HALF * H + H>(tab, NO, lane, bufb, acc);
    if (NT > 4) {
      load(5, bufb);
      band_regs<NB, 8, 64, false, HALF * H, HALF * H + H>(tab, NO, lane, bufa, acc);
      axpy(-1.0, bufa, bufb);
      band_regs<NB, 5, 64, false, HALF * H, HALF * H + H>(tab, NO, lane, bufa, acc);
    }
    // lane holds (x' = g, y = 2q + j) of target cells bx in the half
#pragma unroll
    for (int bx = HALF * H; bx < HALF * H + H; ++bx) {
      const int64_t m = m0 + (int64_t)(4 * spread3(bx)) * R;
      double* o = Y + m * 512 + 64 * zl + 16 * q + g;
      const double* us = n ? src + ((int64_t)(8 * bx + g) + (int64_t)n * (8 * by + 2 * q) +
                                    (int64_t)n * n * (8 * bz + zl)) * R + r
                           : src + m * ldub + zpub * zl + 16 * q + g;
      const int64_t ustep = n ? (int64_t)n * R : 8;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double val = scale * acc[bx][j];
        if (corr_ptr) val = fma(cv, __ldg(us + j * ustep), val);
        o[8 * j] = val;
      }
    }
  }
}

template <int NB, int NT, bool R1>
__global__ void __launch_bounds__(kLineWarps * 32, 1) band_xline_kernel(const double* __restrict__ tables, int NO,
                                                                       int R_, const double* __restrict__ ws2,
                                                                       int64_t tstride, double* __restrict__ Y,
                                                                       const double* __restrict__ src, int ldub,
                                                                       int zpub, int n,
                                                                       const double* __restrict__ corr_ptr,
                                                                       double scale, int zlo, int nz) {
  const int R = R1 ? 1 : R_;
  __shared__ double tab[2 * 15 * kTabSlot];
  stage_tables<128>(tab, tables, NO);
  __syncthreads();
  const int gw = blockIdx.x + gridDim.x * (threadIdx.x >> 5);
  const int ustride = gridDim.x * (blockDim.x >> 5);
  const int nunits = 2 * R * nz * 8 * NB;
  if (gw & 1)
    xline_units<NB, NT, R1, 1>(tab, NO, R, ws2, tstride, Y, src, ldub, zpub, n, corr_ptr, scale, gw, ustride, nunits,
                               zlo, nz);
  else
    xline_units<NB, NT, R1, 0>(tab, NO, R, ws2, tstride, Y, src, ldub, zpub, n, corr_ptr, scale, gw, ustride, nunits,
                               zlo, nz);
}

template <int NB, int NT>
void launch_ylines_t(const double* tab, int NO, int R, const double* ws, double* ws2, double* Y, const double* src,
                     int ldub, int zpub, int n, const double* corr, double scale, cudaStream_t st, int zlo, int zhi) {
  const int64_t tstride = (int64_t)NB * NB * NB * R * 512;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nz = zhi - zlo;
  const int64_t yunits = 2LL * NT * R * nz * 8 * NB;
  const int gy = (int)std::min<int64_t>(sms, std::max<int64_t>(1, yunits / (2 * kLineWarps)));
  if (R == 1) {
    band_yline_kernel<NB, NT, true><<<gy, kLineWarps * 32, 0, st>>>(tab, NO, R, ws, ws2, tstride, zlo, nz);
    band_xline_kernel<NB, NT, true><<<sms, kLineWarps * 32, 0, st>>>(tab, NO, R, ws2, tstride, Y, src, ldub, zpub, n,
                                                                     corr, scale, zlo, nz);
  } else {
    band_yline_kernel<NB, NT, false><<<gy, kLineWarps * 32, 0, st>>>(tab, NO, R, ws, ws2, tstride, zlo, nz);
    band_xline_kernel<NB, NT, false><<<sms, kLineWarps * 32, 0, st>>>(tab, NO, R, ws2, tstride, Y, src, ldub, zpub,
                                                                      n, corr, scale, zlo, nz);
  }
}

template <int NB, int NT>
void launch_lines_t(const double* tab, int NO, int R, const double* ub, int ldub, int zpub, double* ws,
                    cudaStream_t st, int n, int zlo, int zhi, int max_ctas) {
  const int64_t lines = (int64_t)NB * NB * 8 * R;
  const int64_t tstride = (int64_t)NB * NB * NB * R * 512;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one CTA of kLineWarps warps per SM (the stride over the 2 x lines
  // half-line units must be even: a warp keeps its half)
  if (max_ctas > 0) sms = std::min(sms, max_ctas);
  const bool halves = (zlo == 0 || zlo == NB / 2) && (zhi == NB || zhi == NB / 2);
  const int kind = !halves ? 2 : n ? 1 : 0;
  auto go = [&](auto r1, auto kc) {
    constexpr bool r1v = decltype(r1)::value;
    constexpr int kv = decltype(kc)::value;
    // whole-half units: kZWarps warps with one register buffer each, one
    // accumulator (NB / 2 boxes) per warp parked in shared memory; pair units:
    // kLineWarps warps, two register buffers
    constexpr int warps = kv == 2 ? kLineWarps : kZWarps;
    const size_t smem = kv == 2 ? (size_t)0 : (size_t)warps * (NB / 2) * 32 * sizeof(double2);
    auto kern = band_line_kernel<NB, NT, r1v, kv, warps>;
    const int64_t grid = std::min<int64_t>(sms, std::max<int64_t>(1, lines / 4));
    if (smem > 16 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<(unsigned)grid, warps * 32, smem, st>>>(tab, NO, R, ub, ldub, zpub, ws, tstride, n, zlo, zhi);
  };
  using T1 = std::true_type;
  using F1 = std::false_type;
  using K0 = std::integral_constant<int, 0>;
  using K1 = std::integral_constant<int, 1>;
  using K2 = std::integral_constant<int, 2>;
  if (R == 1) kind == 0 ? go(T1{}, K0{}) : kind == 1 ? go(T1{}, K1{}) : go(T1{}, K2{});
  else kind == 0 ? go(F1{}, K0{}) : kind == 1 ? go(F1{}, K1{}) : go(F1{}, K2{});
}

template <int NB, int NT>
void launch_planes_t(const double* tab, int NO, int R, const double* ub, int ldub, int zpub, const double* ws,
                     double* Y, const double* corr, double scale, cudaStream_t st, int n, int zlo, int zhi,
                     double* fred, int nf) {
  if (zhi <= zlo) return;
  const int64_t tstride = (int64_t)NB * NB * NB * R * 512;
  const size_t smem = (size_t)NB * NB * 32 * sizeof(double2) + (size_t)2 * NO * kTabSlot * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(band_plane_kernel<NB, NT, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(band_plane_kernel<NB, NT, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(band_plane_kernel<NB, NT, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(band_plane_kernel<NB, NT, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const dim3 grid(8 * (zhi - zlo), R);
  auto go = [&](auto kern) {
    kern<<<grid, NB * 32, smem, st>>>(tab, NO, R, ub, ldub, zpub, ws, tstride, Y, corr, scale, n, zlo, fred, nf);
  };
  if (fred) R == 1 ? go(band_plane_kernel<NB, NT, true, true>) : go(band_plane_kernel<NB, NT, false, true>);
  else R == 1 ? go(band_plane_kernel<NB, NT, true, false>) : go(band_plane_kernel<NB, NT, false, false>);
}

}  // namespace

bool band_lines_supported(int L) { return L >= 2 && L <= 4; }

void launch_band_lines(int L, int nterms, const double* tab, int NO, int R, const double* ub, int ldub, int zpub,
                       double* ws, cudaStream_t st, int n, int zlo, int zhi, int max_ctas) {
  zpub = zpub ? zpub : 64;
  const int nb = 1 << L;
  zhi = std::min(zhi, nb);
  if (zhi <= zlo) return;
  if (L == 4) nterms == 6 ? launch_lines_t<16, 6>(tab, NO, R, ub, ldub, zpub, ws, st, n, zlo, zhi, max_ctas)
                          : launch_lines_t<16, 4>(tab, NO, R, ub, ldub, zpub, ws, st, n, zlo, zhi, max_ctas);
  else if (L == 3) nterms == 6 ? launch_lines_t<8, 6>(tab, NO, R, ub, ldub, zpub, ws, st, n, zlo, zhi, max_ctas)
                               : launch_lines_t<8, 4>(tab, NO, R, ub, ldub, zpub, ws, st, n, zlo, zhi, max_ctas);
  else nterms == 6 ? launch_lines_t<4, 6>(tab, NO, R, ub, ldub, zpub, ws, st, n, zlo, zhi, max_ctas)
                   : launch_lines_t<4, 4>(tab, NO, R, ub, ldub, zpub, ws, st, n, zlo, zhi, max_ctas);
}

void launch_band_planes(int L, int nterms, const double* tab, int NO, int R, const double* ub, int ldub, int zpub,
                        const double* ws, double* Y, const double* corr, double scale, cudaStream_t st, int n,
                        int zlo, int zhi, double* fred, int nf) {
  zpub = zpub ? zpub : 64;
  zhi = std::min(zhi, 1 << L);
  if (L == 4) nterms == 6 ? launch_planes_t<16, 6>(tab, NO, R, ub, ldub, zpub, ws, Y, corr, scale, st, n, zlo, zhi, fred, nf)
                          : launch_planes_t<16, 4>(tab, NO, R, ub, ldub, zpub, ws, Y, corr, scale, st, n, zlo, zhi, fred, nf);
  else if (L == 3) nterms == 6 ? launch_planes_t<8, 6>(tab, NO, R, ub, ldub, zpub, ws, Y, corr, scale, st, n, zlo, zhi, fred, nf)
                               : launch_planes_t<8, 4>(tab, NO, R, ub, ldub, zpub, ws, Y, corr, scale, st, n, zlo, zhi, fred, nf);
  else nterms == 6 ? launch_planes_t<4, 6>(tab, NO, R, ub, ldub, zpub, ws, Y, corr, scale, st, n, zlo, zhi, fred, nf)
                   : launch_planes_t<4, 4>(tab, NO, R, ub, ldub, zpub, ws, Y, corr, scale, st, n, zlo, zhi, fred, nf);
}

void launch_band_ylines(int L, int nterms, const double* tab, int NO, int R, const double* ws, double* ws2, double* Y,
                        const double* src, int ldub, int zpub, int n, const double* corr, double scale,
                        cudaStream_t st, int zlo, int zhi) {
  zpub = zpub ? zpub : 64;
  zhi = std::min(zhi, 1 << L);
  if (zhi <= zlo) return;
  if (L == 4) nterms == 6 ? launch_ylines_t<16, 6>(tab, NO, R, ws, ws2, Y, src, ldub, zpub, n, corr, scale, st, zlo, zhi)
                          : launch_ylines_t<16, 4>(tab, NO, R, ws, ws2, Y, src, ldub, zpub, n, corr, scale, st, zlo, zhi);
  else if (L == 3)
    nterms == 6 ? launch_ylines_t<8, 6>(tab, NO, R, ws, ws2, Y, src, ldub, zpub, n, corr, scale, st, zlo, zhi)
                : launch_ylines_t<8, 4>(tab, NO, R, ws, ws2, Y, src, ldub, zpub, n, corr, scale, st, zlo, zhi);
  else nterms == 6 ? launch_ylines_t<4, 6>(tab, NO, R, ws, ws2, Y, src, ldub, zpub, n, corr, scale, st, zlo, zhi)
                   : launch_ylines_t<4, 4>(tab, NO, R, ws, ws2, Y, src, ldub, zpub, n, corr, scale, st, zlo, zhi);
}

}  // namespace htlr
