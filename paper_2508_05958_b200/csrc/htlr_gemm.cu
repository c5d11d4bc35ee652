// Persistent, warp-specialised gathered fp64 tensor-core GEMM (sm_100a).
//
// Same contract as gemm_gather_kernel (htlr_apply.cu): a work item is
// (task, row tile); the item computes C[tgt][r][rows] += A_mat[rows][:] .
// B[src][r][:] over its (tgt, src) pairs x RHS columns.  This version keeps
// one CTA resident per SM and streams items through a STAGES-deep shared
// memory ring:
//   * a producer warp issues 1-D TMA bulk copies (cp.async.bulk ->
//     UBLKCP) -- one contiguous copy for the pre-tiled A slab of a 32-wide K
//     chunk and one 256-byte copy per gathered B column -- completing a
//     `full` mbarrier by transaction count;
//   * 8 consumer warps run mma.sync.m16n8k8.f64 (DMMA) from the ring and
//     release each slot with an `empty` mbarrier arrive, so no CTA-wide
//     barrier stalls the tensor pipe and the next item's loads overlap the
//     current item's last chunks and epilogue (fp64 RED into L2).
// Items are assigned round-robin, so at any moment the 148 CTAs work on
// consecutive items (the same or neighbouring offsets): each unique core is
// fetched from HBM once and served to the other CTAs from L2.
#include <cstdlib>
#include <cstring>

#include "htlr_kernels.h"
#include "htlr_mbarrier.cuh"

namespace htlr {

namespace {

// one mma.m8n8k4: (c0, c1) += a (8x4 row) . b (4x8 col)
__device__ __forceinline__ void mma8x8x4_pair(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct ItemInfo {
  int mat, pair_begin, pair_count, r0, rt, ncols, kc0, nkc;
};

__device__ __forceinline__ ItemInfo item_info(const GemmTask* tasks, int item, int RT, int R, int Rc, int NT) {
  ItemInfo it;
  const GemmTask tk = tasks[item / RT];
  it.rt = item % RT;
  it.mat = tk.mat;
  it.pair_begin = tk.pair_begin;
  it.pair_count = tk.pair_count;
  it.r0 = tk.r0;
  it.ncols = (Rc == NT) ? min(NT, R - tk.r0) : tk.pair_count * Rc;
  it.kc0 = tk.kc0;
  it.nkc = tk.nkc;
  return it;
}

}  // namespace

// One pipeline stage of a warp's (16 MI x 8 NTL) tile: the k0..3 products of
// all (m8, n8) accumulators first, then the k4..7 products, so every
// dependent DMMA pair is 2 MI NTL instructions apart (mma.m16n8k8 would emit
// each dependent pair back to back).
template <int NTL, int MI, int KC, int MT, int BST>
__device__ __forceinline__ void stage_mma(double (&acc)[MI][4][4], const double* cA, const double* cB, int wm,
                                          int wn, int lane, int g8, int t) {
#pragma unroll
  for (int ks = 0; ks < KC / 8; ++ks) {
    double a[MI][4];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const double2* pa = reinterpret_cast<const double2*>(
          cA + (ks >> 2) * (MT * kKC) + ((wm * MI + mi) * (kKC / 8) + (ks & 3)) * 128 + lane * 4);
      const double2 v0 = pa[0], v1 = pa[1];
      a[mi][0] = v0.x;
      a[mi][1] = v0.y;
      a[mi][2] = v1.x;
      a[mi][3] = v1.y;
    }
    double b[NTL][2];
#pragma unroll
    for (int ni = 0; ni < NTL; ++ni) {
      const double* pb = cB + (wn * 32 + ni * 8 + g8) * BST + ks * 8 + t;
      b[ni][0] = pb[0];
      b[ni][1] = pb[4];
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NTL; ++ni) {
          mma8x8x4_pair(acc[mi][ni][0], acc[mi][ni][1], a[mi][2 * h], b[ni][h]);
          mma8x8x4_pair(acc[mi][ni][2], acc[mi][ni][3], a[mi][2 * h + 1], b[ni][h]);
        }
  }
}

// Narrow-item stage with the A fragments generated from a near block's
// Toeplitz generator G (3-D, leaf side 8): A[i][j] = G[bi(i) + kb(j)] with
// bi(i) = sum (7 - i_a) 15^a, kb(j) = sum j_a 15^a.  kabs = first K index of
// the stage (a multiple of 32), bia / bib = bi of the thread's rows g8, g8 + 8.
template <int NTL, int KC, int BST>
__device__ __forceinline__ void stage_mma_gen(double (&acc)[1][4][4], const double* G, const double* cB, int bia,
                                              int bib, int kabs, int wn, int g8, int t) {
#pragma unroll
  for (int ks = 0; ks < KC / 8; ++ks) {
    const int kk = kabs + ks * 8;
    const int kb = t + kGenSide * ((kk >> 3) & 7) + kGenSide * kGenSide * (kk >> 6);
    double a[4];
    a[0] = G[bia + kb];
    a[1] = G[bib + kb];
    a[2] = G[bia + kb + 4];
    a[3] = G[bib + kb + 4];
    double b[NTL][2];
#pragma unroll
    for (int ni = 0; ni < NTL; ++ni) {
      const double* pb = cB + (wn * 32 + ni * 8 + g8) * BST + ks * 8 + t;
      b[ni][0] = pb[0];
      b[ni][1] = pb[4];
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int ni = 0; ni < NTL; ++ni) {
        mma8x8x4_pair(acc[0][ni][0], acc[0][ni][1], a[2 * h], b[ni][h]);
        mma8x8x4_pair(acc[0][ni][2], acc[0][ni][3], a[2 * h + 1], b[ni][h]);
      }
  }
}

template <int WM, int WN, int STAGES, int KCS, int MI = 2, bool GEN = false>
__global__ void __launch_bounds__((WM * WN + 1) * 32, 1)
    gemm_persistent_kernel(const double* __restrict__ A, int64_t mat_stride, const double* __restrict__ B,
                           double* __restrict__ C, const GemmTask* __restrict__ tasks, int nitems,
                           const int2* __restrict__ pairs, int R, int Rc, int K_pad, int M_valid, int ldc,
                           int RT, const double* __restrict__ gen) {
  // a pipeline stage covers KCS = 32 or 64 of K (one or two tiled 32-chunks,
  // adjacent in the A layout); fewer, larger stages halve the mbarrier
  // round trips per unit of tensor work
  // warp tile = MI m16 row tiles x 4 n8 column tiles (MI = 1: "narrow" items
  // of 32 columns for passes with few pairs per matrix)
  constexpr int MT = 16 * MI * WM, NT = 32 * WN, KC = KCS, BST = KC + 4;
  constexpr int NCW = WM * WN;   // consumer warps
  // GEN: no A stages; the item's Toeplitz generator goes to one of two
  // slots instead (an item spans more stages than the ring, so the slot of
  // item i - 1 is free when item i + 1's first stage is issued)
  constexpr int ASTAGE = GEN ? 0 : MT * KC;
  extern __shared__ __align__(128) double smem[];
  double* sA = smem;                                  // STAGES x MT*KC
  double* sB = smem + STAGES * ASTAGE;                // STAGES x NT*BST
  double* sG = sB + STAGES * NT * BST;                // GEN: 2 x kGenStride
  uint64_t* full = reinterpret_cast<uint64_t*>(sG + (GEN ? 2 * kGenStride : 0));
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == NCW) {
    // ------------------------------------------------------------ producer
    // the next item's task record and gathered-column bases are loaded while
    // the current item's stages are issued (short items would otherwise
    // stall the ring on two dependent global loads per item)
    uint32_t g = 0;
    int item = blockIdx.x;
    ItemInfo it{};
    int64_t cb[NT / 32];
    auto load_cols = [&](const ItemInfo& x, int64_t (&c)[NT / 32]) {
#pragma unroll
      for (int q = 0; q < NT / 32; ++q) {
        const int n = lane + 32 * q;
        c[q] = -1;
        if (n < x.ncols) {
          const int j = n / Rc, r = x.r0 + n % Rc;
          c[q] = ((int64_t)pairs[x.pair_begin + j].y * R + r) * K_pad;
        }
      }
    };
    if (item < nitems) {
      it = item_info(tasks, item, RT, R, Rc, NT);
      load_cols(it, cb);
    }
    for (int ci = 0; item < nitems; item += gridDim.x, ++ci) {
      const int nxt = item + gridDim.x;
      ItemInfo itn{};
      int64_t cbn[NT / 32];
      if (nxt < nitems) {
        itn = item_info(tasks, nxt, RT, R, Rc, NT);
        load_cols(itn, cbn);
      }
      const double* Ablk = A + (int64_t)it.mat * mat_stride + (int64_t)it.rt * MT * K_pad;
      const unsigned bytes = (unsigned)(ASTAGE * 8 + it.ncols * KC * 8);
      const int kbeg = it.kc0 * kKC / KC, kend = kbeg + it.nkc * kKC / KC;   // stage units
      for (int kc = kbeg; kc < kend; ++kc, ++g) {
        const int s = g % STAGES;
        if (g >= (uint32_t)STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
        if (lane == 0) {
          if constexpr (GEN) {
            const bool first = kc == kbeg;
            mbar_arrive_expect_tx(&full[s], bytes + (first ? kGenStride * 8u : 0u));
            if (first)
              bulk_g2s(sG + (ci & 1) * kGenStride, gen + (int64_t)it.mat * kGenStride, kGenStride * 8, &full[s]);
          } else {
            mbar_arrive_expect_tx(&full[s], bytes);
            bulk_g2s(sA + s * MT * KC, Ablk + (int64_t)kc * MT * KC, MT * KC * 8, &full[s]);
          }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < NT / 32; ++q) {
          const int n = lane + 32 * q;
          if (cb[q] >= 0) bulk_g2s(sB + s * NT * BST + n * BST, B + cb[q] + kc * KC, KC * 8, &full[s]);
        }
      }
      it = itn;
#pragma unroll
      for (int q = 0; q < NT / 32; ++q) cb[q] = cbn[q];
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int wm = warp % WM, wn = warp / WM;
  const int g8 = lane >> 2, t = lane & 3;
  uint32_t g = 0;
  ItemInfo itn{};
  if (blockIdx.x < nitems) itn = item_info(tasks, blockIdx.x, RT, R, Rc, NT);
  for (int item = blockIdx.x, ci = 0; item < nitems; item += gridDim.x, ++ci) {
    const ItemInfo it = itn;
    if (item + (int)gridDim.x < nitems) itn = item_info(tasks, item + gridDim.x, RT, R, Rc, NT);
    const int n_tiles = max(0, min(4, (it.ncols - wn * 32 + 7) >> 3));
    const int row0 = it.rt * MT + wm * 16 * MI;
    // GEN: generator slot and the row halves of the Toeplitz index
    const double* gslot = sG + (ci & 1) * kGenStride;
    auto gen_row = [](int r) {
      return (7 - (r & 7)) + kGenSide * (7 - ((r >> 3) & 7)) + kGenSide * kGenSide * (7 - (r >> 6));
    };
    const int bia = gen_row(row0 + g8), bib = gen_row(row0 + g8 + 8);
    const int m_tiles = max(0, min(MI, (M_valid - row0 + 15) >> 4));
    // epilogue targets of this thread's 8 columns, fetched now so the pair
    // loads' latency hides under the K loop
    int cvec[8];   // target vector index (tgt * R + r) of each of this thread's columns, -1 if empty
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int n = wn * 32 + (q >> 1) * 8 + 2 * t + (q & 1);
      cvec[q] = -1;
      if (n < it.ncols) {
        const int j = n / Rc, r = it.r0 + n % Rc;
        cvec[q] = pairs[it.pair_begin + j].x * R + r;
      }
    }
    double acc[MI][4][4];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
    const int nstage = it.nkc * kKC / KC;
    for (int kc = 0; kc < nstage; ++kc, ++g) {
      const int s = g % STAGES;
      mbar_wait(&full[s], (g / STAGES) & 1);
      const double* cA = sA + s * MT * KC;
      const double* cB = sB + s * NT * BST;
      // full row tiles: explicit m8n8k4 issue order.  The narrow variant
      // (MI = 1, passes whose items are mostly partial) also gets the 1..3
      // column-tile counts as compile-time constants: a predicated-off DMMA
      // still occupies the tensor pipe (measured 1.45x the issued work on
      // cfg 2's leaf pass).  The wide variants keep one specialised body:
      // four of them cost more in instruction-cache misses (cfg 3: +48%).
      if constexpr (GEN) {
        const int kabs = (it.kc0 * kKC / KC + kc) * KC;
        if (n_tiles == 4)
          stage_mma_gen<4, KC, BST>(acc, gslot, cB, bia, bib, kabs, wn, g8, t);
        else if (n_tiles == 3)
          stage_mma_gen<3, KC, BST>(acc, gslot, cB, bia, bib, kabs, wn, g8, t);
        else if (n_tiles == 2)
          stage_mma_gen<2, KC, BST>(acc, gslot, cB, bia, bib, kabs, wn, g8, t);
        else if (n_tiles == 1)
          stage_mma_gen<1, KC, BST>(acc, gslot, cB, bia, bib, kabs, wn, g8, t);
      } else if (m_tiles == MI && n_tiles == 4)
        stage_mma<4, MI, KC, MT, BST>(acc, cA, cB, wm, wn, lane, g8, t);
      else if (MI == 1 && m_tiles == MI && n_tiles == 3)
        stage_mma<3, MI, KC, MT, BST>(acc, cA, cB, wm, wn, lane, g8, t);
      else if (MI == 1 && m_tiles == MI && n_tiles == 2)
        stage_mma<2, MI, KC, MT, BST>(acc, cA, cB, wm, wn, lane, g8, t);
      else if (MI == 1 && m_tiles == MI && n_tiles == 1)
        stage_mma<1, MI, KC, MT, BST>(acc, cA, cB, wm, wn, lane, g8, t);
      else if (n_tiles > 0 && m_tiles > 0) {
#pragma unroll
        for (int ks = 0; ks < KC / 8; ++ks) {
          double a[MI][4];
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) {
            const double2* pa = reinterpret_cast<const double2*>(
                cA + (ks >> 2) * (MT * kKC) + ((wm * MI + mi) * (kKC / 8) + (ks & 3)) * 128 + lane * 4);
            const double2 v0 = pa[0], v1 = pa[1];
            a[mi][0] = v0.x;
            a[mi][1] = v0.y;
            a[mi][2] = v1.x;
            a[mi][3] = v1.y;
          }
          double b[4][2];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            const double* pb = cB + (wn * 32 + ni * 8 + g8) * BST + ks * 8 + t;
            b[ni][0] = pb[0];
            b[ni][1] = pb[4];
          }
#pragma unroll
          for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
              if (mi < m_tiles && ni < n_tiles) mma16x8x8(acc[mi][ni], a[mi], b[ni]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // epilogue: fp64 RED into the accumulators (columns of stale B slots in a
    // partially filled n8 tile only pollute their own, never-stored columns)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
      for (int cix = 0; cix < 2; ++cix) {
        const int cv = cvec[ni * 2 + cix];
        if (cv < 0) continue;
        double* cc = C + (int64_t)cv * ldc;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
#pragma unroll
          for (int hi = 0; hi < 2; ++hi) {
            const int m = row0 + mi * 16 + g8 + 8 * hi;
            if (m < M_valid) atomicAdd(cc + m, acc[mi][ni][2 * hi + cix]);
          }
        }
      }
    }
  }
}

__device__ __forceinline__ void mma8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// One pipeline stage of a thin-kernel warp: row tiles rw, rw + RG, ... (NJ of
// them) x TN n8 column tiles, K = KC in m8n8k4 steps.
template <int NJ, int MJ, int TN, int KC, int M8, int BST, int G = 3>
__device__ __forceinline__ void thin_stage(double (&acc)[MJ][TN][2], const double* cA, const double* cB, int lane,
                                           int rw, int RG) {
  // two k4 steps per 16-byte A load; row tiles in groups of G so the two
  // DMMAs of one accumulator are G * TN instructions apart (G = 3 measured
  // best on config 3's coupling pass: 6.01 ms against 6.16 / 6.32 for 4 / 2)
#pragma unroll
  for (int j = 0; j < KC / 8; ++j) {
    double b[2][TN];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int ni = 0; ni < TN; ++ni) b[h][ni] = cB[ni * 8 * BST + (2 * j + h) * 4];
    const double* pa = cA + j * (M8 * 64) + lane * 2;
#pragma unroll
    for (int i0 = 0; i0 < NJ; i0 += G) {
      double2 a[G];
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (i0 + g < NJ) a[g] = *reinterpret_cast<const double2*>(pa + (rw + RG * (i0 + g)) * 64);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (i0 + g < NJ)
#pragma unroll
            for (int ni = 0; ni < TN; ++ni) mma8x8x4(acc[i0 + g][ni], h ? a[g].y : a[g].x, b[h][ni]);
    }
  }
}

// ---------------------------------------------------------------------------
// "thin" variant for matrices of at most 256 rows (p^d = 216, 64, 36, ...):
// one item covers ALL rows of its matrix (M_pad = 8*M8, no row-tile padding
// beyond 7 rows) and 64 columns; each of the 8 consumer warps owns 8 columns
// and runs M8 independent mma.m8n8k4 chains per k4 step.  Rows tiled in m8
// units keep every SM sub-partition equally busy for P = 216, which the
// 128-row tiles of the wide kernel cannot (216 = 128 + 88).
// ---------------------------------------------------------------------------
template <int M8, int STAGES, int CW, int TN, int G = 3>
__global__ void __launch_bounds__(9 * 32, 1)
    gemm_thin_kernel(const double* __restrict__ A, int64_t mat_stride, const double* __restrict__ B,
                     double* __restrict__ C, const GemmTask* __restrict__ tasks, int nitems,
                     const int2* __restrict__ pairs, int R, int Rc, int K_pad, int M_valid, int ldc) {
  // CW column warps x (8 / CW) row warps: CW = 8 gives each warp 8 columns
  // and all M8 row tiles (64 columns per item); CW = 2 / 1 (16 / 8 columns
  // per item, for passes with few pairs per matrix) split the row tiles
  // round-robin over 4 / 8 warps so every warp has work
  // TN n8 column tiles per warp (TN = 2: each A fragment feeds two DMMAs)
  constexpr int MP = 8 * M8, NT = 8 * CW * TN, KC = kKC, BST = KC + 4, NCW = 8;
  constexpr int RG = 8 / CW, MJ = (M8 + RG - 1) / RG;
  extern __shared__ __align__(128) double smem[];
  double* sA = smem;                      // STAGES x MP*KC
  double* sB = smem + STAGES * MP * KC;   // STAGES x NT*BST
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * NT * BST);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == NCW) {
    uint32_t g = 0;
    int item = blockIdx.x;
    ItemInfo it{};
    int64_t cb[2];
    auto load_cols = [&](const ItemInfo& x, int64_t (&c)[2]) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int n = lane + 32 * q;
        c[q] = -1;
        if (n < x.ncols && n < NT) {
          const int j = n / Rc, r = x.r0 + n % Rc;
          c[q] = ((int64_t)pairs[x.pair_begin + j].y * R + r) * K_pad;
        }
      }
    };
    if (item < nitems) {
      it = item_info(tasks, item, 1, R, Rc, NT);
      load_cols(it, cb);
    }
    for (; item < nitems; item += gridDim.x) {
      const int nxt = item + gridDim.x;
      ItemInfo itn{};
      int64_t cbn[2] = {-1, -1};
      if (nxt < nitems) {
        itn = item_info(tasks, nxt, 1, R, Rc, NT);
        load_cols(itn, cbn);
      }
      const double* Ablk = A + (int64_t)it.mat * mat_stride;
      const unsigned bytes = (unsigned)(MP * KC * 8 + it.ncols * KC * 8);
      const int kbeg = it.kc0 * kKC / KC, kend = kbeg + it.nkc * kKC / KC;   // stage units
      for (int kc = kbeg; kc < kend; ++kc, ++g) {
        const int s = g % STAGES;
        if (g >= (uint32_t)STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[s], bytes);
          bulk_g2s(sA + s * MP * KC, Ablk + (int64_t)kc * MP * KC, MP * KC * 8, &full[s]);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int n = lane + 32 * q;
          if (cb[q] >= 0) bulk_g2s(sB + s * NT * BST + n * BST, B + cb[q] + kc * KC, KC * 8, &full[s]);
        }
      }
      it = itn;
      cb[0] = cbn[0];
      cb[1] = cbn[1];
    }
    return;
  }
  const int g8 = lane >> 2, t = lane & 3;
  const int n0 = (warp % CW) * 8 * TN, rw = warp / CW;
  uint32_t g = 0;
  ItemInfo itn{};
  if (blockIdx.x < nitems) itn = item_info(tasks, blockIdx.x, 1, R, Rc, NT);
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const ItemInfo it = itn;
    if (item + (int)gridDim.x < nitems) itn = item_info(tasks, item + gridDim.x, 1, R, Rc, NT);
    const bool active = n0 < it.ncols;
    int64_t cbase[TN][2];
#pragma unroll
    for (int ni = 0; ni < TN; ++ni)
#pragma unroll
      for (int cix = 0; cix < 2; ++cix) {
        const int n = n0 + ni * 8 + 2 * t + cix;
        cbase[ni][cix] = -1;
        if (n < it.ncols) {
          const int j = n / Rc, r = it.r0 + n % Rc;
          cbase[ni][cix] = ((int64_t)pairs[it.pair_begin + j].x * R + r) * ldc;
        }
      }
    double acc[MJ][TN][2];
#pragma unroll
    for (int i = 0; i < MJ; ++i)
#pragma unroll
      for (int ni = 0; ni < TN; ++ni) acc[i][ni][0] = acc[i][ni][1] = 0.0;
    const int nstage = it.nkc * kKC / KC;
    for (int kc = 0; kc < nstage; ++kc, ++g) {
      const int s = g % STAGES;
      mbar_wait(&full[s], (g / STAGES) & 1);
      if (active) {
        const double* cA = sA + s * MP * KC;
        const double* cB = sB + s * NT * BST + (n0 + g8) * BST + t;
        // warps whose last round-robin row tile is past M8 take the MJ - 1
        // body (warp-uniform branch: a predicated-off DMMA would still
        // occupy the tensor pipe)
        if (rw + RG * (MJ - 1) < M8)
          thin_stage<MJ, MJ, TN, KC, M8, BST, G>(acc, cA, cB, lane, rw, RG);
        else
          thin_stage<MJ - 1, MJ, TN, KC, M8, BST, G>(acc, cA, cB, lane, rw, RG);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (!active) continue;
#pragma unroll
    for (int ni = 0; ni < TN; ++ni)
#pragma unroll
      for (int cix = 0; cix < 2; ++cix) {
        if (cbase[ni][cix] < 0) continue;
        double* cc = C + cbase[ni][cix];
#pragma unroll
        for (int i = 0; i < MJ; ++i) {
          const int m = (rw + RG * i) * 8 + g8;
          if (rw + RG * i < M8 && m < M_valid) atomicAdd(cc + m, acc[i][ni][cix]);
        }
      }
  }
}

template <int M8, int STAGES, int CW, int TN = 1, int G = 3>
static void launch_thin_t(const double* A, int64_t mat_stride, const double* B, double* C, const GemmTask* tasks,
                          int ntasks, const int2* pairs, int R, int Rc, int K_pad, int M_valid, int ldc,
                          cudaStream_t st) {
  constexpr int MP = 8 * M8, KC = kKC;
  const size_t smem =
      sizeof(double) * STAGES * (size_t)(MP * KC + 8 * CW * TN * (KC + 4)) + 2 * STAGES * sizeof(uint64_t);
  cudaFuncSetAttribute(gemm_thin_kernel<M8, STAGES, CW, TN, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  if (ntasks == 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = ntasks < sms ? ntasks : sms;
  gemm_thin_kernel<M8, STAGES, CW, TN, G><<<grid, 9 * 32, smem, st>>>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc,
                                                            K_pad, M_valid, ldc);
}

int gemm_stage_chunks(int MT, int K_pad) {
  if (MT < 0 || MT == 64 || !gemm_use_persistent()) return 1;
  return (gemm_wide_wn() == 2 && K_pad % 64 == 0) ? 2 : 1;
}

int thin_m8_supported(int m8) { return m8 == 5 || m8 == 8 || m8 == 16 || m8 == 27; }

// 64-column thin items: 4 column warps x 2 n8 tiles (each A fragment feeds
// two DMMAs; measured cfg 3 coupling pass -2% against 8 x 1)
static int thin_tn() { return 2; }

template <int M8, int STAGES>
static void launch_thin_cw(int NT, const double* A, int64_t mat_stride, const double* B, double* C,
                           const GemmTask* tasks, int ntasks, const int2* pairs, int R, int Rc, int K_pad,
                           int M_valid, int ldc, cudaStream_t st) {
  if (NT == 8)
    launch_thin_t<M8, STAGES, 1>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, st);
  else if (NT == 16)
    launch_thin_t<M8, STAGES, 2>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, st);
  else if (thin_tn() == 2)
    launch_thin_t<M8, STAGES, 4, 2>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, st);
  else
    launch_thin_t<M8, STAGES, 8>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, st);
}

void launch_gemm_thin(int M_pad, int NT, const double* A, int64_t mat_stride, const double* B, double* C,
                      const GemmTask* tasks, int ntasks, const int2* pairs, int R, int Rc, int K_pad, int M_valid,
                      int ldc, cudaStream_t st) {
  switch (M_pad / 8) {
    case 5: launch_thin_cw<5, 4>(NT, A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, st); break;
    case 8: launch_thin_cw<8, 4>(NT, A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, st); break;
    case 16:
      launch_thin_cw<16, 3>(NT, A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, st);
      break;
    case 27:
      launch_thin_cw<27, 3>(NT, A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, st);
      break;
    default: break;   // not reachable: gemm_mt_for only selects supported sizes
  }
}

bool gemm_use_persistent() { return true; }

template <int WM, int WN, int STAGES, int KCS, int MI = 2, int CPS = 1, bool GEN = false>
static void launch_persistent_t(const double* A, int64_t mat_stride, const double* B, double* C,
                                const GemmTask* tasks, int ntasks, const int2* pairs, int R, int Rc, int K_pad,
                                int M_valid, int ldc, int RT, cudaStream_t st, const double* gen = nullptr) {
  constexpr int MT = 16 * MI * WM, NT = 32 * WN, KC = KCS;
  const size_t smem = sizeof(double) * (STAGES * (size_t)((GEN ? 0 : MT * KC) + NT * (KC + 4)) +
                                        (GEN ? 2 * kGenStride : 0)) +
                      2 * STAGES * sizeof(uint64_t);
  auto kern = gemm_persistent_kernel<WM, WN, STAGES, KCS, MI, GEN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nitems = ntasks * RT;
  if (nitems == 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = nitems < CPS * sms ? nitems : CPS * sms;   // CPS resident CTAs per SM
  kern<<<grid, (WM * WN + 1) * 32, smem, st>>>(A, mat_stride, B, C, tasks, nitems, pairs, R, Rc, K_pad, M_valid,
                                               ldc, RT, gen);
}

void launch_gemm_persistent(int MT, int NT, const double* A, int64_t mat_stride, const double* B, double* C,
                            const GemmTask* tasks, int ntasks, const int2* pairs, int R, int Rc, int K_pad,
                            int M_valid, int ldc, int RT, cudaStream_t st, const double* gen) {
  if (MT == 128 && NT == 32 && gen) {   // narrow items, A generated from Toeplitz generators
    launch_persistent_t<8, 1, 4, 32, 1, 2, true>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid,
                                                 ldc, RT, st, gen);
    return;
  }
  if (MT == 128 && NT == 32) {   // narrow items: 8 warps x (16 rows x 32 columns)
    // two CTAs per SM, two stages each (measured: cfg 2 leaf pass -7%
    // against one CTA with four stages)
    launch_persistent_t<8, 1, 2, 32, 1, 2>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, RT,
                                           st);
    return;
  }
  if (MT == 64)
    launch_persistent_t<2, 2, 6, 32>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, RT, st);
  else if (NT == 96)
    launch_persistent_t<4, 3, 3, 32>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, RT, st);
  else if (K_pad % 64 == 0)
    launch_persistent_t<4, 2, 2, 64>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, RT, st);
  else
    launch_persistent_t<4, 2, 4, 32>(A, mat_stride, B, C, tasks, ntasks, pairs, R, Rc, K_pad, M_valid, ldc, RT,
                                     st);
}

}  // namespace htlr
