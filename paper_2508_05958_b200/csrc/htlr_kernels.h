// Kernel launch interface shared by the plan (htlr_plan.cu) and the kernel
// translation units.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "htlr_device.cuh"

namespace htlr {

constexpr int kMaxRank = 16;
constexpr int kMaxLevels = 16;

struct FactorJob {
  int side;
  double* Q;      // side x p row-major (identity when side == p)
  double* R;      // p x p row-major (raw square factor when side == p)
  double* work;   // side x p scratch
  double* work2;  // side x p scratch
};

struct CoreJob {
  int tlo[3];
  int slo[3];
  int side;
  const double* R;   // level factor folded into the core
  double* dst;       // tiled GEMM table slot
};

struct NearJob {
  int tlo[3];
  int slo[3];
  int self;
  double* dst;
};

// one GEMM task: rows of `mat` applied to up to NT columns (pairs x rhs)
struct GemmTask {
  int mat;
  int pair_begin;
  int pair_count;
  int r0;
  int kc0;   // K range of the item in 32-wide chunks (the whole K extent:
  int nkc;   // kc0 = 0, nkc = K_pad / 32)
};

// coarse-level contribution gathered by the fused downward kernel
struct DownLevel {
  int level;
  int side;        // box side at this level
  int P;           // p^d
  const double* Q; // side x p row-major (uniform), or per-interval tables
  const double* H; // [cluster][R][P]
  int64_t qstride; // 0: one factor for the level; else doubles per interval
  const double* K; // H-matrix baseline: dense Kronecker factor (side^d x P), else null
};

// mapped grid: per (level, interval) nodes and raw factors
struct MappedFactorJob {
  int side;
  int nint;        // intervals per dimension at this level
  double* nodes;   // [nint][p]
  double* L;       // [nint][side][p]   raw Lagrange factor (target side)
  double* WL;      // [nint][side][p]   cell widths x factor (source side)
};

struct DownParams {
  int nlev;
  DownLevel lev[kMaxLevels];
};

void launch_diag(const KernelParams& kp, int d, double h, int q, const double* gx, const double* gw,
                 int singular, double* out, cudaStream_t st);
void launch_factor_qr(int nlev, const FactorJob* jobs, double h, int p, cudaStream_t st);
void launch_core_batch(const CoreJob* jobs, int nbatch, int d, int p, double h, double hd,
                       const KernelParams& kp, double* buf0, double* buf1, int MT, int M_pad, int K_pad,
                       cudaStream_t st);
// Toeplitz generators of 3-D near blocks with leaf side 8: (2*8-1)^3 values
// each, padded to a 16-byte multiple
constexpr int kGenSide = 15;
constexpr int kGenStride = kGenSide * kGenSide * kGenSide + 1;
void launch_near_gen(const double* table, int64_t mat_stride, int nmats, int MT, int K_pad, double* gen,
                     cudaStream_t st);
void launch_near_blocks(const NearJob* jobs, int njobs, int d, int s, double h, double hd,
                        const KernelParams& kp, const double* diag, int MT, int M_pad, int K_pad,
                        cudaStream_t st);

// matvec kernels (htlr_apply.cu)
// index ranges are Morton ids (see htlr_device.cuh)
// accumulators the permute launch also zeroes (saves the memset nodes of an
// unsharded matvec graph)
struct ZeroList {
  double* p[kMaxLevels + 2];
  int64_t n[kMaxLevels + 2];
  int cnt = 0;
};
// zpitch (3-D): doubles between the z-planes of a stored box vector (0 =
// natural layout; the separable passes use 68 so one bulk copy of a box lands
// bank-conflict free in shared memory)
void launch_permute_in(const double* u, double* ub, int d, int n, int s, int R, int K_pad, int64_t b0,
                       int64_t nb, cudaStream_t st, const ZeroList* zero = nullptr, int zpitch = 0);
// one launch for permute + zeroing + the upward pass of every compressed
// level (unsharded matvec); nb_zero and bits_L are filled in by the launcher
struct UpLevel {
  double* W;
  const double* Q;
  int64_t qstride, c0, nc;
  int side, bits, K_pad;
  // nslab > 1 (3-D): each (cluster, rhs) is split over nslab CTAs of
  // side / nslab z-planes; their partial W land in `scratch` and the last CTA
  // to arrive (per-(cluster, rhs) counter, reset by it) sums them into W
  int nslab;
  double* scratch;   // [cluster - c0][rhs][nslab][p^3]
  int* counters;     // [cluster - c0][rhs], zero between launches
  int zpitch;        // z-plane pitch of W (0: natural)
};
// z-slabs per cluster for a level of nc clusters x R right-hand sides (1: whole
// boxes); HTLR_UPWARD_SPLIT=0 disables the split
int upward_nslab(int d, int side, int64_t nc, int R);
struct PrologueParams {
  const double* u;
  double* ub;
  int d, n, p, sL, R, K_pad_leaf, bits_L, zpitch_leaf;
  // overlapped host-vector matvec: only the leaf boxes whose z index lies in
  // [zlo, zhi), and the upward pass only of the clusters whose last leaf-box
  // z index does (zhi == 0: everything)
  int zlo, zhi;
  int64_t b0, nb_perm, nb_zero;
  ZeroList zero;
  int nlev;
  UpLevel lev[kMaxLevels];
};
size_t upward_smem_words(int d, int side, int p);
void launch_prologue(const PrologueParams& pp, cudaStream_t st);
void launch_upward(const double* u, double* W, int d, int n, int side, int p, int level, int R,
                   int K_pad, const double* Q, int64_t qstride, int64_t c0, int64_t nc, cudaStream_t st,
                   int nslab = 1, double* scratch = nullptr, int* counters = nullptr, int zpitch = 0);
// MT selects the tile config (64 or 128)
int gemm_mt_for(int P_out);
// gen: Toeplitz generators of the pass's matrices (near-only 3-D leaf pass
// with leaf side 8) or nullptr; the narrow items then build their A
// fragments from them instead of streaming the stored blocks
void launch_gemm(int MT, int NT, const double* A, int64_t mat_stride, const double* B, double* C,
                 const GemmTask* tasks, int ntasks, const int2* pairs, int R, int Rc, int K_pad,
                 int M_valid, int ldc, int RT, cudaStream_t st, const double* gen = nullptr);
int gemm_nt(int MT);
int gemm_wide_wn();   // warps along N of the wide persistent kernel (default 3: 96 columns; HTLR_GEMM_WN=2: 64)
// persistent warp-specialised variant (htlr_gemm.cu); HTLR_GEMM=legacy selects
// the one-CTA-per-item cp.async kernel instead
bool gemm_use_persistent();
int gemm_stage_chunks(int MT, int K_pad);   // 32-wide K chunks per pipeline stage
int thin_m8_supported(int m8);
void launch_gemm_thin(int M_pad, int NT, const double* A, int64_t mat_stride, const double* B, double* C,
                      const GemmTask* tasks, int ntasks, const int2* pairs, int R, int Rc, int K_pad, int M_valid,
                      int ldc, cudaStream_t st);
void launch_gemm_persistent(int MT, int NT, const double* A, int64_t mat_stride, const double* B, double* C,
                            const GemmTask* tasks, int ntasks, const int2* pairs, int R, int Rc, int K_pad,
                            int M_valid, int ldc, int RT, cudaStream_t st, const double* gen = nullptr);
void launch_downward(const double* u, double* f, const double* Y, int ldy, const double* a_vec,
                     double a_const, const double* dvec, int d, int n, int sL, int L, int R, int p,
                     const DownParams& dp, int64_t b0, int64_t nb, cudaStream_t st);

// separable-core formulation (htlr_sep.cu): tensor-product kernels (the
// Gaussian) on uniform grids with p = leaf side = 8 in 3-D
constexpr int kSepP = 8;
constexpr int kSepSlot = 256;       // doubles per (kind, offset) table slot in HBM
constexpr int kSepSlotSmem = 192;   // the part the apply kernel stages in shared memory
constexpr int kSepWarps = 8;
constexpr int kSepMaxNO = 15;       // per-axis offsets -7..7 (4-bit codes)
struct SepJob {
  int kind;          // 0 admissible core factor, 1 near-block factor
  int o;             // per-axis box offset (source - target)
  int t0;            // representative target box index (t0 and t0 + o inside the domain)
  int side;          // box side at the pass's level
  const double* R;   // level factor (p x p row-major), admissible only
  double* dst;       // kSepSlot doubles
};
// a warp's work: pairs [begin, begin + count) of target `tgt`; flags bit 0:
// the run holds the self pair (near-field diagonal correction)
struct SepItem {
  int tgt, begin, count, flags;
};
// cooperative leaf-pass variant (sep_block_kernel): one CTA per (parent
// cluster, part of its source columns); warp w applies the blocks of child
// target tgt0 + w, the source boxes of a column (equal x, y box coordinates)
// are staged once per CTA by bulk copies and shared by the 8 warps
constexpr int kSepColMax = 10;      // source boxes per column
constexpr int kSepZPitch = 68;      // z-plane pitch of staged (and, in separable plans, stored) boxes
constexpr int kSepBoxSmem = 8 * kSepZPitch; // staged box: 8 z-planes of 64 doubles, padded (bank-conflict-free fragments)
// column slots in flight for NG consumer warp groups
__host__ __device__ constexpr int sep_ring_slots(int NG) { return NG == 1 ? 3 : 4; }
int sep_block_groups();
struct SepCol {
  int n;                                   // boxes in the column
  int src[kSepColMax];                     // source ids, ascending z
  unsigned short code[kSepColMax][8];      // per (box, warp): pair code, 0xFFFF = not in that target's list
  int pad;
};
struct SepBlock {
  int tgt0, col_begin, col_count, corr_mask;   // corr_mask bit w: warp w's self pair is in this part
};
size_t sep_block_smem_bytes(int nslots);
void launch_sep_block(const double* tables, int nslots, int NO, const SepBlock* blocks, int nblocks, const SepCol* cols,
                      const double* B, int ldb, double* C, int ldc, int R, const double* corr, cudaStream_t st,
                      int zpitch = 0);
void launch_sep_tables(const SepJob* jobs, int njobs, int p, int sL, double h, const KernelParams& kp,
                       const double* diag, double hd, double* corr_out, cudaStream_t st);
size_t sep_smem_bytes(int nslots);
// banded leaf pass (eta = 1 strong admissibility, htlr_sep.cu): three line
// sweeps (sweep 0: z, ub -> six term buffers; 1: y, in place; 2: x, Y +=)
size_t sep_band_smem_bytes(int NO, int L);
int64_t sep_band_workspace(int L, int R);   // doubles
cudaError_t sep_band_init();
// nterms: 6 at the leaf level (admissible + near terms), 4 at a coupling
// level (admissible terms only); corr may be null (no self-block correction)
// lo / hi: the own target boxes (a box region; the whole level unsharded):
// the z sweep runs the lines within 5 boxes of it in x and y and outputs its
// z range, the y-x sweep its z planes, storing only its cells
void launch_sep_band(int sweep, const double* tables, int NO, int L, int R, const double* ub, int ldub, int zpub,
                     double* ws, double* Y, const double* corr, double scale, int nterms, cudaStream_t st,
                     const int* lo, const int* hi);
// register-line sweeps (htlr_band.cu): z sweep (source -> term buffers) and
// the fused y-x sweep of every z-point plane (term buffers -> Y), for the
// target z boxes [zlo, zhi) of the level (a z-slab shard; 0, 1 << L whole).
// n > 0: the source (and the self-correction's u) is the F-order grid vector
// u[N][R] of an n^3 grid instead of the level's boxes [box][R][ldub].
bool band_lines_supported(int L);
// per-block drop-in API (htlr_tensor.cu): host arrays, row-major
cudaError_t tensor_mode_product(const double* t, int64_t A, int64_t K, int64_t B, const double* m, int64_t M,
                                double* out);
cudaError_t tensor_gemm(const double* a, const double* b, int64_t m, int64_t k, int64_t n, double* c);
cudaError_t tensor_kron(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc,
                        double* out);
cudaError_t tensor_qr(const double* a, int64_t rows, int64_t cols, double* q, double* r);
// max_ctas > 0 caps the z sweep's persistent grid (SMs left to a concurrent stream)
void launch_band_lines(int L, int nterms, const double* tab, int NO, int R, const double* ub, int ldub, int zpub,
                       double* ws, cudaStream_t st, int n = 0, int zlo = 0, int zhi = 1 << 30, int max_ctas = 0);
void launch_band_planes(int L, int nterms, const double* tab, int NO, int R, const double* ub, int ldub, int zpub,
                        const double* ws, double* Y, const double* corr, double scale, cudaStream_t st, int n = 0,
                        int zlo = 0, int zhi = 1 << 30, double* fred = nullptr, int nf = 0);
// the y-x sweep as two line kernels over all SMs (z-slab shards: a slab has
// few planes): ws (z-swept terms) -> ws2 (y-swept, B-fragment order) -> Y
void launch_band_ylines(int L, int nterms, const double* tab, int NO, int R, const double* ws, double* ws2, double* Y,
                        const double* src, int ldub, int zpub, int n, const double* corr, double scale,
                        cudaStream_t st, int zlo, int zhi);
// pairs: int2 (source id, code), code = kind << 12 | ix << 8 | iy << 4 | iz
// (per-axis offset + (NO - 1) / 2); table slot of (kind, i) = kind * NO + i
void launch_sep_apply(const double* tables, int nslots, int NO, const SepItem* items, int nitems, const int2* pairs,
                      const double* B, int ldb, double* C, int ldc, int R, const double* corr, cudaStream_t st,
                      int zpitch = 0);

struct BandRegion {
  int lo[3], hi[3];
};
// upward / downward passes over cubes (htlr_cube.cu): the level-(L-1) boxes
// of separable plans (p = leaf side = 8, 3-D); coarser compressed levels via
// 8 x 8 transfer matrices M_l = Q_c^T Q_l[cube rows] per axis and sub-position
constexpr int kMaxCubeCoarse = 4;
struct CubeLevel {
  int level;
  const double* M;   // [2^(L-1-level)][8 x 8], M[a'][a] (a' the cube's coefficient)
  double* W;         // [cluster][R][K_pad], pitched z-planes (RED target)
  const double* H;   // [cluster][R][512]
  int K_pad, zpitch;
};
struct CubeLevels {
  const double* Qc;   // level L-1 factor, 16 x 8 row-major; null: no compressed level
  double* Wc;         // W_{L-1} [cube][R][K_pad_c] (stored, no atomics)
  const double* Hc;   // H_{L-1} [cube][R][512]
  int K_pad_c, zpitch_c;
  int ncoarse;
  CubeLevel lev[kMaxCubeCoarse];
};
bool cube_supported(int d, int p, int sL, int L);
// [zlo, zhi): leaf-box z range (whole cubes: even bounds)
void launch_upward_cube(const CubeLevels& cl, int L, int R, int64_t nb, cudaStream_t st, const double* u,
                        double* ub_out, int ldub, int zpub, int n, int zlo = 0, int zhi = 1 << 30);
void launch_downward_cube(const CubeLevels& cl, int L, int R, int64_t b0, int64_t nb, cudaStream_t st,
                          const double* u, double* f, const double* Y, const double* a_vec, double a_const, int n,
                          int zlo = 0, int zhi = 1 << 30, bool red = false);
// mapped grid (htlr_mapped.cu)
void launch_mapped_factors(const MappedFactorJob* jobs, int njobs, int total_intervals, const double* bounds,
                           const double* coords, const double* widths, int p, cudaStream_t st);
void launch_mapped_diag(const KernelParams& kp, int d, int n, int q, const double* gx, const double* gw,
                        const double* bounds, const double* coords, double* out, int64_t npts, cudaStream_t st);
void launch_regen_adm(const KernelParams& kp, int d, int p, int level, const double* nodes, const int64_t* rowptr,
                      const int* cols, int64_t t0, int64_t nt, const double* W, int K_pad, double* H, int R,
                      cudaStream_t st);
void launch_regen_near(const KernelParams& kp, int d, int sL, int L, const double* coords, const double* widths,
                       const int64_t* rowptr, const int* cols, int64_t t0, int64_t nt, const double* ub, int K_pad,
                       double* Y, int R, cudaStream_t st);
// symmetric regeneration (htlr_regen_sym.cu): one CTA per own row of
// `order` (global id t0 + row), its owned pairs from (uptr, ucols); OUT must
// be initialised
bool regen_sym_supported(int d, int pp);
void launch_regen_sym(const KernelParams& kp, int pp, int level, const double* ax, const int* order, int64_t nrows,
                      int64_t t0, const int64_t* uptr, const int* ucols, const double* V, int64_t vstride, double* OUT,
                      int64_t ostride, cudaStream_t st);
void launch_near_weight(int sL, int L, const double* widths, const double* ub, int K_pad, double* V, int64_t nleaf,
                        cudaStream_t st);
void launch_mapped_core_export(const KernelParams& kp, int d, int p, const double* nt, const double* ns, double* out,
                               cudaStream_t st);
void launch_mapped_near_export(const KernelParams& kp, int d, int sL, const double* xt, const double* ys,
                               const double* ws, int self, double* out, cudaStream_t st);

// exact rows (htlr_rows.cu)
void launch_exact_rows(const KernelParams& kp, int d, int n, double h, double hd, const double* coords,
                       const double* widths, const int64_t* rows, int64_t nrows, const double* cell_avg,
                       const double* dvec_all, double* diag_rows, const double* avec, double aconst,
                       const double* u, double* out, cudaStream_t st);

// H-matrix baseline (htlr_lowrank.cu): dense Kronecker factors
void launch_kron_factor(const double* Q, int d, int s, int p, double* K, cudaStream_t st);
void launch_dense_upward(const double* u, double* W, int d, int n, int side, int p, int level, int R, int K_pad,
                         const double* K, int64_t c0, int64_t nc, cudaStream_t st);

// API building blocks (htlr_interp.cu)
void launch_cheb_nodes(double lo, double hi, int p, double* out, cudaStream_t st);
void launch_lagrange(const double* pts, int64_t n, const double* nodes, int p, double* out, cudaStream_t st);
void launch_pairs(const KernelParams& kp, int d, const double* x, int64_t m1, const double* y, int64_t m2, double* out,
                  int* coincident, cudaStream_t st);

// quasi-uniform front end (htlr_quasi.cu)
void launch_overlap(const double* tri_xy, const int* cand, int64_t ncand, int m_side, double* areas,
                    cudaStream_t st);
void launch_csr_spmv(const int64_t* rowptr, const int* cols, const double* vals, int64_t nrows, const double* x,
                     double* y, cudaStream_t st);

}  // namespace htlr
