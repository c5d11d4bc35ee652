// C ABI (include/htlr_b200.h) and host orchestration of the B200 HTLR plan.
//
// construct (operators.py:121-126):
//   host   : block cluster tree, bit-exact DFS leaf list (htlr_lists.cpp)
//            -> per level: admissible (tgt, src) pairs keyed by the unique
//               cluster offset; leaf level: inadmissible pairs likewise
//   device : diagonal quadrature, per-level factor + QR, one core per unique
//            (level, offset), one dense block per unique near offset, all
//            stored pre-tiled for the fp64 tensor-core GEMM
// matvec (operators.py:138-161):
//   permute_in -> upward (per level) -> gathered GEMM passes -> fused downward
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/htlr_b200.h"
#include "htlr_kernels.h"
#include "htlr_lists.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(1, std::string(#expr) + ": " + cudaGetErrorString(_e));              \
  } while (0)

int ipow(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}
int round_up(int v, int m) { return (v + m - 1) / m * m; }

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int alloc(size_t nbytes) {
    if (nbytes <= bytes && ptr) return 0;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    if (nbytes == 0) return 0;
    cudaError_t e = cudaMalloc(&ptr, nbytes);
    if (e != cudaSuccess) return fail(1, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    bytes = nbytes;
    return 0;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  double* d() const { return static_cast<double*>(ptr); }
};

// A batched gathered-GEMM pass over one interaction list.
struct Pass {
  int level = 0;
  int P = 0;               // rows == cols of every matrix (p^d or leaf side^d)
  int MT = 128, M_pad = 0, K_pad = 0, RT = 0;
  int64_t mat_stride = 0;  // doubles per tiled matrix
  int nmats = 0;
  DevBuf table;            // tiled matrices
  std::vector<int> seg;    // pairs of matrix i: [seg[i], seg[i+1])
  DevBuf pairs;            // int2 (tgt, src), sorted by (matrix, tgt)
  std::vector<int2> pairs_host;
  int npairs = 0;
  std::map<int, std::pair<DevBuf, int>> tasks;   // per R
  std::map<int, int> task_nt;                     // columns per item of the R slot's tasks
  DevBuf gen;                                     // Toeplitz generators of the matrices (near-only leaf pass)
  bool from_ub = false;    // B operand = leaf-box-major u (else W of `level`)
  bool to_y = false;       // C accumulator = Y (else H of `level`)
  // separable-core formulation (htlr_sep.cu): per-target pair runs sorted by
  // (kind, o_x, o_y, o_z), warp work items, 1-D factor tables
  DevBuf sep_tab, sep_pairs, sep_items;
  DevBuf sep_blocks, sep_cols;   // cooperative leaf-pass layout (sep_block_kernel), if built
  // leaf pass of an unsharded plan, for the overlapped host-vector matvec:
  // the domain cut into sep_slabs z-slabs of leaf boxes, columns cut at the
  // slab boundaries, parts in three ranges of sep_gcount[0..2] parts: sources
  // in the first slab (every target); later sources, targets before the last
  // slab; later sources, targets in the last slab
  DevBuf sep_gblocks, sep_gcols;
  int sep_slabs = 0;
  std::vector<int> sep_gcount;
  int sep_nitems = 0, sep_NO = 0, sep_nblocks = 0;
  int sep_own_nb = 0;            // sharded plans: parts [0, sep_own_nb) read only own sources
  double sep_own_frac = 1.0;     // their share of the pass's (pair, box) work
  int zpitch = 0;                // z-plane pitch of the pass's stored source vectors (0: natural)
  int64_t sep_groups = 0;
  bool analytic = false;         // no pair list: the level's lists are the product sets of the banded sweeps
                                 // (verified per offset on uniform dyadic grids, htlr_build_lists)
  bool band = false;             // pass as banded line sweeps (sep_band_kernel)
  DevBuf band_ws;                // its term buffers [term][box][rhs][512]
  DevBuf band_ws2;               // y-swept terms of the line-kernel y-x sweep (z-slab shards)
  double band_flops = 0;         // its algorithmic flop count per rhs (mode products it runs)
  int band_lo[3] = {0, 0, 0}, band_hi[3] = {0, 0, 0};   // own target boxes (a box region of the level)
};

// HTLR_TIMING=1: wall-clock split of list building / construction on stderr
// (synchronises the stream at each mark; development aid)
struct PhaseTimer {
  bool on = false;
  bool sync = false;
  cudaStream_t st = nullptr;
  std::chrono::steady_clock::time_point t;
  PhaseTimer() {
    const char* e = std::getenv("HTLR_TIMING");
    on = e && e[0] == '1';
    t = std::chrono::steady_clock::now();
  }
  explicit PhaseTimer(cudaStream_t s) : sync(true), st(s) {
    const char* e = std::getenv("HTLR_TIMING");
    on = e && e[0] == '1';
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    if (sync) cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[htlr timing] %-28s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Run body(i) for i in [0, n) on the host's cores (independent items).
template <typename F>
void parallel_for(size_t n, F&& body) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const unsigned nt = (unsigned)std::max<size_t>(1, std::min<size_t>(hw, n));
  std::atomic<size_t> next{0};
  auto work = [&]() {
    for (size_t i = next++; i < n; i = next++) body(i);
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
}

struct OffsetTable {
  std::unordered_map<int64_t, int> id;   // packed offset -> id (large levels)
  std::vector<int> dense;                // packed offset -> id + 1 (0: none), when (2m+1)^d is small
  std::vector<std::array<int, 6>> rep;    // representative (tc, sc)
  std::vector<std::vector<std::pair<int, int>>> members;   // (tgt, src) per id
};

int64_t pack_offset(const int* tc, const int* sc, int d, int m) {
  int64_t key = 0;
  for (int a = d - 1; a >= 0; --a) key = key * (2 * m + 1) + (sc[a] - tc[a] + m);
  return key;
}

// Upper half (sigma > tau) of a symmetric block list, rows in decreasing
// work order (longest first) for the symmetric regeneration kernel.
struct SymList {
  bool on = false;
  int64_t nrows = 0;
  DevBuf uptr, ucols, order;
  void release() {
    uptr.release();
    ucols.release();
    order.release();
    on = false;
  }
};

struct Level {
  int level = 0, side = 0, m = 0;
  int64_t nclusters = 0;
  int64_t num_adm = 0;
  OffsetTable adm;
  DevBuf Q, R;             // side x p, p x p
  DevBuf Kron;             // H-matrix baseline: dense kron(Q,..,Q), side^d x p^d
  DevBuf W, H;             // workspaces
  bool needs_up = false;   // W via upward pass, H via downward pass
  // mapped grid: per-interval nodes / raw factors, CSR of own targets
  DevBuf nodes, Lm, WLm;
  std::vector<int64_t> csr_ptr;
  std::vector<int> csr_cols;
  DevBuf d_ptr, d_cols;
  SymList sym;             // sources sigma > tau for the symmetric regeneration
  // split upward pass (few large clusters): z-slabs per cluster for the
  // current nrhs, partial-W scratch and per-(cluster, rhs) arrival counters
  int up_ns = 1;
  DevBuf up_scratch, up_count;
  // separable plans: transfer matrices from the cube level (L - 1) to this
  // coarser level, [2^(L-1-level)][8 x 8] (htlr_cube.cu)
  DevBuf Mcube;
};

}  // namespace

struct htlr_plan {
  htlr_desc desc{};
  int device = 0;
  htlr::Tree tree;
  bool lists_built = false, constructed = false;
  int d = 3, n = 0, p = 0, L = 0, sL = 0;
  int64_t N = 0;
  double h = 0, hd = 0;
  htlr::KernelParams kp{};
  std::vector<Level> levels;
  OffsetTable near;
  int64_t num_near = 0;
  std::vector<Pass> passes;   // adm passes for non-merged levels, then the leaf pass
  int leaf_pass = -1;
  int near_mats = 0;          // leaf pass: matrices [0, near_mats) are near blocks
  bool merged = false;        // leaf-level admissible cores live in the leaf pass
  int analytic_from = 0;      // > 0: levels >= this have no pair lists (Pass::analytic); the DFS stops above them
  bool sep = false;           // separable-core formulation (tensor-product kernel, htlr_sep.cu)
  bool cube_ok = false;       // separable plan whose upward / downward passes run over cubes (htlr_cube.cu)
  DevBuf sep_corr;            // self-block diagonal correction of the separable near field
  DevBuf diag, coeff, gl, ub, Y;
  DevBuf u_stage, f_stage;   // graph-replay staging vectors
  bool has_coeff = false;
  int ws_R = 0;
  int64_t last_launches = 0;
  int64_t device_scalars = 0;
  // per-launch profiling of the last matvec (htlr_profile_*)
  // mapped quasi-uniform grid (BASELINE config 5): no translation invariance,
  // cores regenerated in the matvec (htlr_mapped.cu)
  bool mapped = false;
  // H-matrix baseline (dense Kronecker factors, same cores)
  bool lowrank = false;
  std::vector<double> mb, mx, mc;          // cell bounds, coords, widths (per dim)
  DevBuf d_mb, d_mx, d_mc, dvec;
  std::vector<int64_t> near_ptr;
  std::vector<int> near_cols;
  DevBuf d_near_ptr, d_near_cols;
  SymList near_sym;                        // symmetric near field: upper pairs ...
  DevBuf d_self_ptr, d_self_cols, Vn;      // ... + the self pairs (one-sided kernel), w * u
  // sharding by cluster subtrees (multi-GPU): this plan computes the f rows
  // of leaf boxes [own_lo[L], own_hi[L]) and the upward data of its own
  // source clusters; every level's own range is a contiguous Morton range
  int shard_rank = 0, shard_world = 1;
  // z-slab shards of a banded separable plan (htlr_set_zslab): the plan keeps
  // the whole lists; the matvec covers the leaf boxes with z in [zs_lo, zs_hi)
  // (upward contributions, banded passes over the z range of each level,
  // downward, f rows), and the W_l are summed over the shards
  bool zslab = false;
  int zs_rank = 0, zs_world = 1, zs_lo = 0, zs_hi = 0;
  std::vector<int64_t> own_lo, own_hi;
  // caller-bound exchange buffers (ub, then W of each level pass), per R
  int ext_R = 0;
  std::vector<double*> ext_ptrs;
  // caller-bound reduce buffers (mapped grid, symmetric regeneration on a
  // sharded plan): H_l of each symmetric level, then Y; full size, summed
  // over the shards between htlr_matvec_contract and htlr_matvec_expand
  int red_R = 0;
  std::vector<double*> red_ptrs;
  bool profiling = false;
  // CUDA-graph replay of the whole matvec, keyed by (R, u, f, profiling)
  bool graphs = true;
  cudaStream_t cap_stream = nullptr;
  struct GraphEntry {
    int R;
    const double* u;
    double* f;
    bool prof;
    cudaGraphExec_t exec;
    std::vector<int32_t> kind, level;
    std::vector<double> flops, bytes;
    int64_t launches;
    uint64_t stamp = 0;   // last use (graph_clock)
  };
  std::vector<GraphEntry> graph_cache;
  uint64_t graph_clock = 0;
  // overlapped host-vector matvec (htlr_matvec_host): its graphs (keyed by the
  // host pointers), a copy stream and the fork / join events
  std::vector<GraphEntry> host_graphs;
  // staging vectors the host graphs were captured with (a reallocation of
  // u_stage / f_stage by another path invalidates every host graph)
  void* host_graph_stage[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;
  // concurrent level passes (mv_remote): side stream + fork / join events
  cudaStream_t side_stream = nullptr;
  cudaEvent_t side_ev[2] = {nullptr, nullptr};
  // direct-f matvec (mv_remote): the leaf y-x sweep and the downward pass both
  // sum into a zeroed f; f_red is set while that leaf sweep is launched
  cudaEvent_t fz_ev = nullptr;
  cudaEvent_t fd_ev[2] = {nullptr, nullptr};   // fork / join of the third stream (leaf_stream) of that matvec
  double* f_red = nullptr;
  // z-slab shards: the leaf pass reads only u, so the local phase starts it
  // on its own stream, beside the upward pass and the exchange; the remote
  // phase joins it before the downward pass
  cudaStream_t leaf_stream = nullptr;
  cudaEvent_t leaf_ev[2] = {nullptr, nullptr};
  bool leaf_pending = false;
  std::vector<cudaEvent_t> ov_ev;
  std::vector<cudaEvent_t> prof_ev;      // 2 per launch
  std::vector<int32_t> prof_kind;
  std::vector<int32_t> prof_level;
  std::vector<double> prof_flops;
  std::vector<double> prof_bytes;
};

using htlr::Tree;

namespace {

// Gauss-Legendre nodes/weights on [0,1] (kernels.py:195-198 maps numpy's
// leggauss rule the same way); Newton on P_q.
void gauss01(int q, std::vector<double>& x, std::vector<double>& w) {
  x.resize(q);
  w.resize(q);
  for (int i = 0; i < q; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (q + 0.5));
    double pp = 0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= q; ++j) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = q * (z * p1 - p2) / (z * z - 1.0);
      double z1 = z;
      z = z1 - p1 / pp;
      if (std::fabs(z - z1) < 1e-17) break;
    }
    double p1 = 1.0, p2 = 0.0;
    for (int j = 1; j <= q; ++j) {
      double p3 = p2;
      p2 = p1;
      p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
    }
    pp = q * (z * p1 - p2) / (z * z - 1.0);
    double wt = 2.0 / ((1.0 - z * z) * pp * pp);
    x[i] = 0.5 * (-z + 1.0);   // ascending after the map
    w[i] = 0.5 * wt;
  }
}

int validate(const htlr_desc& ds, std::string& err) {
  if (ds.d != 2 && ds.d != 3) return err = "only d = 2 and d = 3 are supported", -1;
  if (ds.n < 1) return err = "n must be positive", -1;
  if (ds.rank < 1) return err = "rank must be positive", -1;
  if (ds.rank > htlr::kMaxRank) return err = "rank above the B200 kernel limit (16)", -1;
  if (ds.rule != 0 && ds.rule != 1) return err = "kind must be 'weak' or 'strong'", -1;
  if (ds.rule == 1 && !(ds.eta > 0)) return err = "strong admissibility needs eta > 0", -1;
  if (ds.kernel < 0 || ds.kernel > 2) return err = "unknown kernel kind", -1;
  if (ds.kernel == HTLR_KERNEL_GAUSSIAN && !(ds.sigma > 0)) return err = "gaussian kernel needs sigma > 0", -1;
  if (ds.kernel == HTLR_KERNEL_SLP2D && ds.d != 2) return err = "slp2d requires dimension 2", -1;
  if (ds.kernel == HTLR_KERNEL_SLP3D && ds.d != 3) return err = "slp3d requires dimension 3", -1;
  if (ds.quad_q < 2) return err = "quadrature order must be >= 2", -1;
  if (ds.quad_q > 64) return err = "quadrature order above 64", -1;
  return 0;
}

// Columns per work item.  The wide 128-row kernel takes 96 columns; a pass
// whose matrices have few (pair, rhs) columns each (the near-field of small
// grids, the coarse far-field levels) would leave two of its three column
// warp groups idle, so it gets the narrow 32-column variant instead, whose
// eight warps all work on the one 32-column slab.
int choose_nt(const Pass& ps, int R) {
  const int NT = htlr::gemm_nt(ps.MT);
  const double cols = (double)ps.npairs / std::max(1, ps.nmats) * std::min(R, NT);
  if (ps.MT < 0 && htlr::gemm_use_persistent()) {
    // thin passes: 8 or 16 columns per item when the matrices have few
    // pairs each (all 8 warps then split the rows of one or two n8 tiles)
    if (cols <= 8.0) return 8;
    return cols <= 16.0 ? 16 : NT;
  }
  if (ps.MT != 128 || !htlr::gemm_use_persistent()) return NT;
  if (cols < 48.0) return 32;
  // 64 or 96 columns per item: whichever wastes fewer column slots on the
  // pass's per-matrix pair counts (ties go to the 12-warp 96-column CTA)
  auto eff = [&](int nt) {
    const int rc = std::min(R, nt), npt = std::max(1, nt / rc);
    double useful = 0.0, cap = 0.0;
    for (int m = 0; m < ps.nmats; ++m) {
      const int cnt = ps.seg[m + 1] - ps.seg[m];
      useful += (double)cnt * R;
      cap += (double)((cnt + npt - 1) / npt) * ((R + rc - 1) / rc) * nt;
    }
    return cap > 0 ? useful / cap : 1.0;
  };
  return eff(64) > eff(96) + 0.005 ? 64 : 96;
}

// y-x sweep of the banded passes as two line kernels (all SMs) instead of the
// plane kernel (one SM per z-point plane): z-slab shards, whose slab has few
// planes (on one GPU the plane kernel is faster: 108 vs 136 us, config 4)
static bool band_xy_lines(const htlr_plan* pl) { return pl->zslab; }
// HTLR_FDIRECT=0: the leaf pass writes Y and the downward pass follows it
// (the formulation the parity tests cross-check the direct-f one against)
static bool fdirect_enabled() {
  const char* e = getenv("HTLR_FDIRECT");
  return !(e && e[0] == '0');
}

int make_tasks(Pass& ps, int R, std::vector<htlr::GemmTask>& out) {
  const int NT = choose_nt(ps, R);
  ps.task_nt[R] = NT;
  const int Rc = std::min(R, NT);
  const int npt = std::max(1, NT / Rc);
  const int nk = ps.K_pad / htlr::kKC;
  // one item = the whole K extent of its matrix (split-K items measured no
  // gain and would break the generated near blocks' two-slot generator ring,
  // which assumes every item spans >= STAGES ring stages)
  out.clear();
  for (int mat = 0; mat < ps.nmats; ++mat) {
    for (int b = ps.seg[mat]; b < ps.seg[mat + 1]; b += npt) {
      int cnt = std::min(npt, ps.seg[mat + 1] - b);
      for (int r0 = 0; r0 < R; r0 += Rc) out.push_back({mat, b, cnt, r0, 0, nk});
    }
  }
  return 0;
}

}  // namespace

extern "C" {

const char* htlr_last_error(void) { return g_last_error.c_str(); }

int htlr_plan_create(const htlr_desc* desc, int device, htlr_plan** out) {
  if (!desc || !out) return fail(-1, "null argument");
  std::string err;
  if (validate(*desc, err)) return fail(-1, err);
  int side = 0;
  if (htlr::compute_leaf_side(desc->n, desc->leaf_side_max, &side, err)) return fail(-1, err);
  if (device != -1) {   // -1: host-only plan (trees, lists, accounting; no device work)
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
      return fail(2, std::string("no CUDA device available: ") + cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(-1, "device index out of range");
  }
  htlr_plan* pl = new htlr_plan();
  pl->desc = *desc;
  pl->device = device;
  pl->d = desc->d;
  pl->n = desc->n;
  pl->p = desc->rank;
  pl->N = 1;
  for (int a = 0; a < pl->d; ++a) pl->N *= desc->n;
  pl->h = 1.0 / (double)desc->n;
  pl->hd = std::pow(pl->h, (double)pl->d);   // Python h**d
  if (desc->grid_kind != 0 && desc->grid_kind != 1) {
    delete pl;
    return fail(-1, "unknown grid kind");
  }
  pl->mapped = desc->grid_kind == 1;
  if (pl->mapped) htlr::mapped_tables(desc->n, desc->amplitude, pl->mb, pl->mx, pl->mc);
  {
    const char* e = std::getenv("HTLR_GRAPHS");   // HTLR_GRAPHS=0: direct launches (tests)
    pl->graphs = !(e && e[0] == '0');
  }
  pl->kp.kind = desc->kernel;
  pl->kp.denom = (2.0 * desc->sigma) * desc->sigma;
  pl->kp.scale = desc->scale;
  *out = pl;
  return 0;
}

int htlr_plan_destroy(htlr_plan* pl) {
  if (!pl) return 0;
  if (pl->device < 0) {
    delete pl;
    return 0;
  }
  cudaSetDevice(pl->device);
  for (auto e : pl->prof_ev) cudaEventDestroy(e);
  for (auto& g : pl->graph_cache) cudaGraphExecDestroy(g.exec);
  if (pl->cap_stream) cudaStreamDestroy(pl->cap_stream);
  if (pl->copy_stream) cudaStreamDestroy(pl->copy_stream);
  if (pl->side_stream) cudaStreamDestroy(pl->side_stream);
  for (auto& e : pl->side_ev)
    if (e) cudaEventDestroy(e);
  if (pl->fz_ev) cudaEventDestroy(pl->fz_ev);
  for (auto& e : pl->fd_ev)
    if (e) cudaEventDestroy(e);
  if (pl->leaf_stream) cudaStreamDestroy(pl->leaf_stream);
  for (auto& e : pl->leaf_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : pl->ov_ev) cudaEventDestroy(e);
  for (auto& lv : pl->levels) {
    lv.Q.release();
    lv.R.release();
    lv.W.release();
    lv.H.release();
    lv.nodes.release();
    lv.Kron.release();
    lv.Lm.release();
    lv.WLm.release();
    lv.d_ptr.release();
    lv.d_cols.release();
    lv.sym.release();
    lv.up_scratch.release();
    lv.up_count.release();
  }
  pl->d_mb.release();
  pl->d_mx.release();
  pl->d_mc.release();
  pl->dvec.release();
  pl->d_near_ptr.release();
  pl->d_near_cols.release();
  pl->near_sym.release();
  pl->d_self_ptr.release();
  pl->d_self_cols.release();
  pl->Vn.release();
  for (auto& ps : pl->passes) {
    ps.table.release();
    ps.pairs.release();
    for (auto& kv : ps.tasks) kv.second.first.release();
    ps.gen.release();
    ps.sep_tab.release();
    ps.sep_pairs.release();
    ps.sep_items.release();
    ps.sep_blocks.release();
    ps.sep_cols.release();
    ps.sep_gblocks.release();
    ps.sep_gcols.release();
    ps.band_ws.release();
  }
  pl->sep_corr.release();
  pl->diag.release();
  pl->coeff.release();
  pl->gl.release();
  pl->ub.release();
  pl->Y.release();
  pl->u_stage.release();
  pl->f_stage.release();
  delete pl;
  return 0;
}

static bool sep_wanted(const htlr_plan* pl);

// In-domain offsets of the banded terms per box position q along a line of nb
// boxes: A = C4's, B = {-2, 2}, M = {-1, 0, 1}, P = {3 - 6c} (htlr_band.cu)
struct BandLine {
  int A, B, M, P;
};
static BandLine band_line(int q, int nb) {
  const int c = q & 1;
  auto in = [&](int o) { return q + o >= 0 && q + o < nb; };
  BandLine v{0, in(-2) + in(2), in(-1) + in(0) + in(1), in(3 - 6 * c)};
  for (int o : {-4 - c, -3 - c, 4 - c, 5 - c}) v.A += in(o);
  return v;
}

// Analytic banded levels.  On a uniform grid with n a power of two the
// predicate is exactly a function of (level, |offset|) (htlr_lists.h
// offset_memo).  If on every level the inadmissible offsets are exactly
// {|o_a| <= 2} minus the corners {|o_a| = 2 for all a} (strong admissibility
// at eta = 1), then by induction over the levels the pairs the DFS reaches on
// level l are the in-domain children of such parent pairs, i.e. per axis the
// offsets R10 = {-4-c..5-c} minus the corner parents' children A4^3 -- the
// product sets the banded sweeps apply (band_check verifies the same
// statement pair by pair on a built list).  Plans that would run those levels
// as banded sweeps then need no pair lists below level 2: the DFS stops
// there, the leaf counts come from the product sets, and the full DFS list
// is built only when an export asks for it (ensure_leaves).
static bool analytic_bands_ok(const htlr_plan* pl, const htlr::TreeSpec& ts, int depth, int leaf_side) {
  const char* e = std::getenv("HTLR_SEP_BAND");
  if (e && e[0] == '0') return false;
  const char* e2 = std::getenv("HTLR_ANALYTIC");
  if (e2 && e2[0] == '0') return false;
  if (pl->mapped || pl->lowrank || pl->shard_world != 1 || pl->d != 3 || ts.rule != 1) return false;
  if (pl->kp.kind != HTLR_KERNEL_GAUSSIAN || pl->p != htlr::kSepP || leaf_side != htlr::kSepP) return false;
  const char* e3 = std::getenv("HTLR_SEPARABLE");
  if (e3 && e3[0] == '0') return false;
  if (depth < 3 || depth > 4) return false;   // band_check: banded passes on levels 3 and 4
  const std::vector<int8_t> memo = htlr::offset_memo(ts, depth);
  if (memo.empty()) return false;
  constexpr int K = htlr::kOffsetMemo;
  for (int l = 0; l <= depth; ++l) {
    const int m = 1 << l;
    for (int ox = 0; ox < K && ox < m; ++ox)
      for (int oy = 0; oy < K && oy < m; ++oy)
        for (int oz = 0; oz < K && oz < m; ++oz) {
          const bool nearshape = ox <= 2 && oy <= 2 && oz <= 2 && !(ox == 2 && oy == 2 && oz == 2);
          if ((memo[(((size_t)l * K + ox) * K + oy) * K + oz] == 0) != nearshape) return false;
        }
  }
  return true;
}

// leaf counts of an analytic level: admissible pairs (R10^3 - A4^3 - R5^3 +
// C2^3 in the domain) and, at the leaf level, near pairs (R5^3 - C2^3)
static void analytic_counts(int level, int64_t& adm, int64_t& near) {
  const int nb = 1 << level;
  int64_t s10 = 0, s4 = 0, s5 = 0, s2 = 0;
  for (int q = 0; q < nb; ++q) {
    const BandLine v = band_line(q, nb);
    s10 += v.A + v.B + v.M + v.P;
    s4 += v.A;
    s5 += v.B + v.M;
    s2 += v.B;
  }
  near = s5 * s5 * s5 - s2 * s2 * s2;
  adm = s10 * s10 * s10 - s4 * s4 * s4 - near;
}

// mode products the three sweeps of a banded pass run (per rhs) over the
// nt target boxes of a box region: the y sweep applies each term's band (28
// offsets away from the boundary at the leaf level); the z and x sweeps share
// band pieces between the terms (htlr_band.cu bcount / boff): z 15 (B, M, P,
// C4 and EB, EM once each), x 19 (C4 + P, M, B, C4 and EM, EB)
static double band_flops_of(int level, bool leaf, int64_t nt, double* z_share = nullptr) {
  const int nb = 1 << level;
  double per_line = 0, z_line = 0;
  for (int q = 0; q < nb; ++q) {
    const BandLine v = band_line(q, nb);
    const int nk = leaf ? 2 : 1;   // factor kinds with a {-2..2} and a {-2, 2} term
    const int ysw = (v.A + v.B + v.M + v.P) + v.A + nk * ((v.B + v.M) + v.B);
    const int zsw = v.A + v.P + nk * (v.B + v.M);
    const int xsw = (v.A + v.P) + v.A + nk * (v.M + v.B);
    per_line += ysw + zsw + xsw;
    z_line += zsw;
  }
  if (z_share) *z_share = z_line / per_line;
  // the region's share of the sweeps (halo lines of the z sweep not counted)
  return (double)nb * nb * per_line * 2.0 * 4096.0 * (double)nt / (double)((int64_t)1 << (3 * level));
}

// the full DFS leaf list of a plan whose tree stopped above its analytic levels
static int ensure_leaves(const htlr_plan* cpl) {
  htlr_plan* pl = const_cast<htlr_plan*>(cpl);
  if (!pl->tree.truncated) return 0;
  htlr::Tree full;
  std::string err;
  if (htlr::build_tree(pl->tree.spec, full, err)) return fail(-1, err);
  if (full.num_adm != pl->tree.num_adm || full.num_near != pl->tree.num_near)
    return fail(2, "analytic banded levels: leaf counts differ from the DFS list");
  pl->tree.leaves.swap(full.leaves);
  pl->tree.truncated = false;
  return 0;
}

int htlr_build_lists(htlr_plan* pl) {
  if (!pl) return fail(-1, "null plan");
  htlr::TreeSpec ts;
  ts.d = pl->d;
  ts.n = pl->n;
  ts.leaf_side_max = pl->desc.leaf_side_max;
  ts.rule = pl->desc.rule;
  ts.eta = pl->desc.eta;
  if (pl->mapped) ts.bounds = pl->mb;
  std::string err;
  PhaseTimer tm;
  pl->analytic_from = 0;
  {
    int side = 0, depth = 0;
    if (pl->n >= 1 && htlr::compute_leaf_side(ts.n, ts.leaf_side_max, &side, err) == 0) {
      for (int sd = ts.n; sd > side; sd /= 2) ++depth;
      if (analytic_bands_ok(pl, ts, depth, side)) pl->analytic_from = 3;
    }
    err.clear();
  }
  if (htlr::build_tree(ts, pl->tree, err, pl->analytic_from ? pl->analytic_from - 1 : -1)) return fail(-1, err);
  tm.mark("lists: tree (DFS)");
  const Tree& tr = pl->tree;
  pl->L = tr.depth;
  pl->sL = tr.leaf_side;
  const int d = pl->d, p = pl->p;
  pl->levels.assign(pl->L + 1, Level());
  for (int l = 0; l <= pl->L; ++l) {
    Level& lv = pl->levels[l];
    lv.level = l;
    lv.side = tr.side(l);
    lv.m = tr.clusters_per_dim(l);
    lv.nclusters = 1;
    for (int a = 0; a < d; ++a) lv.nclusters *= lv.m;
  }
  pl->near = OffsetTable();
  pl->num_near = 0;
  const int world = pl->shard_world, rank = pl->shard_rank;
  pl->own_lo.assign(pl->L + 1, 0);
  pl->own_hi.assign(pl->L + 1, 0);
  for (int l = 0; l <= pl->L; ++l) {
    const int64_t M = pl->levels[l].nclusters;
    if (M % world == 0) {
      pl->own_lo[l] = M / world * rank;
      pl->own_hi[l] = M / world * (rank + 1);
    } else {
      pl->own_lo[l] = pl->own_hi[l] = -1;   // level cannot be split evenly
    }
  }
  if (pl->own_lo[pl->L] < 0)
    return fail(-1, "the leaf level has fewer boxes than shards (or not a multiple of them)");
  auto key_range = [&](int m) {
    int64_t r = 1;
    for (int a = 0; a < d; ++a) r *= 2 * m + 1;
    return r;
  };
  for (int l = 0; l <= pl->L; ++l)
    if (key_range(pl->levels[l].m) <= (1 << 22)) pl->levels[l].adm.dense.assign(key_range(pl->levels[l].m), 0);
  if (key_range(pl->levels[pl->L].m) <= (1 << 22)) pl->near.dense.assign(key_range(pl->levels[pl->L].m), 0);
  // Offset tables.  (1, all cores) per leaf: its packed offset key and, for
  // sharded plans, whether its target is owned; (2, sequential, DFS order)
  // offset ids in order of first appearance -- the only order-dependent step,
  // a tight loop over the keys; (3, all cores) per-chunk counts per id, then
  // every chunk writes its (target, source) Morton ids at precomputed
  // positions of the pre-sized member lists (no shared counters).  The order
  // inside a member list is not kept: every consumer sorts it.
  const size_t nlf = tr.leaves.size();
  const size_t ntab = pl->levels.size() + 1;   // adm per level, then near
  if (pl->mapped) {
    // Mapped grids regenerate their blocks: no offset tables, only the CSR of
    // the own targets per level and of the near field (sources sorted by
    // Morton id), built straight from the leaves: per-chunk counts per
    // (table, target row), an exclusive prefix over (row, chunk), then every
    // chunk writes its sources at its own positions (all cores, no atomics).
    std::vector<int64_t> rbase(ntab + 1, 0);   // first row of each table in the concatenated row space
    auto tlevel = [&](size_t t) { return t + 1 < ntab ? (int)t : pl->L; };
    for (size_t t = 0; t < ntab; ++t) {
      const int l = tlevel(t);
      rbase[t + 1] = rbase[t] + (pl->own_lo[l] < 0 ? 0 : pl->own_hi[l] - pl->own_lo[l]);
    }
    const int64_t nrows = rbase[ntab];
    const size_t chunk = 1 << 15, nchunks = (nlf + chunk - 1) / chunk;
    std::vector<std::vector<int>> cnt(nchunks, std::vector<int>((size_t)nrows, 0));
    std::vector<std::vector<int64_t>> lcount(nchunks, std::vector<int64_t>(ntab, 0));
    std::atomic<bool> bad_level{false};
    auto row_of = [&](const htlr::LeafRec& lf) -> int64_t {   // -1: not an own target
      const size_t t = lf.kind == 0 ? (size_t)lf.level : ntab - 1;
      if (pl->own_lo[lf.level] < 0) return -2;
      const int64_t tl = htlr::morton_encode(lf.tc, d, lf.level);
      if (tl < pl->own_lo[lf.level] || tl >= pl->own_hi[lf.level]) return -1;
      return rbase[t] + tl - pl->own_lo[lf.level];
    };
    parallel_for(nchunks, [&](size_t c) {
      const size_t e = std::min(nlf, (c + 1) * chunk);
      for (size_t i = c * chunk; i < e; ++i) {
        const auto& lf = tr.leaves[i];
        lcount[c][lf.kind == 0 ? (size_t)lf.level : ntab - 1]++;
        const int64_t r = row_of(lf);
        if (r == -2) bad_level = true;
        if (r >= 0) cnt[c][(size_t)r]++;
      }
    });
    if (bad_level) return fail(-1, "admissible blocks on a level with fewer clusters than shards");
    for (size_t c = 0; c < nchunks; ++c) {
      for (size_t t = 0; t + 1 < ntab; ++t) pl->levels[t].num_adm += lcount[c][t];
      pl->num_near += lcount[c][ntab - 1];
    }
    std::vector<int64_t> rptr((size_t)nrows + 1, 0);
    {
      int64_t acc = 0;
      for (int64_t r = 0; r < nrows; ++r) {
        rptr[(size_t)r] = acc;
        for (size_t c = 0; c < nchunks; ++c) {
          const int v = cnt[c][(size_t)r];
          cnt[c][(size_t)r] = (int)(acc - rptr[(size_t)r]);   // offset inside the row
          acc += v;
        }
      }
      rptr[(size_t)nrows] = acc;
    }
    std::vector<int> cols((size_t)rptr[(size_t)nrows]);
    parallel_for(nchunks, [&](size_t c) {
      const size_t e = std::min(nlf, (c + 1) * chunk);
      for (size_t i = c * chunk; i < e; ++i) {
        const auto& lf = tr.leaves[i];
        const int64_t r = row_of(lf);
        if (r >= 0) cols[(size_t)(rptr[(size_t)r] + cnt[c][(size_t)r]++)] = (int)htlr::morton_encode(lf.sc, d, lf.level);
      }
    });
    parallel_for((size_t)nrows, [&](size_t r) { std::sort(cols.begin() + rptr[r], cols.begin() + rptr[r + 1]); });
    tm.mark("lists: mapped CSR (from the leaves)");
    for (const auto& lv : pl->levels) {
      if (lv.num_adm > 0 && lv.side < p) {
        char buf[128];
        snprintf(buf, sizeof buf, "qr requires rows >= cols, got shape (%d, %d)", lv.side, p);
        return fail(-1, buf);
      }
    }
    if (ipow(pl->sL, d) > 4096) return fail(-1, "leaf boxes above 4096 points are not supported by the B200 path");
    if (ipow(p, d) > 4096) return fail(-1, "rank^d above 4096 is not supported by the B200 path");
    pl->passes.clear();
    auto slice = [&](size_t t, std::vector<int64_t>& ptr, std::vector<int>& out) {
      const int64_t r0 = rbase[t], r1 = rbase[t + 1];
      ptr.assign((size_t)(r1 - r0) + 1, 0);
      for (int64_t r = r0; r <= r1; ++r) ptr[(size_t)(r - r0)] = rptr[(size_t)r] - rptr[(size_t)r0];
      out.assign(cols.begin() + rptr[(size_t)r0], cols.begin() + rptr[(size_t)r1]);
    };
    for (int l = 0; l <= pl->L; ++l) {
      Level& lv = pl->levels[l];
      lv.needs_up = lv.num_adm > 0;
      if (lv.needs_up) slice((size_t)l, lv.csr_ptr, lv.csr_cols);
    }
    slice(ntab - 1, pl->near_ptr, pl->near_cols);
    if (pl->sL > 16) return fail(-1, "mapped grids support leaf sides up to 16");
    pl->merged = false;
    pl->lists_built = true;
    pl->constructed = false;
    return 0;
  }
  std::vector<OffsetTable*> tabs;
  for (auto& lv : pl->levels) tabs.push_back(&lv.adm);
  tabs.push_back(&pl->near);
  std::vector<int64_t> keys(nlf);
  std::vector<int> lid(nlf);
  std::vector<char> own(nlf, 1);
  const size_t chunk = 1 << 15;
  const size_t nchunks = (nlf + chunk - 1) / chunk;
  std::atomic<bool> bad_level{false};
  parallel_for(nchunks, [&](size_t c) {
    const size_t e = std::min(nlf, (c + 1) * chunk);
    for (size_t i = c * chunk; i < e; ++i) {
      const auto& lf = tr.leaves[i];
      keys[i] = pack_offset(lf.tc, lf.sc, d, pl->levels[lf.level].m);
      if (world > 1) {
        if (pl->own_lo[lf.level] < 0) {
          bad_level = true;
          continue;
        }
        const int64_t tl = htlr::morton_encode(lf.tc, d, lf.level);
        own[i] = tl >= pl->own_lo[lf.level] && tl < pl->own_hi[lf.level];
      }
    }
  });
  if (bad_level) return fail(-1, "admissible blocks on a level with fewer clusters than shards");
  tm.mark("lists: offset keys");
  bool all_dense = true;
  for (auto* t : tabs) all_dense = all_dense && !t->dense.empty();
  if (all_dense) {
    // (2) in parallel: every chunk lists its leaves whose key is new to the
    // chunk (bitmaps per table), in index order; merged chunk by chunk, the
    // first occurrence of every key gets the next id -- the same ids as the
    // sequential pass; then lid[] and the per-level counts in parallel.
    auto tab_of = [&](size_t i) {
      const auto& lf = tr.leaves[i];
      return lf.kind == 0 ? (size_t)lf.level : ntab - 1;
    };
    std::vector<std::vector<size_t>> cand(nchunks);
    parallel_for(nchunks, [&](size_t c) {
      std::vector<std::vector<char>> seen(ntab);
      const size_t e = std::min(nlf, (c + 1) * chunk);
      for (size_t i = c * chunk; i < e; ++i) {
        const size_t t = tab_of(i);
        if (seen[t].empty()) seen[t].assign(tabs[t]->dense.size(), 0);
        char& f = seen[t][keys[i]];
        if (!f) {
          f = 1;
          cand[c].push_back(i);
        }
      }
    });
    for (size_t c = 0; c < nchunks; ++c)
      for (size_t i : cand[c]) {
        OffsetTable& tab = *tabs[tab_of(i)];
        int& slot = tab.dense[keys[i]];
        if (slot == 0) {
          slot = (int)tab.rep.size() + 1;
          const auto& lf = tr.leaves[i];
          tab.rep.push_back({lf.tc[0], lf.tc[1], lf.tc[2], lf.sc[0], lf.sc[1], lf.sc[2]});
        }
      }
    std::vector<std::vector<int64_t>> lcount(nchunks, std::vector<int64_t>(ntab, 0));
    parallel_for(nchunks, [&](size_t c) {
      const size_t e = std::min(nlf, (c + 1) * chunk);
      for (size_t i = c * chunk; i < e; ++i) {
        const size_t t = tab_of(i);
        lid[i] = tabs[t]->dense[keys[i]] - 1;
        lcount[c][t]++;
      }
    });
    for (size_t c = 0; c < nchunks; ++c) {
      for (size_t t = 0; t + 1 < ntab; ++t) pl->levels[t].num_adm += lcount[c][t];
      pl->num_near += lcount[c][ntab - 1];
    }
  }
  for (size_t i = 0; i < nlf && !all_dense; ++i) {
    const auto& lf = tr.leaves[i];
    OffsetTable& tab = lf.kind == 0 ? pl->levels[lf.level].adm : pl->near;
    const int64_t key = keys[i];
    int id = -1;
    if (!tab.dense.empty()) {
      id = tab.dense[key] - 1;
    } else {
      auto it = tab.id.find(key);
      if (it != tab.id.end()) id = it->second;
    }
    if (id < 0) {
      id = (int)tab.rep.size();
      if (!tab.dense.empty())
        tab.dense[key] = id + 1;
      else
        tab.id.emplace(key, id);
      tab.rep.push_back({lf.tc[0], lf.tc[1], lf.tc[2], lf.sc[0], lf.sc[1], lf.sc[2]});
    }
    lid[i] = id;
    if (lf.kind == 0)
      pl->levels[lf.level].num_adm++;
    else
      pl->num_near++;
  }
  tm.mark("lists: offset ids");
  {
    // global id = base[table] + id
    std::vector<int> base(ntab + 1, 0);
    for (size_t t = 0; t < ntab; ++t) base[t + 1] = base[t] + (int)tabs[t]->rep.size();
    const int nid = base[ntab];
    auto gid = [&](size_t i) {
      const auto& lf = tr.leaves[i];
      return base[lf.kind == 0 ? (size_t)lf.level : ntab - 1] + lid[i];
    };
    std::vector<std::vector<int>> cnt(nchunks, std::vector<int>(nid, 0));
    parallel_for(nchunks, [&](size_t c) {
      const size_t e = std::min(nlf, (c + 1) * chunk);
      for (size_t i = c * chunk; i < e; ++i)
        if (own[i]) cnt[c][gid(i)]++;
    });
    // exclusive prefix over chunks, per id; sizes of the member lists
    std::vector<int> total(nid, 0);
    for (size_t c = 0; c < nchunks; ++c)
      for (int g = 0; g < nid; ++g) {
        const int v = cnt[c][g];
        cnt[c][g] = total[g];
        total[g] += v;
      }
    std::vector<std::pair<int, int>*> dst(nid);
    for (size_t t = 0; t < ntab; ++t) {
      tabs[t]->members.assign(tabs[t]->rep.size(), {});
      for (size_t k = 0; k < tabs[t]->rep.size(); ++k) {
        auto& m = tabs[t]->members[k];
        m.resize((size_t)total[base[t] + (int)k]);
        dst[base[t] + (int)k] = m.data();
      }
    }
    parallel_for(nchunks, [&](size_t c) {
      const size_t e = std::min(nlf, (c + 1) * chunk);
      for (size_t i = c * chunk; i < e; ++i) {
        if (!own[i]) continue;
        const auto& lf = tr.leaves[i];
        const int g = gid(i);
        dst[g][cnt[c][g]++] = std::make_pair((int)htlr::morton_encode(lf.tc, d, lf.level),
                                             (int)htlr::morton_encode(lf.sc, d, lf.level));
      }
    });
  }
  tm.mark("lists: offset tables");
  for (int l = pl->analytic_from; pl->analytic_from && l <= pl->L; ++l) {
    int64_t adm = 0, near = 0;
    analytic_counts(l, adm, near);
    pl->levels[l].num_adm = adm;
    pl->tree.num_adm += adm;
    if (l == pl->L) {
      pl->num_near = near;
      pl->tree.num_near += near;
    }
  }
  // validation the reference performs at build time (tensor.py:112-113 via
  // blocks.py:160): admissible blocks need box side >= rank
  for (const auto& lv : pl->levels) {
    if (lv.num_adm > 0 && lv.side < p) {
      char buf[128];
      snprintf(buf, sizeof buf, "qr requires rows >= cols, got shape (%d, %d)", lv.side, p);
      return fail(-1, buf);
    }
  }
  const int PL = ipow(pl->sL, d);
  const int P = ipow(p, d);
  if (PL > 4096) return fail(-1, "leaf boxes above 4096 points are not supported by the B200 path");
  if (P > 4096) return fail(-1, "rank^d above 4096 is not supported by the B200 path");
  pl->passes.clear();
  pl->merged = pl->levels[pl->L].num_adm > 0 && pl->sL == p;
  // passes
  auto fill_pass = [&](Pass& ps, std::vector<const OffsetTable*> tabs) {
    ps.MT = htlr::gemm_mt_for(ps.P);
    ps.M_pad = ps.MT < 0 ? -ps.MT : round_up(ps.P, ps.MT);
    ps.K_pad = round_up(ps.P, htlr::kKC);
    ps.RT = ps.MT < 0 ? 1 : ps.M_pad / ps.MT;
    ps.mat_stride = (int64_t)ps.M_pad * ps.K_pad;
    ps.seg.assign(1, 0);
    std::vector<const std::vector<std::pair<int, int>>*> mems;
    for (const OffsetTable* tab : tabs)
      for (const auto& mem : tab->members) {
        mems.push_back(&mem);
        ps.seg.push_back(ps.seg.back() + (int)mem.size());
      }
    // every matrix's pairs sorted by (target, source), matrices in parallel
    std::vector<int2> pr((size_t)ps.seg.back());
    parallel_for(mems.size(), [&](size_t i) {
      std::vector<std::pair<int, int>> v = *mems[i];
      std::sort(v.begin(), v.end());
      int2* o = pr.data() + ps.seg[i];
      for (size_t k = 0; k < v.size(); ++k) o[k] = make_int2(v[k].first, v[k].second);
    });
    ps.nmats = (int)ps.seg.size() - 1;
    ps.npairs = (int)pr.size();
    ps.pairs_host.swap(pr);
    return 0;
  };
  for (int l = 0; l <= pl->L; ++l) {
    Level& lv = pl->levels[l];
    lv.needs_up = lv.num_adm > 0 && !(l == pl->L && pl->merged);
    if (!lv.needs_up) continue;
    pl->passes.emplace_back();
    Pass& ps = pl->passes.back();
    ps.level = l;
    ps.P = P;
    ps.from_ub = false;
    ps.to_y = false;
    if (fill_pass(ps, {&lv.adm})) return 1;
    if (pl->analytic_from && l >= pl->analytic_from) {
      ps.analytic = true;
      ps.npairs = (int)lv.num_adm;
    }
  }
  pl->passes.emplace_back();
  pl->leaf_pass = (int)pl->passes.size() - 1;
  {
    Pass& ps = pl->passes.back();
    ps.level = pl->L;
    ps.P = PL;
    ps.from_ub = true;
    ps.to_y = true;
    std::vector<const OffsetTable*> tabs = {&pl->near};
    if (pl->merged) tabs.push_back(&pl->levels[pl->L].adm);
    pl->near_mats = (int)pl->near.members.size();
    if (fill_pass(ps, tabs)) return 1;
    if (pl->analytic_from) {
      ps.analytic = true;
      ps.npairs = (int)(pl->num_near + (pl->merged ? pl->levels[pl->L].num_adm : 0));
    }
  }
  tm.mark("lists: passes (sorted pairs)");
  pl->lists_built = true;
  pl->constructed = false;
  return 0;
}

int htlr_set_lowrank(htlr_plan* pl, int32_t on) {
  if (!pl) return fail(-1, "null plan");
  if (pl->constructed) return fail(-1, "select the representation before construct");
  if (on && pl->mapped) return fail(-1, "the H-matrix baseline is built for uniform grids only");
  pl->lowrank = on != 0;
  return 0;
}

int htlr_set_shard(htlr_plan* pl, int32_t rank, int32_t world) {
  if (!pl) return fail(-1, "null plan");
  if (world < 1 || rank < 0 || rank >= world) return fail(-1, "invalid shard rank/world");
  if (world & (world - 1)) return fail(-1, "the number of shards must be a power of two");
  if (pl->constructed) return fail(-1, "set the shard before construct");
  pl->shard_rank = rank;
  pl->shard_world = world;
  pl->lists_built = false;
  return 0;
}

static void drop_graphs(htlr_plan* pl);

int htlr_set_zslab(htlr_plan* pl, int32_t rank, int32_t world) {
  if (!pl) return fail(-1, "null plan");
  if (world < 1 || rank < 0 || rank >= world) return fail(-1, "invalid shard rank/world");
  if (!pl->constructed) return fail(-1, "construct the plan before setting its z-slab");
  if (pl->shard_world != 1) return fail(-1, "z-slab shards need an unsharded plan (no htlr_set_shard)");
  if (!pl->sep || pl->d != 3 || !pl->passes[pl->leaf_pass].band)
    return fail(-1, "z-slab shards need the banded separable formulation (3-D Gaussian, eta = 1, p = leaf side = 8)");
  const int M = 1 << pl->L;
  if (M % world || (M / world) % 2) return fail(-1, "z-slab shards: 2^L / world must be even");
  drop_graphs(pl);
  pl->zslab = world > 1;
  pl->zs_rank = rank;
  pl->zs_world = world;
  pl->zs_lo = M / world * rank;
  pl->zs_hi = M / world * (rank + 1);
  // each banded pass covers the z range of its level that holds the own leaf
  // boxes (coarse levels shared by several shards are computed by each)
  for (auto& ps : pl->passes) {
    if (!ps.band) continue;
    const int s = pl->L - ps.level, nb = 1 << ps.level;
    for (int a = 0; a < 3; ++a) ps.band_lo[a] = 0, ps.band_hi[a] = nb;
    if (world > 1) {
      ps.band_lo[2] = pl->zs_lo >> s;
      ps.band_hi[2] = (pl->zs_hi + (1 << s) - 1) >> s;
    }
  }
  return 0;
}

int htlr_exchange_kind(const htlr_plan* pl) {
  if (!pl) return fail(-1, "null plan");
  return pl->zslab ? 1 : 0;
}

int htlr_shard_info(const htlr_plan* pl, int64_t* own_leaf_lo, int64_t* own_leaf_hi, int64_t* own_pairs,
                    double* own_flops) {
  if (!pl) return fail(-1, "null plan");
  if (!pl->lists_built) return fail(-1, "lists not built");
  int64_t pairs = 0;
  double fl = 0.0;
  for (const auto& ps : pl->passes) {
    pairs += ps.npairs;
    fl += 2.0 * (double)ps.P * ps.P * ps.npairs;
  }
  if (pl->mapped) {
    const double P = ipow(pl->p, pl->d), PL = ipow(pl->sL, pl->d);
    for (const auto& lv : pl->levels) {
      pairs += (int64_t)lv.csr_cols.size();
      fl += 2.0 * P * P * (double)lv.csr_cols.size();
    }
    pairs += (int64_t)pl->near_cols.size();
    fl += 2.0 * PL * PL * (double)pl->near_cols.size();
  }
  if (own_leaf_lo) *own_leaf_lo = pl->own_lo[pl->L];
  if (own_leaf_hi) *own_leaf_hi = pl->own_hi[pl->L];
  if (own_pairs) *own_pairs = pairs;
  if (own_flops) *own_flops = fl;
  return 0;
}

static void exchange_sizes(const htlr_plan* pl, int R, std::vector<int64_t>& bytes) {
  bytes.clear();
  if (pl->mapped) {
    const int P = ipow(pl->p, pl->d), PL = ipow(pl->sL, pl->d);
    bytes.push_back(pl->levels[pl->L].nclusters * (int64_t)R * PL * (int64_t)sizeof(double));
    for (const auto& lv : pl->levels)
      if (lv.needs_up) bytes.push_back(lv.nclusters * (int64_t)R * P * (int64_t)sizeof(double));
    return;
  }
  const Pass& lp = pl->passes[pl->leaf_pass];
  if (!pl->zslab)   // z-slab shards read u itself: only the W_l are exchanged (summed)
    bytes.push_back(pl->levels[pl->L].nclusters * (int64_t)R * lp.K_pad * (int64_t)sizeof(double));
  for (const auto& ps : pl->passes) {
    if (ps.to_y) continue;
    bytes.push_back(pl->levels[ps.level].nclusters * (int64_t)R * ps.K_pad * (int64_t)sizeof(double));
  }
}

int htlr_exchange_info(const htlr_plan* pl, int64_t nrhs, int64_t* count, int64_t* bytes, int64_t cap) {
  if (!pl || !count) return fail(-1, "null argument");
  if (!pl->lists_built) return fail(-1, "lists not built");
  std::vector<int64_t> b;
  exchange_sizes(pl, (int)nrhs, b);
  *count = (int64_t)b.size();
  if (bytes) {
    if (cap < (int64_t)b.size()) return fail(-1, "exchange info buffer too small");
    for (size_t i = 0; i < b.size(); ++i) bytes[i] = b[i];
  }
  return 0;
}

static void drop_graphs(htlr_plan* pl);

int htlr_bind_exchange(htlr_plan* pl, int64_t nrhs, void* const* ptrs, int64_t count) {
  if (!pl) return fail(-1, "null plan");
  drop_graphs(pl);
  if (!pl->lists_built) return fail(-1, "lists not built");
  std::vector<int64_t> b;
  exchange_sizes(pl, (int)nrhs, b);
  if (!ptrs || count == 0) {
    pl->ext_R = 0;
    pl->ext_ptrs.clear();
    return 0;
  }
  if (count != (int64_t)b.size()) return fail(-1, "exchange buffer count mismatch");
  pl->ext_ptrs.assign(count, nullptr);
  for (int64_t i = 0; i < count; ++i) {
    if (!ptrs[i]) return fail(-1, "null exchange buffer");
    pl->ext_ptrs[i] = static_cast<double*>(ptrs[i]);
  }
  pl->ext_R = (int)nrhs;
  return 0;
}

int htlr_tree_info(const htlr_plan* pl, int32_t* depth, int32_t* leaf_side, int64_t* num_leaves,
                   int64_t* num_adm, int64_t* num_near) {
  if (!pl) return fail(-1, "null plan");
  if (!pl->lists_built) return fail(-1, "lists not built");
  if (depth) *depth = pl->tree.depth;
  if (leaf_side) *leaf_side = pl->tree.leaf_side;
  if (num_leaves) *num_leaves = pl->tree.truncated ? pl->tree.num_adm + pl->tree.num_near : (int64_t)pl->tree.leaves.size();
  if (num_adm) *num_adm = pl->tree.num_adm;
  if (num_near) *num_near = pl->tree.num_near;
  return 0;
}

int htlr_export_lists(const htlr_plan* pl, int32_t* rows, int64_t cap) {
  if (!pl || !rows) return fail(-1, "null argument");
  if (!pl->lists_built) return fail(-1, "lists not built");
  if (int rc = ensure_leaves(pl)) return rc;
  const int d = pl->d, w = 3 + 4 * d;
  const auto& lv = pl->tree.leaves;
  if (cap < (int64_t)lv.size() * w) return fail(-1, "export buffer too small");
  for (size_t i = 0; i < lv.size(); ++i) {
    int32_t* r = rows + i * w;
    const int side = pl->tree.side(lv[i].level);
    r[0] = (int32_t)i;
    r[1] = lv[i].kind;
    r[2] = lv[i].level;
    for (int a = 0; a < d; ++a) {
      r[3 + 2 * a] = lv[i].tc[a] * side;
      r[4 + 2 * a] = lv[i].tc[a] * side + side;
      r[3 + 2 * d + 2 * a] = lv[i].sc[a] * side;
      r[4 + 2 * d + 2 * a] = lv[i].sc[a] * side + side;
    }
  }
  return 0;
}

int htlr_set_coeff(htlr_plan* pl, const double* a_host) {
  if (!pl) return fail(-1, "null plan");
  if (pl->device < 0) return fail(-1, "host-only plan: no device work");
  CUDA_TRY(cudaSetDevice(pl->device));
  if (!a_host) {
    pl->has_coeff = false;
    return 0;
  }
  if (pl->coeff.alloc(pl->N * sizeof(double))) return 1;
  CUDA_TRY(cudaMemcpy(pl->coeff.ptr, a_host, pl->N * sizeof(double), cudaMemcpyHostToDevice));
  pl->has_coeff = true;
  return 0;
}

static int upload(DevBuf& buf, const void* src, size_t bytes) {
  if (buf.alloc(std::max<size_t>(bytes, 8))) return 1;
  if (bytes) CUDA_TRY(cudaMemcpy(buf.ptr, src, bytes, cudaMemcpyHostToDevice));
  return 0;
}

// Pair lists of the symmetric regeneration.  Every unordered pair {a, b}
// (a < b) is evaluated once, by the CTA of its owning endpoint: a when a + b
// is even, else b -- about half of every row's list, so rows (and shards)
// stay balanced.  `ptr`/`cols` is the CSR of the own rows [t0, t0 + rows);
// self pairs (near field) are returned separately for the one-sided kernel.
// `full` (unsharded plans) lets the symmetry of the lists be checked; a
// non-symmetric list leaves the symmetric path off.
static bool pair_owner_is_row(int64_t row, int64_t other) {
  const int64_t a = std::min(row, other), b = std::max(row, other);
  return (((a + b) & 1) == 0) ? row == a : row == b;
}

static int build_sym(const std::vector<int64_t>& ptr, const std::vector<int>& cols, int64_t t0, bool full,
                     SymList& out, std::vector<int64_t>* self_ptr, std::vector<int>* self_cols) {
  out.release();
  const int64_t nrows = (int64_t)ptr.size() - 1;
  // pass 1 (rows in parallel): owned / self counts, symmetry check
  std::vector<int64_t> up(nrows + 1, 0), sp(nrows + 1, 0);
  std::atomic<bool> ok{true};
  parallel_for((size_t)nrows, [&](size_t r) {
    const int64_t t = t0 + (int64_t)r;
    int64_t nu = 0, ns = 0;
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
      const int sg = cols[e];
      if (full) {   // symmetry: tau must appear in sigma's (sorted) list
        if (sg < 0 || sg >= nrows ||
            !std::binary_search(cols.begin() + ptr[sg], cols.begin() + ptr[sg + 1], (int)t)) {
          ok = false;
          return;
        }
      }
      if (sg == t)
        ++ns;
      else if (pair_owner_is_row(t, sg))
        ++nu;
    }
    up[r + 1] = nu;
    sp[r + 1] = ns;
  });
  if (!ok) return 0;
  for (int64_t r = 0; r < nrows; ++r) {
    up[r + 1] += up[r];
    sp[r + 1] += sp[r];
  }
  if (sp[nrows] > 0 && !self_cols) return 0;
  std::vector<int> uc((size_t)up[nrows]);
  if (self_ptr) *self_ptr = sp;
  if (self_cols) self_cols->assign((size_t)sp[nrows], 0);
  // pass 2: fill (sources stay in CSR order)
  parallel_for((size_t)nrows, [&](size_t r) {
    const int64_t t = t0 + (int64_t)r;
    int64_t ku = up[r], ks = sp[r];
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
      const int sg = cols[e];
      if (sg == t)
        (*self_cols)[ks++] = sg;
      else if (pair_owner_is_row(t, sg))
        uc[ku++] = sg;
    }
  });
  std::vector<int> order(nrows);
  for (int64_t r = 0; r < nrows; ++r) order[r] = (int)r;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return up[a + 1] - up[a] > up[b + 1] - up[b]; });
  if (upload(out.uptr, up.data(), up.size() * sizeof(int64_t))) return 1;
  if (upload(out.ucols, uc.data(), std::max<size_t>(1, uc.size()) * sizeof(int))) return 1;
  if (upload(out.order, order.data(), order.size() * sizeof(int))) return 1;
  out.nrows = nrows;
  out.on = true;
  return 0;
}

// near-only leaf passes with Toeplitz near blocks generate their A fragments
// from the 15^3 generators (config 2: 80 -> 73 us against streaming the blocks)
static bool near_gen_enabled() { return true; }

static bool regen_sym_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("HTLR_REGEN_SYM");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// HTLR_SEP_BLOCK=0: passes by per-warp items instead of the cooperative
// per-parent CTAs (A/B runs, tests)
static bool sep_block_enabled(bool leaf) {
  const char* e = std::getenv("HTLR_SEP_BLOCK");
  if (e && e[0] == '0') return false;
  if (e && e[0] == 'l') return leaf;     // "leaf": cooperative leaf pass only
  if (e && e[0] == 'v') return !leaf;    // "levels": cooperative level passes only
  return true;
}

// Cooperative layout of a pass: per parent cluster (8 consecutive Morton
// targets), the union of its children's sources grouped into columns of equal
// (x, y) box coordinates, each box with the pair code of every child (or
// 0xFFFF); columns split into parts of <= HTLR_SEP_COLS (default: ~16 parts
// per SM, <= 12 columns), parts ordered by decreasing work.  Leaves the pass on per-warp items when a
// column is longer than kSepColMax or the own range is not whole parents.
// The self pair of a target is its near-field (kind 1) pair with itself.  The
// target can also be another sibling's source (e.g. weak admissibility makes
// adjacent siblings admissible), with no pair of its own -- code 0xFFFF.
static bool is_self_code(unsigned short code) { return code != 0xFFFF && (code >> 12) == 1; }

static int build_sep_blocks(htlr_plan* pl, Pass& ps, const std::vector<int64_t>& ptr, const std::vector<int2>& ent) {
  const int L = ps.level;
  const int64_t t0 = pl->own_lo[L], nt = pl->own_hi[L] - t0;
  if (t0 % 8 || nt % 8 || pl->d != 3) return 0;
  const int64_t npar = nt / 8;
  std::vector<std::vector<htlr::SepCol>> pcols((size_t)npar);
  std::vector<std::vector<int>> pself((size_t)npar);
  std::atomic<bool> ok{true};
  parallel_for((size_t)npar, [&](size_t P) {
    // (source coords, source id) -> per-child codes; sources indexed through a
    // dense array over their bounding box
    struct Src {
      int x, y, z, id;
      unsigned short code[8];
    };
    int lo[3] = {1 << 30, 1 << 30, 1 << 30}, hi[3] = {-1, -1, -1};
    for (int64_t k = ptr[(int64_t)P * 8]; k < ptr[(int64_t)P * 8 + 8]; ++k) {
      int c[3];
      htlr::morton_decode(ent[k].x, 3, L, c);
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], c[a]);
        hi[a] = std::max(hi[a], c[a]);
      }
    }
    std::vector<Src> v;
    if (hi[0] < 0) {
      pself[P].assign(8, -1);
      return;
    }
    const int ex = hi[0] - lo[0] + 1, ey = hi[1] - lo[1] + 1, ez = hi[2] - lo[2] + 1;
    std::vector<int> at((size_t)ex * ey * ez, -1);
    for (int w = 0; w < 8; ++w) {
      const int64_t t = (int64_t)P * 8 + w;
      for (int64_t k = ptr[t]; k < ptr[t + 1]; ++k) {
        const int src = ent[k].x;
        int c[3];
        htlr::morton_decode(src, 3, L, c);
        int& slot = at[((size_t)(c[2] - lo[2]) * ey + (c[1] - lo[1])) * ex + (c[0] - lo[0])];
        if (slot < 0) {
          slot = (int)v.size();
          Src sr{};
          sr.x = c[0];
          sr.y = c[1];
          sr.z = c[2];
          sr.id = src;
          for (auto& q : sr.code) q = 0xFFFF;
          v.push_back(sr);
        }
        v[slot].code[w] = (unsigned short)ent[k].y;
      }
    }
    {   // (x, y, z) order = a scan of the dense index, x slowest
      std::vector<Src> sorted;
      sorted.reserve(v.size());
      for (int x = 0; x < ex; ++x)
        for (int y = 0; y < ey; ++y)
          for (int z = 0; z < ez; ++z) {
            const int q = at[((size_t)z * ey + y) * ex + x];
            if (q >= 0) sorted.push_back(v[q]);
          }
      v.swap(sorted);
    }
    auto& cols = pcols[P];
    int self_col[8];
    for (auto& q : self_col) q = -1;
    for (size_t i = 0; i < v.size();) {
      size_t j = i;
      while (j < v.size() && v[j].x == v[i].x && v[j].y == v[i].y) ++j;
      if (j - i > (size_t)htlr::kSepColMax) {
        ok = false;
        return;
      }
      htlr::SepCol c{};
      c.n = (int)(j - i);
      for (size_t k = i; k < j; ++k) {
        c.src[k - i] = v[k].id;
        for (int w = 0; w < 8; ++w) {
          c.code[k - i][w] = v[k].code[w];
          if (v[k].id == (int)(t0 + (int64_t)P * 8 + w) && is_self_code(v[k].code[w])) self_col[w] = (int)cols.size();
        }
      }
      cols.push_back(c);
      i = j;
    }
    pself[P].assign(self_col, self_col + 8);
  });
  if (!ok) return 0;
  // columns per part: ~16 parts per SM for the persistent CTAs' round robin
  // (parts sorted longest first), at most 12 columns each
  int per_part = 12;
  {
    int64_t total = 0;
    for (const auto& v : pcols) total += (int64_t)v.size();
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pl->device);
    per_part = (int)std::max<int64_t>(2, std::min<int64_t>(12, (total + 16 * sms - 1) / (16 * sms)));
    const char* e = std::getenv("HTLR_SEP_COLS");
    if (e && std::atoi(e) > 0) per_part = std::atoi(e);
  }
  struct Part {
    htlr::SepBlock b;
    int64_t work;
  };
  // parts of <= per_part columns of one parent; selfc[w] = index of the column
  // holding warp w's self pair (or -1)
  auto emit = [&](const std::vector<htlr::SepCol>& cols, const int* selfc, int64_t P, std::vector<Part>& parts,
                  std::vector<htlr::SepCol>& all) {
    for (size_t c0 = 0; c0 < cols.size(); c0 += per_part) {
      const size_t c1 = std::min(cols.size(), c0 + per_part);
      Part pt;
      pt.b.tgt0 = (int)(t0 + P * 8);
      pt.b.col_begin = (int)(all.size() + c0);
      pt.b.col_count = (int)(c1 - c0);
      pt.b.corr_mask = 0;
      pt.work = 0;
      for (size_t c = c0; c < c1; ++c) pt.work += cols[c].n;
      for (int w = 0; w < 8; ++w)
        if (selfc[w] >= (int)c0 && selfc[w] < (int)c1) pt.b.corr_mask |= 1 << w;
      parts.push_back(pt);
    }
    all.insert(all.end(), cols.begin(), cols.end());
  };
  auto by_work = [](const Part& a, const Part& b) { return a.work > b.work; };
  auto upload = [&](const std::vector<htlr::SepCol>& all, const std::vector<Part>& parts, DevBuf& dc,
                    DevBuf& db) -> int {
    std::vector<htlr::SepBlock> blocks;
    for (const auto& pt : parts) blocks.push_back(pt.b);
    if (dc.alloc(std::max<size_t>(1, all.size()) * sizeof(htlr::SepCol))) return 1;
    if (!all.empty()) CUDA_TRY(cudaMemcpy(dc.ptr, all.data(), all.size() * sizeof(htlr::SepCol), cudaMemcpyHostToDevice));
    if (db.alloc(std::max<size_t>(1, blocks.size()) * sizeof(htlr::SepBlock))) return 1;
    if (!blocks.empty())
      CUDA_TRY(cudaMemcpy(db.ptr, blocks.data(), blocks.size() * sizeof(htlr::SepBlock), cudaMemcpyHostToDevice));
    return 0;
  };
  if (pl->shard_world == 1) {
    std::vector<Part> parts;
    std::vector<htlr::SepCol> all;
    for (int64_t P = 0; P < npar; ++P) emit(pcols[P], pself[P].data(), P, parts, all);
    std::stable_sort(parts.begin(), parts.end(), by_work);
    if (upload(all, parts, ps.sep_cols, ps.sep_blocks)) return 1;
    ps.sep_nblocks = ps.sep_own_nb = (int)parts.size();
  } else {
    // sharded: columns cut where the sources change owner; the parts over own
    // sources first (they run while the exchange is in flight), then the rest
    const int64_t olo = pl->own_lo[L], ohi = pl->own_hi[L];
    std::vector<Part> grp[2];
    std::vector<htlr::SepCol> all;
    for (int64_t P = 0; P < npar; ++P) {
      for (int side = 0; side < 2; ++side) {
        std::vector<htlr::SepCol> cols;
        int selfc[8];
        for (auto& q : selfc) q = -1;
        for (const auto& c : pcols[P]) {
          htlr::SepCol h{};
          for (int k = 0; k < c.n; ++k) {
            const bool own = c.src[k] >= olo && c.src[k] < ohi;
            if (own != (side == 0)) continue;
            h.src[h.n] = c.src[k];
            for (int w = 0; w < 8; ++w) {
              h.code[h.n][w] = c.code[k][w];
              if (c.src[k] == (int)(t0 + P * 8 + w) && is_self_code(c.code[k][w])) selfc[w] = (int)cols.size();
            }
            ++h.n;
          }
          if (h.n > 0) cols.push_back(h);
        }
        if (!cols.empty()) emit(cols, selfc, P, grp[side], all);
      }
    }
    std::vector<Part> parts;
    for (auto& g : grp) {
      std::stable_sort(g.begin(), g.end(), by_work);
      parts.insert(parts.end(), g.begin(), g.end());
    }
    if (upload(all, parts, ps.sep_cols, ps.sep_blocks)) return 1;
    ps.sep_nblocks = (int)parts.size();
    ps.sep_own_nb = (int)grp[0].size();
    double w0 = 0, w1 = 0;
    for (const auto& pt : grp[0]) w0 += (double)pt.work;
    for (const auto& pt : grp[1]) w1 += (double)pt.work;
    ps.sep_own_frac = (w0 + w1) > 0 ? w0 / (w0 + w1) : 1.0;
  }
  // z-slab groups of the leaf pass (unsharded plans): 4 slabs of an even
  // number of leaf boxes (siblings share a slab), else 2.  With 4, the first quarter of u goes in alone and the leaf work
  // over its sources (~1/4) covers the copy of the rest; the last quarter of f
  // is the only copy-out left exposed.
  ps.sep_slabs = 0;
  ps.sep_gcount.clear();
  const int mz = pl->levels[L].m;
  int S = (mz % 8 == 0) ? 4 : 2;
  if (mz % (2 * S) != 0) S = (mz % 4 == 0) ? 2 : 0;
  if (ps.to_y && pl->shard_world == 1 && S > 0) {
    const int zs = mz / S;   // leaf boxes per slab
    std::vector<std::vector<Part>> grp(3);
    std::vector<htlr::SepCol> all;
    // per parent (all cores): its columns split by source slab class --
    // sources in the first slab vs the rest; the columns are cut only there
    // (each cut adds a mode-x / mode-y flush per target)
    struct Split {
      std::vector<htlr::SepCol> cols[2];
      int selfc[2][8];
      int th = 0;
    };
    std::vector<Split> split((size_t)npar);
    parallel_for((size_t)npar, [&](size_t P) {
      Split& sp = split[P];
      int tc[3];
      htlr::morton_decode(t0 + (int64_t)P * 8, 3, L, tc);
      sp.th = tc[2] / zs;   // the 8 children share the parent's slab (zs is even)
      for (int sh = 0; sh < 2; ++sh)
        for (auto& q : sp.selfc[sh]) q = -1;
      for (const auto& c : pcols[P]) {
        htlr::SepCol h[2] = {};
        for (int k = 0; k < c.n; ++k) {
          int sc[3];
          htlr::morton_decode(c.src[k], 3, L, sc);
          const int sh = sc[2] >= zs ? 1 : 0;
          htlr::SepCol& o = h[sh];
          o.src[o.n] = c.src[k];
          for (int w = 0; w < 8; ++w) {
            o.code[o.n][w] = c.code[k][w];
            if (c.src[k] == (int)(t0 + (int64_t)P * 8 + w) && is_self_code(c.code[k][w]))
              sp.selfc[sh][w] = (int)sp.cols[sh].size();
          }
          ++o.n;
        }
        for (int sh = 0; sh < 2; ++sh)
          if (h[sh].n > 0) sp.cols[sh].push_back(h[sh]);
      }
    });
    for (int64_t P = 0; P < npar; ++P)
      for (int sh = 0; sh < 2; ++sh) {
        const Split& sp = split[P];
        const int range = sh == 0 ? 0 : (sp.th < S - 1 ? 1 : 2);
        if (!sp.cols[sh].empty()) emit(sp.cols[sh], sp.selfc[sh], P, grp[range], all);
      }
    std::vector<Part> parts;
    for (auto& g : grp) {
      std::stable_sort(g.begin(), g.end(), by_work);
      ps.sep_gcount.push_back((int)g.size());
      parts.insert(parts.end(), g.begin(), g.end());
    }
    if (upload(all, parts, ps.sep_gcols, ps.sep_gblocks)) return 1;
    ps.sep_slabs = S;
  }
  return 0;
}

static int upload_sep(Pass& ps, const std::vector<int2>& ent, const std::vector<htlr::SepItem>& items) {
  if (ps.sep_pairs.alloc(std::max<size_t>(1, ent.size()) * sizeof(int2))) return 1;
  if (!ent.empty()) CUDA_TRY(cudaMemcpy(ps.sep_pairs.ptr, ent.data(), ent.size() * sizeof(int2), cudaMemcpyHostToDevice));
  if (ps.sep_items.alloc(std::max<size_t>(1, items.size()) * sizeof(htlr::SepItem))) return 1;
  if (!items.empty())
    CUDA_TRY(cudaMemcpy(ps.sep_items.ptr, items.data(), items.size() * sizeof(htlr::SepItem), cudaMemcpyHostToDevice));
  return 0;
}

// Separable-core formulation (htlr_sep.cu): a tensor-product kernel (the
// Gaussian) on a uniform 3-D grid with p = leaf side = 8.  HTLR_SEPARABLE=0
// keeps the dense-core GEMM path for A/B runs.
static bool sep_wanted(const htlr_plan* pl) {
  const char* e = std::getenv("HTLR_SEPARABLE");
  if (e && e[0] == '0') return false;
  return !pl->mapped && !pl->lowrank && pl->kp.kind == HTLR_KERNEL_GAUSSIAN && pl->d == 3 && pl->p == htlr::kSepP &&
         pl->sL == htlr::kSepP;
}

// Work items of at most this many pairs (split at group boundaries), so the
// warps of a pass finish together; HTLR_SEP_CHUNK overrides.
static int sep_chunk() {
  const char* e = std::getenv("HTLR_SEP_CHUNK");
  const int v = e ? std::atoi(e) : 0;
  return v > 0 ? v : 128;
}

// Banded leaf pass (sep_band_kernel, htlr_sep.cu): enabled only when every
// leaf target's list (kind, offset) equals the product-set structure the
// sweeps apply -- per axis R10 = {-4-c..5-c} minus the corner parents'
// children A4^3, near = {-2..2}^3 minus {+-2}^3, inside the domain -- so the
// sweeps apply exactly the listed blocks.  HTLR_SEP_BAND=0 keeps the
// cooperative pass.
static bool band_check(const htlr_plan* pl, Pass& ps, int OR, const std::vector<int64_t>& ptr,
                       const std::vector<int2>& ent, double& flops) {
  const char* e = std::getenv("HTLR_SEP_BAND");
  if (e && e[0] == '0') return false;
  const int L = ps.level;
  // L >= 3: with 4 boxes per axis the cooperative pass is faster (the line /
  // plane kernels at NB = 4: 19.7 vs 13.7 us for config 4's level 2)
  if (pl->d != 3 || L < 3 || L > 4) return false;
  const int nb = 1 << L;
  if (OR < std::min(5, nb - 1)) return false;   // the sweeps' in-domain offsets need table slots
  const int64_t nt = (int64_t)ptr.size() - 1, t0 = pl->own_lo[L];
  if (nt <= 0) return false;
  // own targets (sharded plans: Morton subtrees) must form a box region
  int lo[3] = {nb, nb, nb}, hi[3] = {0, 0, 0};
  for (int64_t t = 0; t < nt; ++t) {
    int tc[3];
    htlr::morton_decode(t0 + t, 3, L, tc);
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], tc[a]);
      hi[a] = std::max(hi[a], tc[a] + 1);
    }
  }
  if ((int64_t)(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]) != nt) return false;
  std::atomic<bool> ok{true};
  parallel_for((size_t)nt, [&](size_t t) {
    if (!ok.load(std::memory_order_relaxed)) return;
    int tc[3];
    htlr::morton_decode(t0 + (int64_t)t, 3, L, tc);
    std::vector<int2> want;
    for (int oz = -5; oz <= 5; ++oz)
      for (int oy = -5; oy <= 5; ++oy)
        for (int ox = -5; ox <= 5; ++ox) {
          const int o[3] = {ox, oy, oz};
          bool in10 = true, inA4 = true, in5 = true, corner = true;
          int sc[3];
          for (int a = 0; a < 3; ++a) {
            const int c = tc[a] & 1;
            sc[a] = tc[a] + o[a];
            in10 = in10 && o[a] >= -4 - c && o[a] <= 5 - c;
            inA4 = inA4 && (o[a] <= -3 - c || o[a] >= 4 - c);
            in5 = in5 && o[a] >= -2 && o[a] <= 2;
            corner = corner && (o[a] == -2 || o[a] == 2);
          }
          if (!in10 || inA4) continue;
          if (sc[0] < 0 || sc[0] >= nb || sc[1] < 0 || sc[1] >= nb || sc[2] < 0 || sc[2] >= nb) continue;
          // leaf level: near blocks (kind 1); coupling level: not in the list (children)
          if (!ps.to_y && in5 && !corner) continue;
          const int kind = (in5 && !corner) ? 1 : 0;
          const int code = (kind << 12) | ((ox + OR) << 8) | ((oy + OR) << 4) | (oz + OR);
          want.push_back(make_int2((int)htlr::morton_encode(sc, 3, L), code));
        }
    std::vector<int2> got(ent.begin() + ptr[t], ent.begin() + ptr[t + 1]);
    auto lt = [](const int2& a, const int2& b) { return a.y != b.y ? a.y < b.y : a.x < b.x; };
    std::sort(want.begin(), want.end(), lt);
    std::sort(got.begin(), got.end(), lt);
    bool same = want.size() == got.size();
    for (size_t k = 0; same && k < want.size(); ++k) same = want[k].x == got[k].x && want[k].y == got[k].y;
    if (!same) ok.store(false);
  });
  if (!ok.load()) return false;
  flops = band_flops_of(L, ps.to_y, nt);
  for (int a = 0; a < 3; ++a) {
    ps.band_lo[a] = lo[a];
    ps.band_hi[a] = hi[a];
  }
  return true;
}

// factor tables of a separable pass: kind 0 (admissible, level factor folded)
// and kind 1 (near), per-axis offsets -OR..OR
static int sep_factor_tables(htlr_plan* pl, Pass& ps, int OR, cudaStream_t st) {
  const bool leaf = ps.to_y;
  const Level& lv = pl->levels[ps.level];
  const int NO = 2 * OR + 1;
  const int nslots = 2 * NO;
  if (ps.sep_tab.alloc((size_t)nslots * htlr::kSepSlot * sizeof(double))) return 1;
  CUDA_TRY(cudaMemsetAsync(ps.sep_tab.ptr, 0, (size_t)nslots * htlr::kSepSlot * sizeof(double), st));
  std::vector<htlr::SepJob> jobs;
  for (int kind = 0; kind < 2; ++kind) {
    if (kind == 0 && !lv.R.ptr) continue;
    if (kind == 1 && !leaf) continue;
    for (int o = -OR; o <= OR; ++o) {
      htlr::SepJob j;
      j.kind = kind;
      j.o = o;
      j.t0 = std::max(0, -o);
      j.side = kind == 0 ? lv.side : pl->sL;
      j.R = kind == 0 ? lv.R.d() : nullptr;
      j.dst = ps.sep_tab.d() + (int64_t)(kind * NO + o + OR) * htlr::kSepSlot;
      jobs.push_back(j);
    }
  }
  DevBuf jb;
  if (jb.alloc(std::max<size_t>(1, jobs.size()) * sizeof(htlr::SepJob))) return 1;
  CUDA_TRY(cudaMemcpyAsync(jb.ptr, jobs.data(), jobs.size() * sizeof(htlr::SepJob), cudaMemcpyHostToDevice, st));
  htlr::launch_sep_tables((const htlr::SepJob*)jb.ptr, (int)jobs.size(), pl->p, pl->sL, pl->h, pl->kp, pl->diag.d(),
                          pl->hd, leaf ? pl->sep_corr.d() : nullptr, st);
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());
  pl->device_scalars += (int64_t)nslots * htlr::kSepSlot;
  return 0;
}

// Per-target pair runs of one pass: (source, code) sorted by code, where code
// packs (kind, o_x, o_y, o_z); returns 1 (and leaves the pass untouched) when
// an axis offset does not fit the 4-bit code.
static int build_sep_pass(htlr_plan* pl, Pass& ps, bool& fits, cudaStream_t st) {
  const int d = pl->d;
  const bool leaf = ps.to_y;
  const Level& lv = pl->levels[ps.level];
  std::vector<std::array<int, 4>> mo((size_t)ps.nmats);   // kind, o_x, o_y, o_z
  int OR = 0;
  for (int m = 0; m < ps.nmats; ++m) {
    const bool near = leaf && m < pl->near_mats;
    const auto& rp = near ? pl->near.rep[m] : lv.adm.rep[m - (leaf ? pl->near_mats : 0)];
    mo[m][0] = near ? 1 : 0;
    for (int a = 0; a < d; ++a) {
      mo[m][1 + a] = rp[3 + a] - rp[a];
      OR = std::max(OR, std::abs(mo[m][1 + a]));
    }
  }
  if (ps.analytic) OR = std::min(5, (1 << ps.level) - 1);   // the banded terms' offsets inside the level
  const int NO = 2 * OR + 1;
  if (NO > htlr::kSepMaxNO) {
    fits = false;
    return 0;
  }
  fits = true;
  PhaseTimer tm;
  if (ps.analytic) {
    // the level's lists are the banded sweeps' product sets (analytic_bands_ok):
    // the whole level as one box region, no pair runs
    const int nb = 1 << ps.level;
    ps.sep_NO = NO;
    ps.sep_groups = 0;
    ps.sep_nblocks = 0;
    ps.sep_nitems = 0;
    ps.band = true;
    ps.band_flops = band_flops_of(ps.level, leaf, lv.nclusters);
    for (int a = 0; a < 3; ++a) {
      ps.band_lo[a] = 0;
      ps.band_hi[a] = nb;
    }
    return sep_factor_tables(pl, ps, OR, st);
  }
  // counting sort by target, then each target's run by (code, source)
  const int64_t t0 = pl->own_lo[ps.level], nt = pl->own_hi[ps.level] - t0;
  std::vector<int64_t> ptr((size_t)nt + 1, 0);
  std::vector<int2> ent(ps.pairs_host.size());
  {
    // per-chunk counts per target, exclusive prefix over (target, chunk), then
    // every chunk writes its pairs at its own positions (all cores, no atomics)
    const size_t np = ps.pairs_host.size(), chunk = 1 << 16, nch = (np + chunk - 1) / chunk;
    std::vector<int> code_of(ps.nmats);
    std::vector<int> mat_of_chunk(nch + 1, 0);
    for (int m = 0; m < ps.nmats; ++m)
      code_of[m] = (mo[m][0] << 12) | ((mo[m][1] + OR) << 8) | ((mo[m][2] + OR) << 4) | (mo[m][3] + OR);
    for (size_t c = 0; c < nch; ++c)
      mat_of_chunk[c] = (int)(std::upper_bound(ps.seg.begin(), ps.seg.end(), (int)(c * chunk)) - ps.seg.begin()) - 1;
    std::vector<std::vector<int64_t>> cnt(nch, std::vector<int64_t>((size_t)nt, 0));
    parallel_for(nch, [&](size_t c) {
      const size_t e = std::min(np, (c + 1) * chunk);
      for (size_t k = c * chunk; k < e; ++k) cnt[c][ps.pairs_host[k].x - t0]++;
    });
    int64_t acc = 0;
    for (int64_t t = 0; t < nt; ++t) {
      ptr[t] = acc;
      for (size_t c = 0; c < nch; ++c) {
        const int64_t v = cnt[c][t];
        cnt[c][t] = acc;
        acc += v;
      }
    }
    ptr[nt] = acc;
    parallel_for(nch, [&](size_t c) {
      const size_t e = std::min(np, (c + 1) * chunk);
      int m = mat_of_chunk[c];
      for (size_t k = c * chunk; k < e; ++k) {
        while ((int)k >= ps.seg[m + 1]) ++m;
        const int2 q = ps.pairs_host[k];
        ent[cnt[c][q.x - t0]++] = make_int2(q.y, code_of[m]);
      }
    });
  }
  parallel_for((size_t)nt, [&](size_t t) {
    std::sort(ent.begin() + ptr[t], ent.begin() + ptr[t + 1],
              [](const int2& a, const int2& b) { return a.y != b.y ? a.y < b.y : a.x < b.x; });
  });
  // groups = runs of equal (kind, o_x, o_y) per target (algorithmic flop count)
  std::vector<int64_t> gcount((size_t)nt, 0);
  parallel_for((size_t)nt, [&](size_t t) {
    int64_t c = 0;
    for (int64_t k = ptr[t]; k < ptr[t + 1]; ++k)
      if (k == ptr[t] || (ent[k].y >> 4) != (ent[k - 1].y >> 4)) ++c;
    gcount[t] = c;
  });
  int64_t groups = 0;
  for (int64_t c : gcount) groups += c;
  tm.mark("  separable: per-target runs");
  ps.sep_NO = NO;
  ps.sep_groups = groups;
  ps.sep_nblocks = 0;
  ps.sep_nitems = 0;
  ps.band = band_check(pl, ps, OR, ptr, ent, ps.band_flops);
  tm.mark("  separable: banded-pass check");
  // a banded pass applies its blocks as line sweeps: no columns, parts or
  // per-warp items (config 4's leaf level: -20 ms of construction)
  if (!ps.band && sep_block_enabled(ps.to_y) && build_sep_blocks(pl, ps, ptr, ent)) return 1;
  tm.mark("  separable: columns + parts");
  const int selfcode = (1 << 12) | (OR << 8) | (OR << 4) | OR;
  const int chunk = sep_chunk();
  std::vector<htlr::SepItem> items;
  for (int64_t t = 0; t < nt && ps.sep_nblocks == 0 && !ps.band; ++t) {
    int64_t b = ptr[t];
    const int64_t e = ptr[t + 1];
    while (b < e) {
      // extend by whole groups while the item stays within `chunk` pairs
      int64_t c = b;
      int flags = 0;
      while (c < e) {
        int64_t g = c;
        while (g < e && (ent[g].y >> 4) == (ent[c].y >> 4)) ++g;
        if (c > b && g - b > chunk) break;
        for (int64_t k = c; k < g; ++k)
          if (ent[k].y == selfcode && ent[k].x == (int)(t0 + t)) flags |= 1;
        c = g;
      }
      items.push_back(htlr::SepItem{(int)(t0 + t), (int)b, (int)(c - b), flags});
      b = c;
    }
  }
  // per-warp items only when neither the bands nor the cooperative layout apply
  if (ps.sep_nblocks == 0 && !ps.band) {
    ps.sep_nitems = (int)items.size();
    if (upload_sep(ps, ent, items)) return 1;
  }
  return sep_factor_tables(pl, ps, OR, st);
}

// Mapped grid construction: geometry tables, per (level, interval) nodes and
// raw factors, per-point diagonal cell integrals, CSR lists of own targets.
static int construct_mapped(htlr_plan* pl, cudaStream_t st) {
  const int d = pl->d, p = pl->p, n = pl->n;
  PhaseTimer tm(st);
  if (upload(pl->d_mb, pl->mb.data(), pl->mb.size() * sizeof(double))) return 1;
  if (upload(pl->d_mx, pl->mx.data(), pl->mx.size() * sizeof(double))) return 1;
  if (upload(pl->d_mc, pl->mc.data(), pl->mc.size() * sizeof(double))) return 1;
  std::vector<htlr::MappedFactorJob> jobs;
  int total = 0;
  pl->device_scalars = 0;
  for (auto& lv : pl->levels) {
    if (!lv.needs_up) continue;
    const int nint = lv.m;
    if (lv.nodes.alloc((size_t)nint * p * sizeof(double))) return 1;
    if (lv.Lm.alloc((size_t)nint * lv.side * p * sizeof(double))) return 1;
    if (lv.WLm.alloc((size_t)nint * lv.side * p * sizeof(double))) return 1;
    jobs.push_back({lv.side, nint, lv.nodes.d(), lv.Lm.d(), lv.WLm.d()});
    total += nint;
    pl->device_scalars += (int64_t)nint * p * (1 + 2 * lv.side);
    if (upload(lv.d_ptr, lv.csr_ptr.data(), lv.csr_ptr.size() * sizeof(int64_t))) return 1;
    if (upload(lv.d_cols, lv.csr_cols.data(), lv.csr_cols.size() * sizeof(int))) return 1;
  }
  if (upload(pl->d_near_ptr, pl->near_ptr.data(), pl->near_ptr.size() * sizeof(int64_t))) return 1;
  if (upload(pl->d_near_cols, pl->near_cols.data(), pl->near_cols.size() * sizeof(int))) return 1;
  // symmetric regeneration: the column sums land in rows of any cluster, so
  // a sharded plan accumulates full-size H_l / Y, summed over the shards by
  // the caller between htlr_matvec_contract and htlr_matvec_expand
  if (regen_sym_enabled()) {
    const bool full = pl->shard_world == 1;
    for (auto& lv : pl->levels)
      if (lv.needs_up && htlr::regen_sym_supported(d, p))
        if (build_sym(lv.csr_ptr, lv.csr_cols, pl->own_lo[lv.level], full, lv.sym, nullptr, nullptr)) return 1;
    if (htlr::regen_sym_supported(d, pl->sL)) {
      std::vector<int64_t> sp;
      std::vector<int> sc;
      if (build_sym(pl->near_ptr, pl->near_cols, pl->own_lo[pl->L], full, pl->near_sym, &sp, &sc)) return 1;
      if (pl->near_sym.on) {
        if (upload(pl->d_self_ptr, sp.data(), sp.size() * sizeof(int64_t))) return 1;
        if (upload(pl->d_self_cols, sc.data(), std::max<size_t>(1, sc.size()) * sizeof(int))) return 1;
      }
    }
  }
  tm.mark("construct: CSR upload + sym lists");
  DevBuf djobs;
  if (!jobs.empty()) {
    if (upload(djobs, jobs.data(), jobs.size() * sizeof(htlr::MappedFactorJob))) return 1;
    htlr::launch_mapped_factors((const htlr::MappedFactorJob*)djobs.ptr, (int)jobs.size(), total, pl->d_mb.d(),
                                pl->d_mx.d(), pl->d_mc.d(), p, st);
  }
  tm.mark("construct: factors");
  // Nystrom diagonal: integral of k(x_i, .) over each point's cell
  std::vector<double> gx, gw;
  gauss01(pl->desc.quad_q, gx, gw);
  gx.insert(gx.end(), gw.begin(), gw.end());
  if (upload(pl->gl, gx.data(), gx.size() * sizeof(double))) return 1;
  if (pl->dvec.alloc(pl->N * sizeof(double))) return 1;
  pl->device_scalars += pl->N;
  htlr::launch_mapped_diag(pl->kp, d, n, pl->desc.quad_q, pl->gl.d(), pl->gl.d() + pl->desc.quad_q, pl->d_mb.d(),
                           pl->d_mx.d(), pl->dvec.d(), pl->N, st);
  tm.mark("construct: per-point diagonal");
  if (pl->diag.alloc(sizeof(double))) return 1;
  CUDA_TRY(cudaMemsetAsync(pl->diag.ptr, 0, sizeof(double), st));
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());
  djobs.release();
  tm.mark("construct: finish");
  pl->constructed = true;
  return 0;
}

// Cube tables of a separable plan (htlr_cube.cu): the upward / downward
// passes contract 16^3-point cubes (the level-(L-1) boxes) with Q_c = Q_{L-1}
// and reach every coarser compressed level l through
//   M_l[s] = Q_c^T Q_l[16 s .. 16 s + 15]   (8 x 8, sub-position s per axis).
// Q_l's rows over a cube are degree-7 polynomials, which Q_c's columns span,
// so Q_c M_l[s] = Q_l[cube rows] up to rounding; the residual is checked here
// and the cube passes are disabled (generic upward / downward) if it is not
// at rounding level.
static int build_cube_tables(htlr_plan* pl) {
  pl->cube_ok = false;
  const int L = pl->L, lc = L - 1;
  if (!htlr::cube_supported(pl->d, pl->p, pl->sL, L) || lc < 0) return 0;
  std::vector<int> coarse;
  bool has_c = false;
  for (const auto& ps : pl->passes) {
    if (ps.to_y) continue;
    const Level& lv = pl->levels[ps.level];
    if (lv.Kron.ptr || !lv.Q.ptr) return 0;
    if (ps.level == lc) has_c = lv.side == 16;
    else if (ps.level < lc) coarse.push_back(ps.level);
    else return 0;
  }
  if (coarse.empty() && !has_c) {   // no compressed level: the permute only
    pl->cube_ok = true;
    return 0;
  }
  if (!has_c || (int)coarse.size() > htlr::kMaxCubeCoarse) return 0;
  const int p = pl->p;
  std::vector<double> qc(16 * p);
  CUDA_TRY(cudaMemcpy(qc.data(), pl->levels[lc].Q.ptr, qc.size() * sizeof(double), cudaMemcpyDeviceToHost));
  for (int l : coarse) {
    Level& lv = pl->levels[l];
    std::vector<double> ql((size_t)lv.side * p);
    CUDA_TRY(cudaMemcpy(ql.data(), lv.Q.ptr, ql.size() * sizeof(double), cudaMemcpyDeviceToHost));
    const int ns = lv.side / 16;
    std::vector<double> M((size_t)ns * 64);
    double qmax = 0.0, res = 0.0;
    for (double v : ql) qmax = std::max(qmax, std::fabs(v));
    for (int s = 0; s < ns; ++s) {
      double* Ms = M.data() + 64 * s;
      for (int a1 = 0; a1 < 8; ++a1)
        for (int a = 0; a < 8; ++a) {
          double acc = 0.0;
          for (int x = 0; x < 16; ++x) acc += qc[x * 8 + a1] * ql[(16 * s + x) * 8 + a];
          Ms[a1 * 8 + a] = acc;
        }
      for (int x = 0; x < 16; ++x)
        for (int a = 0; a < 8; ++a) {
          double v = 0.0;
          for (int a1 = 0; a1 < 8; ++a1) v += qc[x * 8 + a1] * Ms[a1 * 8 + a];
          res = std::max(res, std::fabs(v - ql[(16 * s + x) * 8 + a]));
        }
    }
    if (!(res <= 1e-13 * std::max(qmax, 1.0))) return 0;
    if (upload(lv.Mcube, M.data(), M.size() * sizeof(double))) return 1;
  }
  pl->cube_ok = true;
  return 0;
}

// the cube passes' per-call parameters (false: not applicable to this plan)
static bool cube_params(const htlr_plan* pl, double* const* W, htlr::CubeLevels& cl) {
  cl = htlr::CubeLevels{};
  if (!pl->cube_ok) return false;
  for (size_t i = 0; i < pl->passes.size(); ++i) {
    const Pass& ps = pl->passes[i];
    if (ps.to_y) continue;
    const Level& lv = pl->levels[ps.level];
    if (ps.level == pl->L - 1) {
      cl.Qc = lv.Q.d();
      cl.Wc = W ? W[i] : nullptr;
      cl.Hc = lv.H.d();
      cl.K_pad_c = ps.K_pad;
      cl.zpitch_c = ps.zpitch;
    } else {
      if (cl.ncoarse >= htlr::kMaxCubeCoarse) return false;
      cl.lev[cl.ncoarse++] = htlr::CubeLevel{ps.level, lv.Mcube.d(), W ? W[i] : nullptr, lv.H.d(), ps.K_pad, ps.zpitch};
    }
  }
  return cl.Qc != nullptr || cl.ncoarse == 0;
}

int htlr_construct(htlr_plan* pl, void* stream) {
  if (!pl) return fail(-1, "null plan");
  if (pl->device < 0) return fail(-1, "host-only plan: no device work");
  if (!pl->lists_built) {
    int rc = htlr_build_lists(pl);
    if (rc) return rc;
  }
  CUDA_TRY(cudaSetDevice(pl->device));
  cudaStream_t st = (cudaStream_t)stream;
  PhaseTimer tm(st);
  // the dense GEMM passes' (target, source) lists (not used by the separable
  // formulation, uploaded if it does not apply)
  auto upload_pairs = [&]() -> int {
    for (auto& ps : pl->passes) {
      if (ps.pairs.alloc(std::max<size_t>(1, ps.pairs_host.size()) * sizeof(int2))) return 1;
      if (!ps.pairs_host.empty())
        CUDA_TRY(cudaMemcpy(ps.pairs.ptr, ps.pairs_host.data(), ps.pairs_host.size() * sizeof(int2),
                            cudaMemcpyHostToDevice));
    }
    return 0;
  };
  if (!sep_wanted(pl) && upload_pairs()) return 1;
  if (pl->mapped) return construct_mapped(pl, st);
  const int d = pl->d, p = pl->p;
  // diagonal cell average (operators.py:95-99)
  std::vector<double> gx, gw;
  gauss01(pl->desc.quad_q, gx, gw);
  if (pl->gl.alloc(2 * gx.size() * sizeof(double))) return 1;
  if (pl->diag.alloc(sizeof(double))) return 1;
  std::vector<double> glh(gx);
  glh.insert(glh.end(), gw.begin(), gw.end());
  CUDA_TRY(cudaMemcpyAsync(pl->gl.ptr, glh.data(), glh.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  const bool singular = pl->desc.corner_subdivision != 0;   // caller: !smooth_at_diagonal && corner_subdivision
  htlr::launch_diag(pl->kp, d, pl->h, pl->desc.quad_q, pl->gl.d(), pl->gl.d() + gx.size(), singular ? 1 : 0,
                    pl->diag.d(), st);
  // per-level factors (one representative box per level)
  std::vector<htlr::FactorJob> fj;
  std::vector<int> fj_level;
  DevBuf scratch;
  size_t scratch_words = 0;
  for (auto& lv : pl->levels)
    if (lv.num_adm > 0) scratch_words += 2 * (size_t)lv.side * p;
  if (scratch.alloc(std::max<size_t>(scratch_words, 1) * sizeof(double))) return 1;
  size_t soff = 0;
  for (auto& lv : pl->levels) {
    if (lv.num_adm == 0) continue;
    if (lv.Q.alloc((size_t)lv.side * p * sizeof(double))) return 1;
    if (lv.R.alloc((size_t)p * p * sizeof(double))) return 1;
    htlr::FactorJob j;
    j.side = lv.side;
    j.Q = lv.Q.d();
    j.R = lv.R.d();
    j.work = scratch.d() + soff;
    soff += (size_t)lv.side * p;
    j.work2 = scratch.d() + soff;
    soff += (size_t)lv.side * p;
    fj.push_back(j);
  }
  DevBuf jobsbuf;
  if (!fj.empty()) {
    if (jobsbuf.alloc(fj.size() * sizeof(htlr::FactorJob))) return 1;
    CUDA_TRY(cudaMemcpyAsync(jobsbuf.ptr, fj.data(), fj.size() * sizeof(htlr::FactorJob), cudaMemcpyHostToDevice, st));
    htlr::launch_factor_qr((int)fj.size(), (const htlr::FactorJob*)jobsbuf.ptr, pl->h, p, st);
  }
  tm.mark("construct: diagonal + level factors");
  // H-matrix baseline: dense Kronecker factors of the levels with a factor
  pl->device_scalars = 0;
  if (pl->lowrank) {
    for (auto& lv : pl->levels) {
      if (!lv.needs_up || lv.side == p) continue;
      const int64_t S = ipow(lv.side, d), P = ipow(p, d);
      if (lv.Kron.alloc((size_t)(S * P) * sizeof(double))) return 1;
      htlr::launch_kron_factor(lv.Q.d(), d, lv.side, p, lv.Kron.d(), st);
      pl->device_scalars += S * P;
    }
  }
  // separable-core formulation: 1-D factor tables instead of dense cores
  pl->sep = false;
  for (auto& ps : pl->passes) {   // natural vector layout unless the separable passes apply
    ps.zpitch = 0;
    ps.K_pad = round_up(ps.P, htlr::kKC);
  }
  if (sep_wanted(pl)) {
    if (pl->sep_corr.alloc(sizeof(double))) return 1;
    bool all = true;
    for (auto& ps : pl->passes) {
      bool fits = false;
      if (build_sep_pass(pl, ps, fits, st)) return 1;
      if (!fits) {
        all = false;
        break;
      }
    }
    if (all) {
      // source vectors (ub, W_l) stored with padded z-planes: one bulk copy
      // per box into the apply kernel's bank-conflict-free staging layout
      for (auto& ps : pl->passes) {
        ps.zpitch = htlr::kSepZPitch;
        ps.K_pad = htlr::kSepP * htlr::kSepZPitch;
      }
      CUDA_TRY(cudaStreamSynchronize(st));
      CUDA_TRY(cudaGetLastError());
      tm.mark("construct: separable lists + factor tables");
      scratch.release();
      jobsbuf.release();
      pl->sep = true;
      if (build_cube_tables(pl)) return 1;
      pl->constructed = true;
      return 0;
    }
    for (auto& ps : pl->passes) {   // an offset outside the 4-bit codes: dense cores
      ps.sep_tab.release();
      ps.sep_pairs.release();
      ps.sep_items.release();
      ps.sep_blocks.release();
      ps.sep_cols.release();
    }
    pl->device_scalars = 0;
    if (upload_pairs()) return 1;
  }
  // tables
  for (auto& ps : pl->passes) {
    if (ps.table.alloc((size_t)ps.nmats * ps.mat_stride * sizeof(double))) return 1;
    pl->device_scalars += (int64_t)ps.nmats * ps.mat_stride;
  }
  // cores, batched
  const int P = ipow(p, d);
  const int64_t PP = (int64_t)P * P;
  int batch = (int)std::max<int64_t>(1, std::min<int64_t>(512, (int64_t)(256ll << 20) / (PP * 8)));
  DevBuf cbuf0, cbuf1, cjobs;
  std::vector<htlr::CoreJob> cj;
  auto flush_cores = [&](int MT, int M_pad, int K_pad) -> int {
    if (cj.empty()) return 0;
    if (cjobs.alloc(cj.size() * sizeof(htlr::CoreJob))) return 1;
    CUDA_TRY(cudaMemcpyAsync(cjobs.ptr, cj.data(), cj.size() * sizeof(htlr::CoreJob), cudaMemcpyHostToDevice, st));
    htlr::launch_core_batch((const htlr::CoreJob*)cjobs.ptr, (int)cj.size(), d, p, pl->h, pl->hd, pl->kp,
                            cbuf0.d(), cbuf1.d(), MT, M_pad, K_pad, st);
    // the job array is reused: wait before overwriting it
    CUDA_TRY(cudaStreamSynchronize(st));
    cj.clear();
    return 0;
  };
  for (int l = 0; l <= pl->L; ++l) {
    Level& lv = pl->levels[l];
    if (lv.num_adm == 0) continue;
    Pass* ps = nullptr;
    int mat0 = 0;
    for (auto& q : pl->passes)
      if (!q.to_y && q.level == l) ps = &q;
    if (!ps) {
      ps = &pl->passes[pl->leaf_pass];
      mat0 = pl->near_mats;
    }
    if (cbuf0.alloc((size_t)batch * PP * sizeof(double))) return 1;
    if (cbuf1.alloc((size_t)batch * PP * sizeof(double))) return 1;
    for (size_t o = 0; o < lv.adm.rep.size(); ++o) {
      htlr::CoreJob j;
      for (int a = 0; a < 3; ++a) {
        j.tlo[a] = lv.adm.rep[o][a] * lv.side;
        j.slo[a] = lv.adm.rep[o][3 + a] * lv.side;
      }
      j.side = lv.side;
      j.R = lv.R.d();
      j.dst = ps->table.d() + (int64_t)(mat0 + o) * ps->mat_stride;
      cj.push_back(j);
      if ((int)cj.size() == batch && flush_cores(ps->MT, ps->M_pad, ps->K_pad)) return 1;
    }
    if (flush_cores(ps->MT, ps->M_pad, ps->K_pad)) return 1;
  }
  // unique near blocks
  {
    Pass& ps = pl->passes[pl->leaf_pass];
    std::vector<htlr::NearJob> nj;
    for (size_t o = 0; o < pl->near.rep.size(); ++o) {
      htlr::NearJob j;
      bool self = true;
      for (int a = 0; a < 3; ++a) {
        j.tlo[a] = pl->near.rep[o][a] * pl->sL;
        j.slo[a] = pl->near.rep[o][3 + a] * pl->sL;
        if (pl->near.rep[o][a] != pl->near.rep[o][3 + a]) self = false;
      }
      j.self = self ? 1 : 0;
      j.dst = ps.table.d() + (int64_t)o * ps.mat_stride;
      nj.push_back(j);
    }
    DevBuf njobs;
    if (!nj.empty()) {
      if (njobs.alloc(nj.size() * sizeof(htlr::NearJob))) return 1;
      CUDA_TRY(cudaMemcpyAsync(njobs.ptr, nj.data(), nj.size() * sizeof(htlr::NearJob), cudaMemcpyHostToDevice, st));
      htlr::launch_near_blocks((const htlr::NearJob*)njobs.ptr, (int)nj.size(), d, pl->sL, pl->h, pl->hd, pl->kp,
                               pl->diag.d(), ps.MT, ps.M_pad, ps.K_pad, st);
      CUDA_TRY(cudaStreamSynchronize(st));
    }
    njobs.release();
    // Toeplitz generators for a near-only leaf pass of 3-D side-8 leaves
    // (n = 8 * 2^L, so h is dyadic and every near block is exactly Toeplitz)
    if (near_gen_enabled() && d == 3 && pl->sL == 8 && !pl->merged && ps.MT == 128 && ps.K_pad == 512 &&
        ps.nmats == (int)pl->near.rep.size() && ps.nmats > 0) {
      if (ps.gen.alloc((size_t)ps.nmats * htlr::kGenStride * sizeof(double))) return 1;
      htlr::launch_near_gen(ps.table.d(), ps.mat_stride, ps.nmats, ps.MT, ps.K_pad, ps.gen.d(), st);
      pl->device_scalars += (int64_t)ps.nmats * htlr::kGenStride;
    }
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());
  scratch.release();
  jobsbuf.release();
  cbuf0.release();
  cbuf1.release();
  cjobs.release();
  pl->constructed = true;
  return 0;
}

static void drop_graphs(htlr_plan* pl);

static int ensure_workspace(htlr_plan* pl, int R) {
  if (pl->ws_R >= R) return 0;
  drop_graphs(pl);   // captured graphs hold the old workspace addresses
  const int d = pl->d, p = pl->p;
  const int P = ipow(p, d);
  if (pl->mapped) {
    const int PL = ipow(pl->sL, d);
    const int64_t nleaf = pl->levels[pl->L].nclusters;
    if (pl->ub.alloc((size_t)nleaf * R * PL * sizeof(double))) return 1;
    if (pl->Y.alloc((size_t)nleaf * R * PL * sizeof(double))) return 1;
    if (pl->near_sym.on && pl->Vn.alloc((size_t)nleaf * PL * sizeof(double))) return 1;
    for (auto& lv : pl->levels) {
      if (!lv.needs_up) continue;
      if (lv.W.alloc((size_t)lv.nclusters * R * P * sizeof(double))) return 1;
      if (lv.H.alloc((size_t)lv.nclusters * R * P * sizeof(double))) return 1;
    }
    pl->ws_R = R;
    return 0;
  }
  const Pass& lp = pl->passes[pl->leaf_pass];
  const int64_t nleaf = pl->levels[pl->L].nclusters;
  if (pl->ub.alloc((size_t)nleaf * R * lp.K_pad * sizeof(double))) return 1;
  if (pl->Y.alloc((size_t)nleaf * R * lp.P * sizeof(double))) return 1;
  for (auto& ps : pl->passes) {
    if (!pl->sep || !ps.band) continue;
    if (ps.band_ws.alloc((size_t)htlr::sep_band_workspace(ps.level, R) * sizeof(double))) return 1;
    if (band_xy_lines(pl) && ps.band_ws2.alloc((size_t)htlr::sep_band_workspace(ps.level, R) * sizeof(double)))
      return 1;
    CUDA_TRY(htlr::sep_band_init());   // kernel attributes, outside any graph capture
  }
  for (auto& ps : pl->passes) {
    if (ps.to_y) continue;
    Level& lv = pl->levels[ps.level];
    if (lv.W.alloc((size_t)lv.nclusters * R * ps.K_pad * sizeof(double))) return 1;
    if (lv.H.alloc((size_t)lv.nclusters * R * P * sizeof(double))) return 1;
  }
  pl->ws_R = R;
  return 0;
}

// Matvec phases.  local: permute own leaf boxes + upward of own source
// clusters into the exchange buffers (ub, W_l); remote: gathered GEMMs for the
// own target clusters + fused downward of the own leaf boxes.  Between them a
// multi-GPU caller all-gathers the exchange buffers (contiguous Morton chunks).
namespace {

// Host-vector pipeline of a banded plan (htlr_matvec_host): u arrives and f
// leaves in S z slabs of leaf boxes (contiguous in F-order) on a copy stream;
// the cube upward runs per slab as it lands, the cube downward per slab before its copy out.
struct HostPipe {
  int S = 0;                   // slabs
  int zu[5] = {}, zf[5] = {};  // slab bounds (leaf boxes along z) of u and of f
  size_t zrow = 0;             // doubles per leaf-box row along z (points x rhs)
  const double* uh = nullptr;  // caller's page-locked u / f
  double* fh = nullptr;
  cudaStream_t cs = nullptr;
  cudaEvent_t* ev = nullptr;   // 2 S + 2: fork, S landed, S written, join
};

struct MvCtx {
  htlr_plan* pl;
  cudaStream_t st;
  HostPipe* pipe = nullptr;
  bool zeroed = false;      // the permute launch zeroed the remote phase's accumulators
  bool whole = false;       // local and remote phase in one call (htlr_matvec): they may share the side stream
  bool side_forked = false; // the upward pass already runs on the side stream (mv_local forked it)
  int R, d, p, P;
  double* ub;
  std::vector<double*> W;   // per pass (nullptr for the leaf pass)
  std::vector<double*> Wl;  // mapped grid: per level
  size_t ev_used = 0;
  int64_t launches = 0;

  // inside a graph capture the event must be an external record node; on a
  // direct launch (sharded plans, graphs off) a plain record
  cudaError_t record(cudaEvent_t e) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal)
                                               : cudaEventRecord(e, st);
  }
  int prof_begin(int kind, int level, double flops, double bytes) {
    if (!pl->profiling) return 0;
    while (pl->prof_ev.size() < ev_used + 2) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      pl->prof_ev.push_back(e);
    }
    CUDA_TRY(record(pl->prof_ev[ev_used]));
    pl->prof_kind.push_back(kind);
    pl->prof_level.push_back(level);
    pl->prof_flops.push_back(flops);
    pl->prof_bytes.push_back(bytes);
    return 0;
  }
  int prof_end() {
    ++launches;
    if (!pl->profiling) return 0;
    CUDA_TRY(record(pl->prof_ev[ev_used + 1]));
    ev_used += 2;
    return 0;
  }
};

int mv_prepare(htlr_plan* pl, int64_t nrhs, void* stream, MvCtx& cx) {
  if (!pl) return fail(-1, "null plan");
  if (pl->device < 0) return fail(-1, "host-only plan: no device work");
  if (!pl->constructed) return fail(-1, "plan not constructed");
  if (nrhs < 1 || nrhs > 4096) return fail(-1, "nrhs must be in [1, 4096]");
  CUDA_TRY(cudaSetDevice(pl->device));
  cx.pl = pl;
  cx.st = (cudaStream_t)stream;
  cx.R = (int)nrhs;
  cx.d = pl->d;
  cx.p = pl->p;
  cx.P = ipow(pl->p, pl->d);
  if (ensure_workspace(pl, cx.R)) return 1;
  if (!pl->mapped) {
    // split upward of levels with few clusters (outside any graph capture:
    // a grown scratch invalidates the captured graphs)
    for (auto& ps : pl->passes) {
      if (ps.to_y) continue;
      Level& lv = pl->levels[ps.level];
      const int64_t nc = pl->own_hi[ps.level] - pl->own_lo[ps.level];
      lv.up_ns = lv.Kron.ptr ? 1 : htlr::upward_nslab(cx.d, lv.side, nc, cx.R);
      if (lv.up_ns <= 1) continue;
      const size_t sb = (size_t)nc * cx.R * lv.up_ns * cx.P * sizeof(double), cb = (size_t)nc * cx.R * sizeof(int);
      if (lv.up_scratch.bytes < sb || lv.up_count.bytes < cb) {
        drop_graphs(pl);
        if (lv.up_scratch.alloc(sb) || lv.up_count.alloc(cb)) return 1;
        CUDA_TRY(cudaMemset(lv.up_count.ptr, 0, lv.up_count.bytes));
      }
    }
  }
  for (auto& ps : pl->passes) {
    if (pl->sep || ps.tasks.count(cx.R)) continue;
    std::vector<htlr::GemmTask> tv;
    make_tasks(ps, cx.R, tv);
    auto& slot = ps.tasks[cx.R];
    if (slot.first.alloc(std::max<size_t>(1, tv.size()) * sizeof(htlr::GemmTask))) return 1;
    if (!tv.empty())
      CUDA_TRY(cudaMemcpy(slot.first.ptr, tv.data(), tv.size() * sizeof(htlr::GemmTask), cudaMemcpyHostToDevice));
    slot.second = (int)tv.size();
  }
  const bool ext = pl->ext_R == cx.R && !pl->ext_ptrs.empty();
  size_t xi = 0;
  cx.ub = (ext && !pl->zslab) ? pl->ext_ptrs[xi++] : pl->ub.d();
  cx.Wl.assign(pl->levels.size(), nullptr);
  if (pl->mapped) {
    for (size_t l = 0; l < pl->levels.size(); ++l)
      if (pl->levels[l].needs_up) cx.Wl[l] = ext ? pl->ext_ptrs[xi++] : pl->levels[l].W.d();
    return 0;
  }
  cx.W.assign(pl->passes.size(), nullptr);
  for (size_t i = 0; i < pl->passes.size(); ++i) {
    if (pl->passes[i].to_y) continue;
    cx.W[i] = ext ? pl->ext_ptrs[xi++] : pl->levels[pl->passes[i].level].W.d();
  }
  return 0;
}

void prof_reset(htlr_plan* pl) {
  pl->prof_kind.clear();
  pl->prof_level.clear();
  pl->prof_flops.clear();
  pl->prof_bytes.clear();
}

int mv_local_mapped(MvCtx& cx, const double* u) {
  htlr_plan* pl = cx.pl;
  const int d = cx.d, p = cx.p, P = cx.P, R = cx.R;
  const double R8 = 8.0 * R;
  const int PL = ipow(pl->sL, d);
  const int64_t b0 = pl->own_lo[pl->L], nb = pl->own_hi[pl->L] - b0;
  const double frac = (double)nb / (double)pl->levels[pl->L].nclusters;
  htlr::ZeroList zl;
  if (pl->shard_world == 1 && R == 1) {   // the symmetric levels accumulate with RED
    for (const auto& lv : pl->levels)
      if (lv.needs_up && lv.sym.on) {
        zl.p[zl.cnt] = lv.H.d();
        zl.n[zl.cnt++] = lv.nclusters * P;
      }
    cx.zeroed = true;
  }
  if (cx.zeroed && !pl->profiling) {   // one launch, as in mv_local
    htlr::PrologueParams pp{};
    pp.u = u;
    pp.ub = cx.ub;
    pp.d = d;
    pp.n = pl->n;
    pp.p = p;
    pp.sL = pl->sL;
    pp.R = R;
    pp.K_pad_leaf = PL;
    pp.b0 = b0;
    pp.nb_perm = nb;
    pp.zero = zl;
    bool fused = true;
    for (auto& lv : pl->levels) {
      if (!lv.needs_up) continue;
      if (pp.nlev >= htlr::kMaxLevels || htlr::upward_smem_words(d, lv.side, p) * sizeof(double) > 200 * 1024) {
        fused = false;
        break;
      }
      pp.lev[pp.nlev++] = htlr::UpLevel{cx.Wl[lv.level], lv.WLm.d(), (int64_t)lv.side * p, pl->own_lo[lv.level],
                                        pl->own_hi[lv.level] - pl->own_lo[lv.level], lv.side, lv.level, P};
    }
    if (fused) {
      htlr::launch_prologue(pp, cx.st);
      ++cx.launches;
      return 0;
    }
  }
  if (cx.prof_begin(0, pl->L, 0.0, 2.0 * R8 * (double)pl->N * frac)) return 1;
  htlr::launch_permute_in(u, cx.ub, d, pl->n, pl->sL, R, PL, b0, nb, cx.st, cx.zeroed ? &zl : nullptr);
  if (cx.prof_end()) return 1;
  for (auto& lv : pl->levels) {
    if (!lv.needs_up) continue;
    const int64_t c0 = pl->own_lo[lv.level], nc = pl->own_hi[lv.level] - c0;
    double s1 = lv.side;
    double macs = (d == 2) ? (p * s1 * s1 + (double)p * p * s1)
                           : (p * s1 * s1 * s1 + (double)p * p * s1 * s1 + (double)p * p * p * s1);
    if (cx.prof_begin(1, lv.level, 2.0 * macs * nc * R, R8 * ((double)pl->N * frac + (double)nc * P))) return 1;
    htlr::launch_upward(u, cx.Wl[lv.level], d, pl->n, lv.side, p, lv.level, R, P, lv.WLm.d(),
                        (int64_t)lv.side * p, c0, nc, cx.st);
    if (cx.prof_end()) return 1;
  }
  return 0;
}

// kernel sampling is counted as 10 flops per evaluation plus the MAC
// Accumulators of the mapped remote phase: H_l per level and Y, or the
// caller-bound full-size reduce buffers of a sharded symmetric plan.
static bool mapped_sym(const htlr_plan* pl, int R) {
  if (R != 1) return false;
  for (const auto& lv : pl->levels)
    if (lv.needs_up && lv.sym.on) return true;
  return pl->near_sym.on;
}

static void mapped_accumulators(htlr_plan* pl, int R, std::vector<double*>& H, double*& Y) {
  const bool bound = pl->shard_world > 1 && pl->red_R == R && !pl->red_ptrs.empty();
  size_t k = 0;
  H.assign(pl->levels.size(), nullptr);
  for (size_t l = 0; l < pl->levels.size(); ++l) {
    Level& lv = pl->levels[l];
    if (!lv.needs_up) continue;
    H[l] = (bound && lv.sym.on) ? pl->red_ptrs[k++] : lv.H.d();
  }
  Y = (bound && pl->near_sym.on) ? pl->red_ptrs[k++] : pl->Y.d();
}

// stages: bit 0 = contract (regenerated cores and near blocks into H_l, Y),
// bit 1 = expand (downward pass).  A sharded symmetric plan needs the shards'
// H_l / Y summed in between (htlr_reduce_info); otherwise stages = 3.
int mv_remote_mapped(MvCtx& cx, const double* u, double* f, int stages) {
  htlr_plan* pl = cx.pl;
  const int d = cx.d, p = cx.p, P = cx.P, R = cx.R;
  const int PL = ipow(pl->sL, d);
  const double R8 = 8.0 * R;
  const bool sharded = pl->shard_world > 1;
  std::vector<double*> Hl;
  double* Y = nullptr;
  mapped_accumulators(pl, R, Hl, Y);
  htlr::DownParams dp{};
  dp.nlev = 0;
  double down_macs = 0.0;
  const int64_t nleaf = pl->levels[pl->L].nclusters;
  const int64_t b0 = pl->own_lo[pl->L], nb = pl->own_hi[pl->L] - b0;
  for (auto& lv : pl->levels) {
    if (!lv.needs_up) continue;
    if (dp.nlev >= htlr::kMaxLevels) return fail(-1, "too many levels");
    dp.lev[dp.nlev++] = htlr::DownLevel{lv.level, lv.side, P, lv.Lm.d(), Hl[lv.level], (int64_t)lv.side * p, nullptr};
    double sl = pl->sL;
    down_macs += (d == 2) ? (sl * p * p + sl * sl * p) : (sl * p * p * p + sl * sl * p * p + sl * sl * sl * p);
    if (!(stages & 1)) continue;
    const int64_t t0 = pl->own_lo[lv.level], nt = pl->own_hi[lv.level] - t0;
    const double npair = (double)lv.csr_cols.size();
    // symmetric regeneration: one 10-flop evaluation per unordered pair
    const bool sym = lv.sym.on && R == 1;
    const double evals = sym ? 0.5 : 1.0;
    if (cx.prof_begin(5, lv.level, npair * P * P * (10.0 * evals + 2.0 * R), R8 * npair * P)) return 1;
    if (sym) {
      if (!cx.zeroed) CUDA_TRY(cudaMemsetAsync(Hl[lv.level], 0, (size_t)lv.nclusters * P * sizeof(double), cx.st));
      htlr::launch_regen_sym(pl->kp, p, lv.level, lv.nodes.d(), (const int*)lv.sym.order.ptr, lv.sym.nrows, t0,
                             (const int64_t*)lv.sym.uptr.ptr, (const int*)lv.sym.ucols.ptr, cx.Wl[lv.level], P,
                             Hl[lv.level], P, cx.st);
    } else {
      htlr::launch_regen_adm(pl->kp, d, p, lv.level, lv.nodes.d(), (const int64_t*)lv.d_ptr.ptr,
                             (const int*)lv.d_cols.ptr, t0, nt, cx.Wl[lv.level], P, Hl[lv.level], R, cx.st);
    }
    if (cx.prof_end()) return 1;
  }
  if (stages & 1) {
    const double npair = (double)pl->near_cols.size();
    const bool sym = pl->near_sym.on && R == 1;
    const double evals = sym ? 0.5 : 1.0;
    if (cx.prof_begin(6, pl->L, npair * PL * PL * (10.0 * evals + 2.0 * R), R8 * npair * PL)) return 1;
    if (sym) {
      // self pairs first (plain stores initialise the own rows of Y), then
      // the owned pairs, whose column sums may land in any leaf's rows
      if (sharded) CUDA_TRY(cudaMemsetAsync(Y, 0, (size_t)nleaf * PL * sizeof(double), cx.st));
      htlr::launch_regen_near(pl->kp, d, pl->sL, pl->L, pl->d_mx.d(), pl->d_mc.d(),
                              (const int64_t*)pl->d_self_ptr.ptr, (const int*)pl->d_self_cols.ptr, b0, nb, cx.ub,
                              PL, Y, R, cx.st);
      htlr::launch_near_weight(pl->sL, pl->L, pl->d_mc.d(), cx.ub, PL, pl->Vn.d(), nleaf, cx.st);
      htlr::launch_regen_sym(pl->kp, pl->sL, pl->L, pl->d_mx.d(), (const int*)pl->near_sym.order.ptr,
                             pl->near_sym.nrows, b0, (const int64_t*)pl->near_sym.uptr.ptr,
                             (const int*)pl->near_sym.ucols.ptr, pl->Vn.d(), PL, Y, PL, cx.st);
    } else {
      htlr::launch_regen_near(pl->kp, d, pl->sL, pl->L, pl->d_mx.d(), pl->d_mc.d(),
                              (const int64_t*)pl->d_near_ptr.ptr, (const int*)pl->d_near_cols.ptr, b0, nb, cx.ub,
                              PL, Y, R, cx.st);
    }
    if (cx.prof_end()) return 1;
  }
  if (stages & 2) {
    const double frac = (double)nb / (double)nleaf;
    if (cx.prof_begin(4, pl->L, 2.0 * down_macs * nb * R, R8 * 3.0 * (double)pl->N * frac)) return 1;
    htlr::launch_downward(u, f, Y, PL, pl->has_coeff ? pl->coeff.d() : nullptr, pl->desc.coeff_const,
                          pl->dvec.d(), d, pl->n, pl->sL, pl->L, R, p, dp, b0, nb, cx.st);
    if (cx.prof_end()) return 1;
  }
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Parameters of the fused prologue launch (permute + zeroing + every level's
// upward pass) of a uniform plan; false if a level cannot be fused.
bool prologue_params(MvCtx& cx, const double* u, const htlr::ZeroList& zl, htlr::PrologueParams& pp) {
  htlr_plan* pl = cx.pl;
  const int d = cx.d, p = cx.p;
  const Pass& lp = pl->passes[pl->leaf_pass];
  pp.u = u;
  pp.ub = cx.ub;
  pp.d = d;
  pp.n = pl->n;
  pp.p = p;
  pp.sL = pl->sL;
  pp.R = cx.R;
  pp.K_pad_leaf = lp.K_pad;
  pp.zpitch_leaf = lp.zpitch;
  pp.b0 = pl->own_lo[pl->L];
  pp.nb_perm = pl->own_hi[pl->L] - pp.b0;
  pp.zero = zl;
  for (size_t i = 0; i < pl->passes.size(); ++i) {
    const Pass& ps = pl->passes[i];
    if (ps.to_y) continue;
    const Level& lv = pl->levels[ps.level];
    if (lv.Kron.ptr || pp.nlev >= htlr::kMaxLevels ||
        htlr::upward_smem_words(d, lv.side, p) * sizeof(double) > 200 * 1024)
      return false;
    pp.lev[pp.nlev++] = htlr::UpLevel{cx.W[i],       lv.Q.d(),      0,
                                      pl->own_lo[ps.level], pl->own_hi[ps.level] - pl->own_lo[ps.level],
                                      lv.side,         lv.level,      ps.K_pad,
                                      lv.up_ns,        lv.up_ns > 1 ? lv.up_scratch.d() : nullptr,
                                      lv.up_ns > 1 ? (int*)lv.up_count.ptr : nullptr, ps.zpitch};
  }
  return true;
}

static void launch_band_sweep(htlr_plan* pl, const Pass& ps, int sweep, const double* B, double* C, int R,
                              cudaStream_t st, const double* u, int max_ctas, int zlo_o = -1, int zhi_o = -1);

// The banded leaf pass of an unsharded plan reads the F-order u itself (line /
// plane kernels over whole x-y planes), so nothing on the leaf pass's path
// waits for the upward pass: that runs on the side stream, before the level
// passes, beside the leaf z sweep -- and writes no permuted copy of u.
static bool leaf_from_u(const htlr_plan* pl, int R) {
  // several right-hand sides: u is [point][rhs], a line's points are R doubles
  // apart; the permuted boxes keep each rhs contiguous
  if (R != 1) return false;
  if (!pl->sep || pl->mapped || pl->d != 3 || pl->leaf_pass < 0) return false;
  const Pass& lp = pl->passes[pl->leaf_pass];
  const int nb = 1 << lp.level;
  return lp.band && lp.from_ub && htlr::band_lines_supported(lp.level) && lp.band_lo[0] == 0 && lp.band_lo[1] == 0 &&
         lp.band_hi[0] == nb && lp.band_hi[1] == nb;
}

int mv_local(MvCtx& cx, const double* u) {
  htlr_plan* pl = cx.pl;
  if (pl->mapped) return mv_local_mapped(cx, u);
  const int d = cx.d, p = cx.p, P = cx.P, R = cx.R;
  const double R8 = 8.0 * R;
  const Pass& lp = pl->passes[pl->leaf_pass];
  const int64_t b0 = pl->own_lo[pl->L], nb = pl->own_hi[pl->L] - b0;
  const double frac = (double)nb / (double)pl->levels[pl->L].nclusters;
  // unsharded plans: the permute launch also zeroes H_l and Y (one launch
  // instead of permute + a memset node per accumulator)
  htlr::ZeroList zl;
  if (pl->shard_world == 1) {
    for (const auto& ps : pl->passes) {
      if (ps.to_y) continue;
      const Level& lv = pl->levels[ps.level];
      zl.p[zl.cnt] = lv.H.d();
      zl.n[zl.cnt++] = lv.nclusters * R * P;
    }
    zl.p[zl.cnt] = pl->Y.d();
    zl.n[zl.cnt++] = pl->levels[pl->L].nclusters * R * lp.P;
    cx.zeroed = zl.cnt <= htlr::kMaxLevels + 2;
  }
  // separable plans (p = leaf side = 8): the permute and the upward pass of
  // every compressed level in one launch over cubes (htlr_cube.cu)
  htlr::CubeLevels cl;
  if (pl->shard_world == 1 && pl->sep && cx.zeroed && cube_params(pl, cx.W.data(), cl)) {
    // accumulators: W_l of the coarser levels (RED targets), W_{L-1} when a
    // z-slab shard stores only its own cubes (the ranks sum W_l), and those
    // of the passes that accumulate (the banded passes store every entry)
    htlr::ZeroList z2;
    for (int li = 0; li < cl.ncoarse; ++li) {
      z2.p[z2.cnt] = cl.lev[li].W;
      z2.n[z2.cnt++] = pl->levels[cl.lev[li].level].nclusters * R * cl.lev[li].K_pad;
    }
    if (cl.Qc && pl->zslab) {
      z2.p[z2.cnt] = cl.Wc;
      z2.n[z2.cnt++] = pl->levels[pl->L - 1].nclusters * R * cl.K_pad_c;
    }
    {
      int q = 0;
      for (const auto& ps : pl->passes) {
        if (ps.to_y) continue;
        if (!ps.band && z2.cnt < htlr::kMaxLevels + 2) z2.p[z2.cnt] = zl.p[q], z2.n[z2.cnt++] = zl.n[q];
        ++q;
      }
      if (!lp.band && z2.cnt < htlr::kMaxLevels + 2) z2.p[z2.cnt] = zl.p[q], z2.n[z2.cnt++] = zl.n[q];
    }
    // leaf pass reading u itself: no permuted copy, and (unprofiled, outside
    // the host pipeline) the zeroing and the upward pass go to the side stream
    const bool from_u = leaf_from_u(pl, R);
    double* const ub_out = from_u ? nullptr : cx.ub;
    cudaStream_t ust = cx.st;
    if (from_u && cx.whole && !pl->zslab && !pl->profiling && !cx.pipe) {
      if (!pl->side_stream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->side_stream, cudaStreamNonBlocking));
      for (auto& ev : pl->side_ev)
        if (!ev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(pl->side_ev[0], cx.st));
      CUDA_TRY(cudaStreamWaitEvent(pl->side_stream, pl->side_ev[0], 0));
      cx.side_forked = true;
      ust = pl->side_stream;
    }
    for (int q = 0; q < z2.cnt; ++q) CUDA_TRY(cudaMemsetAsync(z2.p[q], 0, (size_t)z2.n[q] * sizeof(double), ust));
    // algorithmic work per cube: 16^3 x 8 + 16^2 x 8^2 + 16 x 8^3 MAC (the
    // three mode products of W_{L-1}) + 3 x 8^4 per coarser level; bytes: u
    // read + ub written
    const double ncube = (double)nb / 8.0;
    const double flops = 2.0 * ncube * R * ((cl.Qc ? 57344.0 : 0.0) + 12288.0 * cl.ncoarse);
    if (cx.prof_begin(1, pl->L - 1, flops, 2.0 * R8 * (double)pl->N)) return 1;
    if (HostPipe* hp = cx.pipe) {
      // one launch per slab of u, each after its copy landed
      for (int k = 0; k < hp->S; ++k) {
        CUDA_TRY(cudaStreamWaitEvent(cx.st, hp->ev[1 + k], 0));
        htlr::launch_upward_cube(cl, pl->L, R, nb, cx.st, u, ub_out, lp.K_pad, lp.zpitch, pl->n, hp->zu[k],
                                 hp->zu[k + 1]);
      }
      cx.launches += hp->S;
      return 0;
    }
    if (pl->zslab && lp.band && !pl->profiling && !cx.pipe) {
      // z-slab shard: the whole leaf pass of the own slab beside the upward pass
      if (!pl->leaf_stream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->leaf_stream, cudaStreamNonBlocking));
      for (auto& ev : pl->leaf_ev)
        if (!ev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(pl->leaf_ev[0], cx.st));
      CUDA_TRY(cudaStreamWaitEvent(pl->leaf_stream, pl->leaf_ev[0], 0));
      for (int sw = 0; sw < 3; ++sw) launch_band_sweep(pl, lp, sw, cx.ub, pl->Y.d(), R, pl->leaf_stream, u, 0);
      CUDA_TRY(cudaEventRecord(pl->leaf_ev[1], pl->leaf_stream));
      pl->leaf_pending = true;
    }
    htlr::launch_upward_cube(cl, pl->L, R, nb, ust, u, ub_out, lp.K_pad, lp.zpitch, pl->n,
                             pl->zslab ? pl->zs_lo : 0, pl->zslab ? pl->zs_hi : 1 << 30);
    if (cx.prof_end()) return 1;
    cx.launches += 1;
    return 0;
  }
  if (cx.pipe) return fail(2, "host pipeline: cube upward not applicable");
  // unprofiled unsharded matvec: permute + zeroing + every level's upward in
  // one launch (profiling keeps them apart so each phase is timed)
  if (cx.zeroed && !pl->profiling) {
    htlr::PrologueParams pp{};
    if (prologue_params(cx, u, zl, pp)) {
      htlr::launch_prologue(pp, cx.st);
      ++cx.launches;
      return 0;
    }
  }
  if (cx.prof_begin(0, pl->L, 0.0, 2.0 * R8 * (double)pl->N * frac)) return 1;
  htlr::launch_permute_in(u, cx.ub, d, pl->n, pl->sL, R, lp.K_pad, b0, nb, cx.st, cx.zeroed ? &zl : nullptr,
                          lp.zpitch);
  if (cx.prof_end()) return 1;
  for (size_t i = 0; i < pl->passes.size(); ++i) {
    const Pass& ps = pl->passes[i];
    if (ps.to_y) continue;
    Level& lv = pl->levels[ps.level];
    const int64_t c0 = pl->own_lo[ps.level], nc = pl->own_hi[ps.level] - c0;
    double s1 = lv.side;
    double macs = (d == 2) ? (p * s1 * s1 + (double)p * p * s1)
                           : (p * s1 * s1 * s1 + (double)p * p * s1 * s1 + (double)p * p * p * s1);
    if (cx.prof_begin(1, lv.level, 2.0 * macs * nc * R, R8 * ((double)pl->N * frac + (double)nc * P))) return 1;
    if (lv.Kron.ptr)
      htlr::launch_dense_upward(u, cx.W[i], d, pl->n, lv.side, p, lv.level, R, ps.K_pad, lv.Kron.d(), c0, nc, cx.st);
    else
      htlr::launch_upward(u, cx.W[i], d, pl->n, lv.side, p, lv.level, R, ps.K_pad, lv.Q.d(), 0, c0, nc, cx.st,
                          lv.up_ns, lv.up_scratch.d(), (int*)lv.up_count.ptr, ps.zpitch);
    if (cx.prof_end()) return 1;
  }
  return 0;
}

// SMs the leaf z sweep leaves to the passes running beside it on the side
// stream: the level passes (20), or the upward pass and the level passes
// (48: the z sweep is bound by its memory traffic, not by its SM count, and
// the upward pass then ends with it; measured 20 / 40 / 48 / 56 / 64: config
// 4's step 0.1307 (upward first, on the main stream) / 0.1323 / 0.1280 /
// 0.1286 / 0.1284 ms)
static int level_sms(bool with_upward) { return with_upward ? 48 : 20; }

// One sweep of a banded pass (0: z sweep, 1: the fused y-x sweep; 2: the
// legacy separate x sweep, a no-op for the line/plane kernels).  Regions that
// are whole in x and y (unsharded, or a z-slab shard) run the register-line
// kernels (htlr_band.cu) over the region's z boxes; the leaf pass reads the
// F-order u itself (no permuted copy).  Octant regions of Morton-sharded
// plans keep the staged sweeps of htlr_sep.cu.
static void launch_band_sweep(htlr_plan* pl, const Pass& ps, int sweep, const double* B, double* C, int R,
                              cudaStream_t st, const double* u, int max_ctas, int zlo_o, int zhi_o) {
  const int nb = 1 << ps.level;
  // target z boxes: the pass's region, or a part of it (host pipeline)
  const int zlo = zlo_o >= 0 ? zlo_o : ps.band_lo[2], zhi = zhi_o >= 0 ? zhi_o : ps.band_hi[2];
  const bool xy_full = ps.band_lo[0] == 0 && ps.band_lo[1] == 0 && ps.band_hi[0] == nb && ps.band_hi[1] == nb;
  const double* corr = ps.to_y ? pl->sep_corr.d() : nullptr;
  const int nterms = ps.to_y ? 6 : 4;
  if (xy_full && htlr::band_lines_supported(ps.level)) {
    // sharded plans: u itself (every rank holds it; the permuted copy covers
    // the own boxes only); unsharded: the permuted boxes the cube upward wrote (the
    // pitched box rows load with fewer address instructions: 108 vs 115 us)
    const bool fo = ps.from_ub && u != nullptr && (pl->shard_world > 1 || pl->zslab || leaf_from_u(pl, R));
    const double* src = fo ? u : B;
    const int n = fo ? pl->n : 0;
    if (sweep == 0)
      htlr::launch_band_lines(ps.level, nterms, ps.sep_tab.d(), ps.sep_NO, R, src, ps.K_pad, ps.zpitch,
                              ps.band_ws.d(), st, n, zlo, zhi, max_ctas);
    else if (sweep == 1 && band_xy_lines(pl))
      htlr::launch_band_ylines(ps.level, nterms, ps.sep_tab.d(), ps.sep_NO, R, ps.band_ws.d(), ps.band_ws2.d(), C, src,
                               ps.K_pad, ps.zpitch, n, corr, pl->kp.scale, st, zlo, zhi);
    else if (sweep == 1)
      htlr::launch_band_planes(ps.level, nterms, ps.sep_tab.d(), ps.sep_NO, R, src, ps.K_pad, ps.zpitch,
                               ps.band_ws.d(), C, corr, pl->kp.scale, st, n, zlo, zhi, ps.to_y ? pl->f_red : nullptr,
                               pl->n);
    return;
  }
  htlr::launch_sep_band(sweep, ps.sep_tab.d(), ps.sep_NO, ps.level, R, B, ps.K_pad, ps.zpitch, ps.band_ws.d(), C, corr,
                        pl->kp.scale, nterms, st, ps.band_lo, ps.band_hi);
}

int mv_remote(MvCtx& cx, const double* u, double* f, int stages = 3) {
  htlr_plan* pl = cx.pl;
  if (pl->mapped) return mv_remote_mapped(cx, u, f, stages);
  const int d = cx.d, p = cx.p, P = cx.P, R = cx.R;
  const double R8 = 8.0 * R;
  const Pass& lp = pl->passes[pl->leaf_pass];
  const int64_t nleaf = pl->levels[pl->L].nclusters;
  // stages: 1 contract, 2 expand; 4 = contract only the separable parts over
  // own sources (+ the zeroing), 8 = contract the rest without zeroing
  // (htlr_matvec_remote_begin / _finish: the exchange overlaps the first)
  const bool own_only = (stages & 4) != 0, rest_only = (stages & 8) != 0;
  for (auto& ps : pl->passes) {
    if (!(stages & 1) || cx.zeroed || rest_only) break;
    if (ps.to_y) continue;
    Level& lv = pl->levels[ps.level];
    CUDA_TRY(cudaMemsetAsync(lv.H.ptr, 0, (size_t)lv.nclusters * R * P * sizeof(double), cx.st));
  }
  if ((stages & 1) && !cx.zeroed && !rest_only && !pl->leaf_pending)
    CUDA_TRY(cudaMemsetAsync(pl->Y.ptr, 0, (size_t)nleaf * R * lp.P * sizeof(double), cx.st));
  // The level passes (-> H_l) and the leaf pass (-> Y) are independent: the
  // level passes go to a side stream (a parallel branch of the graph), so
  // they fill the SMs the leaf pass leaves idle (its tail rounds).  Serial
  // when profiling (per-launch events on one stream).
  bool fork = false;
  if ((stages & 1) && !pl->profiling) {
    int nlev = 0;
    for (const auto& ps : pl->passes) nlev += ps.to_y ? 0 : 1;
    fork = nlev > 0;
  }
  if (fork) {
    if (!pl->side_stream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->side_stream, cudaStreamNonBlocking));
    for (auto& ev : pl->side_ev)
      if (!ev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  // banded leaf pass: the fork first, then its z sweep on all but
  // level_sms SMs, which the upward and level passes (side stream) run on meanwhile; they
  // go on filling the SMs the y-x sweep leaves idle (128 planes on 148 SMs)
  bool leaf_z_done = false;
  if (fork && !cx.side_forked) {
    CUDA_TRY(cudaEventRecord(pl->side_ev[0], cx.st));
    CUDA_TRY(cudaStreamWaitEvent(pl->side_stream, pl->side_ev[0], 0));
  }
  // Host pipeline: the leaf pass in two parts on its own stream.  The target
  // boxes z < za reach no source in the last slab of u, so their sweeps start
  // when the slab before it has landed and run under the last slab's copy;
  // the rest starts when the last slab has landed.  The first slabs of f need
  // only the first part (and the level passes) before their downward pass.
  int pipe_za = 0;
  if (cx.pipe && fork && !own_only && !rest_only && !pl->leaf_pending && pl->sep && leaf_from_u(pl, R)) {
    HostPipe* hp = cx.pipe;
    const Pass& lq = pl->passes[pl->leaf_pass];
    const int nbz = 1 << lq.level;
    const int za = hp->S >= 2 ? ((hp->zu[hp->S - 1] - 5) & ~1) : 0;
    if (za >= 2 && za < nbz) {
      if (!pl->leaf_stream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->leaf_stream, cudaStreamNonBlocking));
      for (auto& ev : pl->leaf_ev)
        if (!ev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CUDA_TRY(cudaStreamWaitEvent(pl->leaf_stream, hp->ev[1 + hp->S - 2], 0));
      for (int sw = 0; sw < 2; ++sw) launch_band_sweep(pl, lq, sw, cx.ub, pl->Y.d(), R, pl->leaf_stream, u, 0, 0, za);
      CUDA_TRY(cudaEventRecord(pl->leaf_ev[0], pl->leaf_stream));
      CUDA_TRY(cudaStreamWaitEvent(pl->leaf_stream, hp->ev[1 + hp->S - 1], 0));
      for (int sw = 0; sw < 2; ++sw) launch_band_sweep(pl, lq, sw, cx.ub, pl->Y.d(), R, pl->leaf_stream, u, 0, za, nbz);
      CUDA_TRY(cudaEventRecord(pl->leaf_ev[1], pl->leaf_stream));
      cx.launches += 4;
      pipe_za = za;
    }
  }
  if (fork && !own_only && !rest_only && !pl->leaf_pending && !pipe_za) {
    const Pass& lq = pl->passes[pl->leaf_pass];
    if (pl->sep && lq.band) {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pl->device);
      launch_band_sweep(pl, lq, 0, cx.ub, pl->Y.d(), R, cx.st, u, sms - level_sms(cx.side_forked));
      leaf_z_done = true;
    }
  }
  // Direct f: nothing but the downward pass reads Y, and f = Y + (expansion of
  // H_eff) + a u is a sum of two independent parts.  With f zeroed, the plane
  // kernel adds the leaf pass's share straight into the F-order f and the cube
  // downward adds the rest, both with fp64 REDs (0 + a + b: the same value in
  // either order) -- so the downward pass leaves the critical path: it runs
  // on the side stream after the level passes, beside the leaf y-x sweep, and
  // Y is neither written nor read.
  bool fdirect = false;
  htlr::CubeLevels fcl;
  if (leaf_z_done && (stages & 2) && !cx.pipe && pl->shard_world == 1 && !pl->zslab && !band_xy_lines(pl) &&
      fdirect_enabled()) {
    const Pass& lq = pl->passes[pl->leaf_pass];
    const int nbx = 1 << lq.level;
    const bool planes = htlr::band_lines_supported(lq.level) && lq.band_lo[0] == 0 && lq.band_lo[1] == 0 &&
                        lq.band_hi[0] == nbx && lq.band_hi[1] == nbx && lq.band_lo[2] == 0 && lq.band_hi[2] == nbx;
    if (planes && lq.P == htlr::kSepP * htlr::kSepP * htlr::kSepP && cube_params(pl, nullptr, fcl)) {
      // a third stream, forked behind the upward pass: the zeroing of f and
      // the cooperative (non-banded) level passes run beside the banded ones
      if (!pl->fz_ev) CUDA_TRY(cudaEventCreateWithFlags(&pl->fz_ev, cudaEventDisableTiming));
      for (auto& ev : pl->fd_ev)
        if (!ev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      if (!pl->leaf_stream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->leaf_stream, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventRecord(pl->fd_ev[0], pl->side_stream));
      CUDA_TRY(cudaStreamWaitEvent(pl->leaf_stream, pl->fd_ev[0], 0));
      CUDA_TRY(cudaMemsetAsync(f, 0, (size_t)pl->N * R * sizeof(double), pl->leaf_stream));
      CUDA_TRY(cudaEventRecord(pl->fz_ev, pl->leaf_stream));
      fdirect = true;
    }
  }
  for (size_t i = 0; i < pl->passes.size() && (stages & 1); ++i) {
    Pass& ps = pl->passes[i];
    if (ps.to_y && pl->leaf_pending) continue;   // started by the local phase (z-slab shards)
    if (ps.to_y && pipe_za) continue;            // running in two parts on the leaf stream (host pipeline)
    // level passes on the side stream; with the leaf pass already running
    // elsewhere (z-slab shards, host pipeline) the main stream is free, so
    // they alternate between the two
    cudaStream_t sst = (fork && !ps.to_y && !((pl->leaf_pending || pipe_za) && (i & 1))) ? pl->side_stream : cx.st;
    if (fdirect && !ps.to_y && !ps.band) sst = pl->leaf_stream;
    if (!pl->sep && own_only) continue;   // dense passes all run after the exchange
    if (pl->sep) {
      if (ps.band && own_only) continue;   // the sweeps need every (gathered) source box
      if (ps.band) {
        const double* B = cx.ub;   // the banded passes are built for the leaf level and level passes alike
        if (!ps.from_ub) B = cx.W[i];
        double* C = ps.to_y ? pl->Y.d() : pl->levels[ps.level].H.d();
        // banded pass: a z sweep and the fused y-x sweep; algorithmic work =
        // the mode products they run; HBM bytes: the source vectors, the term
        // buffers written and read back, the accumulator read and written
        const double nv = R8 * (double)ps.P * (double)pl->levels[ps.level].nclusters;
        const double nterm = ps.to_y ? 6.0 : 4.0;
        // profiled per kernel: the z sweep (kind 9: reads the sources, writes
        // the term buffers) and the y-x sweep (kind 10: reads the term buffers
        // and the self pairs' sources, writes the accumulator)
        double zs = 0.0;
        band_flops_of(ps.level, ps.to_y, 1, &zs);
        if (ps.to_y && fdirect) {
          CUDA_TRY(cudaStreamWaitEvent(sst, pl->fz_ev, 0));
          pl->f_red = f;
        }
        for (int sw = (ps.to_y && leaf_z_done) ? 1 : 0; sw < 3; ++sw) {
          if (sw == 0 && cx.prof_begin(9, ps.level, zs * ps.band_flops * R, nv * (1.0 + nterm))) return 1;
          if (sw == 1 && cx.prof_begin(10, ps.level, (1.0 - zs) * ps.band_flops * R, nv * (nterm + 2.0))) return 1;
          launch_band_sweep(pl, ps, sw, B, C, R, sst, u, 0);
          if (sw == 0 && cx.prof_end()) return 1;
          if (sw == 2 && cx.prof_end()) return 1;
        }
        pl->f_red = nullptr;
        continue;
      }
      if (ps.sep_nitems == 0 && ps.sep_nblocks == 0) continue;
      // part range of this stage (per-warp items: everything in the rest stage)
      int b0 = 0, nbk = ps.sep_nblocks;
      if (own_only) nbk = ps.sep_nblocks > 0 ? ps.sep_own_nb : 0;
      if (rest_only) {
        b0 = ps.sep_nblocks > 0 ? ps.sep_own_nb : 0;
        nbk = ps.sep_nblocks - b0;
      }
      if (ps.sep_nblocks > 0 && nbk == 0) continue;
      if (ps.sep_nblocks == 0 && own_only) continue;
      const double* B = ps.from_ub ? cx.ub : cx.W[i];
      double* C = ps.to_y ? pl->Y.d() : pl->levels[ps.level].H.d();
      // algorithmic work: 8^4 MAC per pair (mode z) + 2 * 8^4 per group
      // (modes x, y); HBM bytes: the level's source vectors and accumulators
      // once (the per-pair gathers are L2 traffic) + the factor tables
      const double ncl = (double)pl->levels[ps.level].nclusters;
      const double m4 = 4096.0;
      const double share =
          own_only ? ps.sep_own_frac : (rest_only && ps.sep_nblocks > 0) ? 1.0 - ps.sep_own_frac : 1.0;
      const double flops = share * 2.0 * m4 * ((double)ps.npairs + 2.0 * (double)ps.sep_groups) * R;
      const double bytes = 2.0 * R8 * (double)ps.P * ncl + 8.0 * 2 * ps.sep_NO * htlr::kSepSlot;
      if (cx.prof_begin(ps.to_y ? 8 : 7, ps.level, flops, bytes)) return 1;
      if (ps.sep_nblocks > 0)
        htlr::launch_sep_block(ps.sep_tab.d(), 2 * ps.sep_NO, ps.sep_NO,
                               (const htlr::SepBlock*)ps.sep_blocks.ptr + b0, nbk,
                               (const htlr::SepCol*)ps.sep_cols.ptr, B, ps.K_pad, C, ps.P, R, pl->sep_corr.d(), sst,
                               ps.zpitch);
      else
        htlr::launch_sep_apply(ps.sep_tab.d(), 2 * ps.sep_NO, ps.sep_NO, (const htlr::SepItem*)ps.sep_items.ptr,
                               ps.sep_nitems, (const int2*)ps.sep_pairs.ptr, B, ps.K_pad, C, ps.P, R,
                               pl->sep_corr.d(), sst, ps.zpitch);
      if (cx.prof_end()) return 1;
      continue;
    }
    auto& slot = ps.tasks[R];
    if (slot.second == 0) continue;
    const int NT = ps.task_nt[R];
    const int Rc = std::min(R, NT);
    const double* B = ps.from_ub ? cx.ub : cx.W[i];
    double* C = ps.to_y ? pl->Y.d() : pl->levels[ps.level].H.d();
    // algorithmic work: 2 P^2 per (pair, rhs); HBM bytes: every unique
    // matrix once + the level's source vectors B and accumulators C once (the
    // per-pair gathers of B are L2 traffic)
    const double ncl = (double)pl->levels[ps.level].nclusters;
    const bool gen = ps.gen.ptr && ps.MT == 128 && NT == 32;   // A generated from Toeplitz generators
    const double mat_bytes = gen ? 8.0 * htlr::kGenStride : 8.0 * (double)ps.P * ps.P;
    double flops = 2.0 * (double)ps.P * ps.P * (double)ps.npairs * R;
    double bytes = mat_bytes * ps.nmats + 2.0 * R8 * (double)ps.P * ncl;
    if (cx.prof_begin(ps.to_y ? 3 : 2, ps.level, flops, bytes)) return 1;
    htlr::launch_gemm(ps.MT, NT, ps.table.d(), ps.mat_stride, B, C, (const htlr::GemmTask*)slot.first.ptr,
                      slot.second, (const int2*)ps.pairs.ptr, R, Rc, ps.K_pad, ps.P, ps.P, ps.RT, sst,
                      ps.gen.ptr ? ps.gen.d() : nullptr);
    if (cx.prof_end()) return 1;
  }
  if (fdirect) {
    CUDA_TRY(cudaEventRecord(pl->fd_ev[1], pl->leaf_stream));
    CUDA_TRY(cudaStreamWaitEvent(pl->side_stream, pl->fd_ev[1], 0));
    const int64_t fb0 = pl->own_lo[pl->L], fnb = pl->own_hi[pl->L] - fb0;
    htlr::launch_downward_cube(fcl, pl->L, R, fb0, fnb, pl->side_stream, u, f, nullptr,
                               pl->has_coeff ? pl->coeff.d() : nullptr, pl->desc.coeff_const, pl->n, 0, 1 << 30, true);
    ++cx.launches;
  }
  if (fork || cx.side_forked) {
    CUDA_TRY(cudaEventRecord(pl->side_ev[1], pl->side_stream));
    CUDA_TRY(cudaStreamWaitEvent(cx.st, pl->side_ev[1], 0));
  }
  if (fdirect) {
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  if (pl->leaf_pending && (stages & 1)) {
    CUDA_TRY(cudaStreamWaitEvent(cx.st, pl->leaf_ev[1], 0));
    pl->leaf_pending = false;
  }
  htlr::DownParams dp{};
  dp.nlev = 0;
  double down_macs = 0.0;
  for (auto& ps : pl->passes) {
    if (ps.to_y) continue;
    Level& lv = pl->levels[ps.level];
    if (dp.nlev >= htlr::kMaxLevels) return fail(-1, "too many levels");
    dp.lev[dp.nlev++] = htlr::DownLevel{lv.level, lv.side, P, lv.Q.d(), lv.H.d(), 0, lv.Kron.d()};
    double sl = pl->sL;
    down_macs += (d == 2) ? (sl * p * p + sl * sl * p) : (sl * p * p * p + sl * sl * p * p + sl * sl * sl * p);
  }
  const int64_t b0 = pl->own_lo[pl->L], nb = pl->own_hi[pl->L] - b0;
  const double frac = (double)nb / (double)nleaf;
  if (!(stages & 2)) return 0;
  if (cx.prof_begin(4, pl->L, 2.0 * down_macs * nb * R, R8 * 3.0 * (double)pl->N * frac)) return 1;
  htlr::CubeLevels cl;
  const bool cube = lp.P == htlr::kSepP * htlr::kSepP * htlr::kSepP && cube_params(pl, nullptr, cl);
  const double* av = pl->has_coeff ? pl->coeff.d() : nullptr;
  if (HostPipe* hp = cx.pipe) {
    if (!cube) return fail(2, "host pipeline: cube downward not applicable");
    // one launch per slab of f, each copied out while the next is computed
    bool joined_b = false;
    if (pipe_za) CUDA_TRY(cudaStreamWaitEvent(cx.st, pl->leaf_ev[0], 0));
    for (int k = 0; k < hp->S; ++k) {
      if (pipe_za && hp->zf[k + 1] > pipe_za && !joined_b) {
        CUDA_TRY(cudaStreamWaitEvent(cx.st, pl->leaf_ev[1], 0));
        joined_b = true;
      }
      htlr::launch_downward_cube(cl, pl->L, R, b0, nb, cx.st, u, f, pl->Y.d(), av, pl->desc.coeff_const, pl->n,
                                 hp->zf[k], hp->zf[k + 1]);
      CUDA_TRY(cudaEventRecord(hp->ev[1 + hp->S + k], cx.st));
      CUDA_TRY(cudaStreamWaitEvent(hp->cs, hp->ev[1 + hp->S + k], 0));
      const size_t o = hp->zf[k] * hp->zrow, c = (hp->zf[k + 1] - hp->zf[k]) * hp->zrow;
      CUDA_TRY(cudaMemcpyAsync(hp->fh + o, f + o, c * sizeof(double), cudaMemcpyDefault, hp->cs));
    }
    cx.launches += hp->S;
    if (pipe_za && !joined_b) CUDA_TRY(cudaStreamWaitEvent(cx.st, pl->leaf_ev[1], 0));
    CUDA_TRY(cudaEventRecord(hp->ev[2 * hp->S + 1], hp->cs));
    CUDA_TRY(cudaStreamWaitEvent(cx.st, hp->ev[2 * hp->S + 1], 0));
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  if (cube)
    htlr::launch_downward_cube(cl, pl->L, R, b0, nb, cx.st, u, f, pl->Y.d(), av, pl->desc.coeff_const, pl->n,
                               pl->zslab ? pl->zs_lo : 0, pl->zslab ? pl->zs_hi : 1 << 30);
  else
    htlr::launch_downward(u, f, pl->Y.d(), lp.P, pl->has_coeff ? pl->coeff.d() : nullptr, pl->desc.coeff_const,
                          nullptr, d, pl->n, pl->sL, pl->L, R, p, dp, b0, nb, cx.st);
  if (cx.prof_end()) return 1;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace

// The capture stream has the highest priority, the side stream the default
// (lowest): captured kernel nodes keep their stream's priority, so when the
// leaf z sweep and the upward pass become ready together the z sweep's CTAs
// are placed first and the upward pass takes the SMs it leaves.
static cudaError_t make_cap_stream(cudaStream_t* st) {
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  return cudaStreamCreateWithPriority(st, cudaStreamNonBlocking, greatest);
}

static void drop_graphs(htlr_plan* pl) {
  for (auto& g : pl->graph_cache) cudaGraphExecDestroy(g.exec);
  pl->graph_cache.clear();
  for (auto& g : pl->host_graphs) cudaGraphExecDestroy(g.exec);
  pl->host_graphs.clear();
}

int htlr_matvec(htlr_plan* pl, const double* u, double* f, int64_t nrhs, void* stream) {
  MvCtx cx;
  if (int rc = mv_prepare(pl, nrhs, stream, cx)) return rc;
  if (!u || !f) return fail(-1, "null vector");
  if (pl->shard_world > 1 || (pl->zslab && pl->zs_world > 1))
    return fail(-1, "sharded plan: use htlr_matvec_local / exchange / htlr_matvec_remote");
  if (pl->graphs) {
    // replay a captured graph of the whole launch sequence (one CPU call
    // instead of ~10 launches + memsets), keyed by the caller's u / f.  A
    // miss captures the sequence again; up to kGraphsPerShape graphs of one
    // shape are kept, beyond that the least recently used one has its
    // parameters rewritten in place (cudaGraphExecUpdate: pointer changes
    // only, no re-instantiation) -- callers that rotate many buffers pay one
    // capture per call, never a D2D copy of u or f.
    constexpr int kGraphsPerShape = 4;
    for (auto& g : pl->graph_cache) {
      if (g.R == cx.R && g.u == u && g.f == f && g.prof == pl->profiling) {
        g.stamp = ++pl->graph_clock;
        pl->prof_kind = g.kind;
        pl->prof_level = g.level;
        pl->prof_flops = g.flops;
        pl->prof_bytes = g.bytes;
        CUDA_TRY(cudaGraphLaunch(g.exec, cx.st));
        pl->last_launches = g.launches;
        return 0;
      }
    }
    if (!pl->cap_stream) CUDA_TRY(make_cap_stream(&pl->cap_stream));
    MvCtx cc = cx;
    cc.st = pl->cap_stream;
    cc.whole = true;
    prof_reset(pl);
    CUDA_TRY(cudaStreamBeginCapture(cc.st, cudaStreamCaptureModeThreadLocal));
    int rc = mv_local(cc, u);
    if (!rc) rc = mv_remote(cc, u, f);
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(cc.st, &graph);
    if (!rc && ce == cudaSuccess && graph) {
      htlr_plan::GraphEntry* hit = nullptr;
      int same = 0;
      for (auto& g : pl->graph_cache) {
        if (g.R != cx.R || g.prof != pl->profiling) continue;
        ++same;
        if (!hit || g.stamp < hit->stamp) hit = &g;
      }
      if (hit && same >= kGraphsPerShape) {
        cudaGraphExecUpdateResultInfo info{};
        if (cudaGraphExecUpdate(hit->exec, graph, &info) != cudaSuccess) {
          cudaGetLastError();
          hit = nullptr;
        }
      } else {
        hit = nullptr;
      }
      cudaGraphExec_t exec = nullptr;
      if (!hit && cudaGraphInstantiate(&exec, graph, cudaGraphInstantiateFlagUseNodePriority) == cudaSuccess) {
        if (pl->graph_cache.size() >= 8) drop_graphs(pl);
        pl->graph_cache.push_back({cx.R, u, f, pl->profiling, exec, {}, {}, {}, {}, 0});
        hit = &pl->graph_cache.back();
      }
      if (hit) {
        cudaGraphDestroy(graph);
        hit->u = u;
        hit->f = f;
        hit->kind = pl->prof_kind;
        hit->level = pl->prof_level;
        hit->flops = pl->prof_flops;
        hit->bytes = pl->prof_bytes;
        hit->launches = cc.launches;
        hit->stamp = ++pl->graph_clock;
        CUDA_TRY(cudaGraphLaunch(hit->exec, cx.st));
        pl->last_launches = cc.launches;
        return 0;
      }
    }
    // capture not possible here: fall back to direct launches from now on
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    pl->graphs = false;
    if (rc > 0) return rc;
  }
  prof_reset(pl);
  cx.whole = true;
  if (int rc = mv_local(cx, u)) return rc;
  if (int rc = mv_remote(cx, u, f)) return rc;
  pl->last_launches = cx.launches;
  return 0;
}

// ---------------------------------------------------------------------------
// Host-vector matvec with the PCIe copies overlapped (unsharded separable
// plans).  u and f are cut at z-slab boundaries of leaf boxes (contiguous in
// F-order, S = 4 slabs): the first slab of u is copied in alone; the device
// permutes its boxes and runs the leaf pass over its sources (~1/S of the
// work) while the rest of u is copied on a copy stream; then the remaining
// prologue, the level passes, the leaf pass for the targets before the last
// slab and their downward pass; their f is copied out while the last slab's
// targets run; the last slab of f goes last.  Captured once per (nrhs, host
// pointers) into a two-stream graph.
// ---------------------------------------------------------------------------
static bool overlap_ok(const htlr_plan* pl) {
  if (!pl->sep || pl->mapped || pl->shard_world != 1 || pl->d != 3 || !pl->graphs) return false;

  for (const auto& ps : pl->passes) {
    if (ps.sep_nblocks == 0) return false;
    if (ps.to_y && ps.sep_slabs == 0) return false;
    if (ps.band) return false;   // the banded sweeps read whole lines of boxes
    // the slab prologues are launches of the fused prologue kernel
    if (!ps.to_y && htlr::upward_smem_words(pl->d, pl->levels[ps.level].side, pl->p) * sizeof(double) > 200 * 1024)
      return false;
  }
  return true;
}

namespace {

int mv_overlap(MvCtx& cx, const double* uh, double* fh, cudaStream_t cs) {
  htlr_plan* pl = cx.pl;
  const int R = cx.R, P = cx.P;
  const Pass& lp = pl->passes[pl->leaf_pass];
  const int S = lp.sep_slabs;
  const int mz = pl->levels[pl->L].m, zs = mz / S;   // leaf boxes per axis / per slab
  const int64_t Ns = pl->N / S;                      // points per slab (contiguous in F-order)
  double* us = pl->u_stage.d();
  double* fs = pl->f_stage.d();
  if (pl->ov_ev.size() < 6 || lp.sep_gcount.size() != 3) return fail(2, "overlapped matvec: not prepared");
  cudaEvent_t* ev = pl->ov_ev.data();
  const size_t first = (size_t)Ns * R, rest = (size_t)(pl->N - Ns) * R, last = first;
  const size_t lead = (size_t)(pl->N - Ns) * R;     // points before the last slab
  // u: the first slab, then the rest, on the copy stream
  CUDA_TRY(cudaEventRecord(ev[0], cx.st));
  CUDA_TRY(cudaStreamWaitEvent(cs, ev[0], 0));
  CUDA_TRY(cudaMemcpyAsync(us, uh, first * sizeof(double), cudaMemcpyDefault, cs));
  CUDA_TRY(cudaEventRecord(ev[1], cs));
  CUDA_TRY(cudaMemcpyAsync(us + first, uh + first, rest * sizeof(double), cudaMemcpyDefault, cs));
  CUDA_TRY(cudaEventRecord(ev[2], cs));
  htlr::ZeroList zl;
  for (const auto& ps : pl->passes) {
    if (ps.to_y) continue;
    const Level& lv = pl->levels[ps.level];
    zl.p[zl.cnt] = lv.H.d();
    zl.n[zl.cnt++] = lv.nclusters * R * P;
  }
  zl.p[zl.cnt] = pl->Y.d();
  zl.n[zl.cnt++] = pl->levels[pl->L].nclusters * R * lp.P;
  auto leaf_range = [&](int g) {
    int off = 0;
    for (int q = 0; q < g; ++q) off += lp.sep_gcount[q];
    if (lp.sep_gcount[g] == 0) return;
    htlr::launch_sep_block(lp.sep_tab.d(), 2 * lp.sep_NO, lp.sep_NO, (const htlr::SepBlock*)lp.sep_gblocks.ptr + off,
                           lp.sep_gcount[g], (const htlr::SepCol*)lp.sep_gcols.ptr, cx.ub, lp.K_pad, pl->Y.d(), lp.P,
                           R, pl->sep_corr.d(), cx.st, lp.zpitch);
    ++cx.launches;
  };
  auto prologue = [&](int zlo, int zhi, const htlr::ZeroList& z) -> int {
    htlr::PrologueParams pp{};
    if (!prologue_params(cx, us, z, pp)) return fail(2, "overlapped matvec: prologue not fusable");
    pp.zlo = zlo;
    pp.zhi = zhi;
    htlr::launch_prologue(pp, cx.st);
    ++cx.launches;
    return 0;
  };
  // first slab: its boxes (and the accumulators zeroed), the clusters it
  // completes, the leaf pass over its sources while the rest is copied
  CUDA_TRY(cudaStreamWaitEvent(cx.st, ev[1], 0));
  if (prologue(0, zs, zl)) return 1;
  leaf_range(0);
  // the rest: boxes, upward passes, level passes, the leaf pass for the
  // targets before the last slab, their f copied out while the last slab's
  // targets run
  CUDA_TRY(cudaStreamWaitEvent(cx.st, ev[2], 0));
  if (prologue(zs, mz, htlr::ZeroList())) return 1;
  // level passes on the side stream, next to the leaf pass (joined before the
  // downward passes)
  if (!pl->side_stream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->side_stream, cudaStreamNonBlocking));
  for (auto& e : pl->side_ev)
    if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(pl->side_ev[0], cx.st));
  CUDA_TRY(cudaStreamWaitEvent(pl->side_stream, pl->side_ev[0], 0));
  for (size_t i = 0; i < pl->passes.size(); ++i) {
    const Pass& ps = pl->passes[i];
    if (ps.to_y) continue;
    Level& lv = pl->levels[ps.level];
    htlr::launch_sep_block(ps.sep_tab.d(), 2 * ps.sep_NO, ps.sep_NO, (const htlr::SepBlock*)ps.sep_blocks.ptr,
                           ps.sep_nblocks, (const htlr::SepCol*)ps.sep_cols.ptr, cx.W[i], ps.K_pad, lv.H.d(), ps.P, R,
                           pl->sep_corr.d(), pl->side_stream, ps.zpitch);
    ++cx.launches;
  }
  CUDA_TRY(cudaEventRecord(pl->side_ev[1], pl->side_stream));
  htlr::CubeLevels cl;
  if (!cube_params(pl, nullptr, cl)) return fail(2, "overlapped matvec: downward not supported");
  const int64_t nb = pl->levels[pl->L].nclusters;
  const double* av = pl->has_coeff ? pl->coeff.d() : nullptr;
  leaf_range(1);
  CUDA_TRY(cudaStreamWaitEvent(cx.st, pl->side_ev[1], 0));
  htlr::launch_downward_cube(cl, pl->L, R, 0, nb, cx.st, us, fs, pl->Y.d(), av, pl->desc.coeff_const, pl->n, 0,
                             mz - zs);
  ++cx.launches;
  CUDA_TRY(cudaEventRecord(ev[3], cx.st));
  CUDA_TRY(cudaStreamWaitEvent(cs, ev[3], 0));
  CUDA_TRY(cudaMemcpyAsync(fh, fs, lead * sizeof(double), cudaMemcpyDefault, cs));
  leaf_range(2);
  htlr::launch_downward_cube(cl, pl->L, R, 0, nb, cx.st, us, fs, pl->Y.d(), av, pl->desc.coeff_const, pl->n,
                             mz - zs, mz);
  ++cx.launches;
  CUDA_TRY(cudaEventRecord(ev[4], cx.st));
  CUDA_TRY(cudaStreamWaitEvent(cs, ev[4], 0));
  CUDA_TRY(cudaMemcpyAsync(fh + lead, fs + lead, last * sizeof(double), cudaMemcpyDefault, cs));
  CUDA_TRY(cudaEventRecord(ev[5], cs));
  CUDA_TRY(cudaStreamWaitEvent(cx.st, ev[5], 0));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Slabs of the banded host pipeline (0: not applicable): a single-GPU banded
// separable plan whose upward and downward passes are the per-box-octet
// kernels, which take z ranges of leaf boxes (even bounds).  Four equal
// slabs: a slab's cube upward / downward lasts about one CTA's latency (12-16
// us) whatever its size (thinner end slabs measured no faster), the copy of
// a slab ~80 us, so all but the last upward and the first downward hide.
int band_pipe_slabs(const htlr_plan* pl, int* zu = nullptr, int* zf = nullptr) {
  if (!pl->sep || pl->mapped || pl->shard_world != 1 || pl->zslab || pl->d != 3 || !pl->graphs) return 0;
  if (!pl->passes[pl->leaf_pass].band || !pl->cube_ok) return 0;
  const int mz = pl->levels[pl->L].m;
  for (int S : {4, 2}) {
    if (mz % (2 * S)) continue;
    for (int k = 0; zu && k <= S; ++k) zu[k] = zf[k] = k * (mz / S);
    return S;
  }
  return 0;
}

int mv_band_host(MvCtx& cx, const double* uh, double* fh, cudaStream_t cs) {
  htlr_plan* pl = cx.pl;
  HostPipe hp;
  hp.S = band_pipe_slabs(pl, hp.zu, hp.zf);
  hp.zrow = (size_t)pl->sL * pl->n * pl->n * cx.R;
  hp.uh = uh;
  hp.fh = fh;
  hp.cs = cs;
  hp.ev = pl->ov_ev.data();
  if (hp.S == 0 || pl->ov_ev.size() < (size_t)(2 * hp.S + 2)) return fail(2, "banded host pipeline: not prepared");
  double* us = pl->u_stage.d();
  CUDA_TRY(cudaEventRecord(hp.ev[0], cx.st));
  CUDA_TRY(cudaStreamWaitEvent(cs, hp.ev[0], 0));
  for (int k = 0; k < hp.S; ++k) {
    const size_t o = hp.zu[k] * hp.zrow, c = (hp.zu[k + 1] - hp.zu[k]) * hp.zrow;
    CUDA_TRY(cudaMemcpyAsync(us + o, uh + o, c * sizeof(double), cudaMemcpyDefault, cs));
    CUDA_TRY(cudaEventRecord(hp.ev[1 + k], cs));
  }
  cx.pipe = &hp;
  int rc = mv_local(cx, us);
  if (!rc) rc = mv_remote(cx, us, pl->f_stage.d());
  cx.pipe = nullptr;
  return rc;
}

bool page_locked(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace

int htlr_matvec_host(htlr_plan* pl, const double* u, double* f, int64_t nrhs, void* stream) {
  MvCtx cx;
  if (int rc = mv_prepare(pl, nrhs, stream, cx)) return rc;
  if (!u || !f) return fail(-1, "null vector");
  if (pl->shard_world > 1 || (pl->zslab && pl->zs_world > 1))
    return fail(-1, "sharded plan: use htlr_matvec_local / exchange / htlr_matvec_remote");
  if (!page_locked(u) || !page_locked(f))
    return fail(-1, "host vectors must be page-locked (pinned or registered)");
  const size_t vbytes = (size_t)pl->N * cx.R * sizeof(double);
  if (pl->u_stage.alloc(vbytes) || pl->f_stage.alloc(vbytes)) return 1;
  const bool banded = band_pipe_slabs(pl) > 0;
  if ((!banded && !overlap_ok(pl)) || pl->profiling) {
    CUDA_TRY(cudaMemcpyAsync(pl->u_stage.ptr, u, vbytes, cudaMemcpyDefault, cx.st));
    if (int rc = htlr_matvec(pl, pl->u_stage.d(), pl->f_stage.d(), nrhs, stream)) return rc;
    CUDA_TRY(cudaMemcpyAsync(f, pl->f_stage.ptr, vbytes, cudaMemcpyDefault, cx.st));
    return 0;
  }
  if (pl->host_graph_stage[0] != pl->u_stage.ptr || pl->host_graph_stage[1] != pl->f_stage.ptr) {
    for (auto& g : pl->host_graphs) cudaGraphExecDestroy(g.exec);
    pl->host_graphs.clear();
    pl->host_graph_stage[0] = pl->u_stage.ptr;
    pl->host_graph_stage[1] = pl->f_stage.ptr;
  }
  for (auto& g : pl->host_graphs) {
    if (g.R == cx.R && g.u == u && g.f == f) {
      CUDA_TRY(cudaGraphLaunch(g.exec, cx.st));
      pl->last_launches = g.launches;
      return 0;
    }
  }
  if (!pl->cap_stream) CUDA_TRY(make_cap_stream(&pl->cap_stream));
  if (!pl->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->copy_stream, cudaStreamNonBlocking));
  while (pl->ov_ev.size() < 10) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    pl->ov_ev.push_back(e);
  }
  MvCtx cc = cx;
  cc.st = pl->cap_stream;
  cc.launches = 0;
  CUDA_TRY(cudaStreamBeginCapture(cc.st, cudaStreamCaptureModeThreadLocal));
  int rc = banded ? mv_band_host(cc, u, f, pl->copy_stream) : mv_overlap(cc, u, f, pl->copy_stream);
  cudaGraph_t graph = nullptr;
  cudaError_t ce = cudaStreamEndCapture(cc.st, &graph);
  cudaGraphExec_t exec = nullptr;
  if (rc || ce != cudaSuccess || !graph || cudaGraphInstantiate(&exec, graph, cudaGraphInstantiateFlagUseNodePriority) != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return rc ? rc : fail(2, std::string("overlapped matvec capture failed: ") + cudaGetErrorString(ce));
  }
  cudaGraphDestroy(graph);
  if (pl->host_graphs.size() >= 8) {
    for (auto& g : pl->host_graphs) cudaGraphExecDestroy(g.exec);
    pl->host_graphs.clear();
  }
  pl->host_graphs.push_back({cx.R, u, f, false, exec, {}, {}, {}, {}, cc.launches});
  CUDA_TRY(cudaGraphLaunch(exec, cx.st));
  pl->last_launches = cc.launches;
  return 0;
}

int htlr_set_graphs(htlr_plan* pl, int32_t on) {
  if (!pl) return fail(-1, "null plan");
  pl->graphs = on != 0;
  if (!pl->graphs && pl->device >= 0) {
    cudaSetDevice(pl->device);
    drop_graphs(pl);
  }
  return 0;
}

int htlr_matvec_local(htlr_plan* pl, const double* u, int64_t nrhs, void* stream) {
  MvCtx cx;
  if (int rc = mv_prepare(pl, nrhs, stream, cx)) return rc;
  if (!u) return fail(-1, "null vector");
  prof_reset(pl);
  if (int rc = mv_local(cx, u)) return rc;
  pl->last_launches = cx.launches;
  return 0;
}

static void reduce_sizes(const htlr_plan* pl, int R, std::vector<int64_t>& b);

int htlr_matvec_remote(htlr_plan* pl, const double* u, double* f, int64_t nrhs, void* stream) {
  MvCtx cx;
  if (int rc = mv_prepare(pl, nrhs, stream, cx)) return rc;
  if (!u || !f) return fail(-1, "null vector");
  {
    std::vector<int64_t> b;
    reduce_sizes(pl, cx.R, b);
    if (!b.empty())
      return fail(-1, "sharded symmetric plan: use htlr_matvec_contract, the reduction, htlr_matvec_expand");
  }
  cx.ev_used = 2 * pl->prof_kind.size();   // continue the local phase's records
  if (int rc = mv_remote(cx, u, f)) return rc;
  pl->last_launches += cx.launches;
  return 0;
}

// full-size accumulators a sharded symmetric plan sums over the shards
static void reduce_sizes(const htlr_plan* pl, int R, std::vector<int64_t>& b) {
  b.clear();
  if (!pl->mapped || pl->shard_world == 1 || !mapped_sym(pl, R)) return;
  const int P = ipow(pl->p, pl->d), PL = ipow(pl->sL, pl->d);
  for (const auto& lv : pl->levels)
    if (lv.needs_up && lv.sym.on) b.push_back(lv.nclusters * (int64_t)R * P * (int64_t)sizeof(double));
  if (pl->near_sym.on) b.push_back(pl->levels[pl->L].nclusters * (int64_t)R * PL * (int64_t)sizeof(double));
}

int htlr_reduce_info(const htlr_plan* pl, int64_t nrhs, int64_t* count, int64_t* bytes, int64_t cap) {
  if (!pl || !count) return fail(-1, "null argument");
  if (!pl->lists_built) return fail(-1, "lists not built");
  if (pl->mapped && !pl->constructed) return fail(-1, "plan not constructed");
  std::vector<int64_t> b;
  reduce_sizes(pl, (int)nrhs, b);
  *count = (int64_t)b.size();
  if (bytes) {
    if (cap < (int64_t)b.size()) return fail(-1, "reduce info buffer too small");
    for (size_t i = 0; i < b.size(); ++i) bytes[i] = b[i];
  }
  return 0;
}

int htlr_bind_reduce(htlr_plan* pl, int64_t nrhs, void* const* ptrs, int64_t count) {
  if (!pl) return fail(-1, "null plan");
  drop_graphs(pl);
  std::vector<int64_t> b;
  reduce_sizes(pl, (int)nrhs, b);
  if (!ptrs || count == 0) {
    pl->red_R = 0;
    pl->red_ptrs.clear();
    return 0;
  }
  if (count != (int64_t)b.size()) return fail(-1, "reduce buffer count mismatch");
  pl->red_ptrs.assign(count, nullptr);
  for (int64_t i = 0; i < count; ++i) {
    if (!ptrs[i]) return fail(-1, "null reduce buffer");
    pl->red_ptrs[i] = static_cast<double*>(ptrs[i]);
  }
  pl->red_R = (int)nrhs;
  return 0;
}

static int matvec_stage(htlr_plan* pl, const double* u, double* f, int64_t nrhs, void* stream, int stages) {
  MvCtx cx;
  if (int rc = mv_prepare(pl, nrhs, stream, cx)) return rc;
  if (!u || (!f && (stages & 2))) return fail(-1, "null vector");
  std::vector<int64_t> b;
  reduce_sizes(pl, cx.R, b);
  if (!b.empty() && !(pl->red_R == cx.R && pl->red_ptrs.size() == b.size()))
    return fail(-1, "sharded symmetric plan: bind the reduce buffers first (htlr_bind_reduce)");
  cx.ev_used = 2 * pl->prof_kind.size();
  if (int rc = mv_remote(cx, u, f, stages)) return rc;
  pl->last_launches += cx.launches;
  return 0;
}

int htlr_matvec_contract(htlr_plan* pl, const double* u, int64_t nrhs, void* stream) {
  return matvec_stage(pl, u, nullptr, nrhs, stream, 1);
}

int htlr_matvec_expand(htlr_plan* pl, const double* u, double* f, int64_t nrhs, void* stream) {
  return matvec_stage(pl, u, f, nrhs, stream, 2);
}

int htlr_matvec_remote_begin(htlr_plan* pl, const double* u, int64_t nrhs, void* stream) {
  return matvec_stage(pl, u, nullptr, nrhs, stream, 1 | 4);
}

int htlr_matvec_remote_finish(htlr_plan* pl, const double* u, double* f, int64_t nrhs, void* stream) {
  return matvec_stage(pl, u, f, nrhs, stream, 1 | 2 | 8);
}

int htlr_cell_average(int32_t kernel, double sigma, double scale, int32_t d, double h, int32_t q,
                      int32_t corner_subdivision, int device, double* out) {
  if (!out) return fail(-1, "null argument");
  if (!(h > 0)) return fail(-1, "cell width must be positive");
  if (d != 2 && d != 3) return fail(-1, "only d = 2 and d = 3 are supported");
  if (q < 2 || q > 64) return fail(-1, "quadrature order must be in [2, 64]");
  if (kernel < 0 || kernel > 2) return fail(-1, "unknown kernel kind");
  if (kernel == HTLR_KERNEL_GAUSSIAN && !(sigma > 0)) return fail(-1, "gaussian kernel needs sigma > 0");
  CUDA_TRY(cudaSetDevice(device));
  std::vector<double> gx, gw;
  gauss01(q, gx, gw);
  gx.insert(gx.end(), gw.begin(), gw.end());
  DevBuf g, o;
  if (g.alloc(gx.size() * sizeof(double)) || o.alloc(sizeof(double))) return 1;
  CUDA_TRY(cudaMemcpy(g.ptr, gx.data(), gx.size() * sizeof(double), cudaMemcpyHostToDevice));
  htlr::KernelParams kp;
  kp.kind = kernel;
  kp.denom = (2.0 * sigma) * sigma;
  kp.scale = scale;
  const bool singular = corner_subdivision != 0;
  htlr::launch_diag(kp, d, h, q, g.d(), g.d() + q, singular ? 1 : 0, o.d(), 0);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(out, o.ptr, sizeof(double), cudaMemcpyDeviceToHost));
  g.release();
  o.release();
  return 0;
}

int htlr_profile_enable(htlr_plan* pl, int32_t on) {
  if (!pl) return fail(-1, "null plan");
  pl->profiling = on != 0;
  return 0;
}

int htlr_profile_read(htlr_plan* pl, int32_t* kinds, int32_t* levels, double* ms, double* flops, double* bytes,
                      int64_t cap, int64_t* count) {
  if (!pl || !count) return fail(-1, "null argument");
  const int64_t nl = (int64_t)pl->prof_kind.size();
  *count = nl;
  if (!pl->profiling || nl == 0) return 0;
  if (!kinds && !levels && !ms && !flops && !bytes) return 0;   // count query
  if (cap < nl) return fail(-1, "profile buffer too small");
  CUDA_TRY(cudaSetDevice(pl->device));
  CUDA_TRY(cudaEventSynchronize(pl->prof_ev[2 * nl - 1]));
  for (int64_t i = 0; i < nl; ++i) {
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, pl->prof_ev[2 * i], pl->prof_ev[2 * i + 1]));
    if (kinds) kinds[i] = pl->prof_kind[i];
    if (levels) levels[i] = pl->prof_level[i];
    if (ms) ms[i] = t;
    if (flops) flops[i] = pl->prof_flops[i];
    if (bytes) bytes[i] = pl->prof_bytes[i];
  }
  return 0;
}

int htlr_exact_rows(htlr_plan* pl, const int64_t* rows, int64_t nrows, const double* u, double* out,
                    void* stream) {
  if (!pl || !rows || !u || !out) return fail(-1, "null argument");
  if (pl->device < 0) return fail(-1, "host-only plan: no device work");
  if (nrows < 0) return fail(-1, "negative row count");
  CUDA_TRY(cudaSetDevice(pl->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int d = pl->d, n = pl->n;
  std::vector<double> gx, gw;
  gauss01(pl->desc.quad_q, gx, gw);
  gx.insert(gx.end(), gw.begin(), gw.end());
  DevBuf gl, cavg, drows;
  if (upload(gl, gx.data(), gx.size() * sizeof(double))) return 1;
  if (cavg.alloc(sizeof(double)) || drows.alloc(std::max<int64_t>(nrows, 1) * sizeof(double))) return 1;
  const double* dv = nullptr;
  if (pl->mapped) {
    if (!pl->dvec.ptr) {   // per-point cell integrals (also built by construct)
      if (upload(pl->d_mb, pl->mb.data(), pl->mb.size() * sizeof(double))) return 1;
      if (upload(pl->d_mx, pl->mx.data(), pl->mx.size() * sizeof(double))) return 1;
      if (upload(pl->d_mc, pl->mc.data(), pl->mc.size() * sizeof(double))) return 1;
      if (pl->dvec.alloc(pl->N * sizeof(double))) return 1;
      htlr::launch_mapped_diag(pl->kp, d, n, pl->desc.quad_q, gl.d(), gl.d() + pl->desc.quad_q, pl->d_mb.d(),
                               pl->d_mx.d(), pl->dvec.d(), pl->N, st);
    }
    dv = pl->dvec.d();
  } else {
    htlr::launch_diag(pl->kp, d, pl->h, pl->desc.quad_q, gl.d(), gl.d() + pl->desc.quad_q,
                      pl->desc.corner_subdivision ? 1 : 0, cavg.d(), st);
  }
  htlr::launch_exact_rows(pl->kp, d, n, pl->h, pl->hd, pl->mapped ? pl->d_mx.d() : nullptr,
                          pl->mapped ? pl->d_mc.d() : nullptr, rows, nrows, cavg.d(), dv, drows.d(),
                          pl->has_coeff ? pl->coeff.d() : nullptr, pl->desc.coeff_const, u, out, st);
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaGetLastError());
  gl.release();
  cavg.release();
  drows.release();
  return 0;
}

int htlr_overlap_areas(const double* tri_xy, const int32_t* cand, int64_t ncand, int32_t m_side, double* areas,
                       void* stream) {
  if (!tri_xy || !cand || !areas) return fail(-1, "null argument");
  if (m_side < 1 || ncand < 0) return fail(-1, "invalid sizes");
  htlr::launch_overlap(tri_xy, cand, ncand, m_side, areas, (cudaStream_t)stream);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int htlr_csr_spmv(const int64_t* rowptr, const int32_t* cols, const double* vals, int64_t nrows, const double* x,
                  double* y, void* stream) {
  if (!rowptr || !x || !y) return fail(-1, "null argument");
  htlr::launch_csr_spmv(rowptr, cols, vals, nrows, x, y, (cudaStream_t)stream);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int htlr_cheb_nodes(double lo, double hi, int32_t order, double* out_host) {
  if (!out_host) return fail(-1, "null argument");
  if (!(lo < hi)) return fail(-1, "interval must satisfy lo < hi");
  if (order < 1 || order > 64) return fail(-1, "order must be in [1, 64]");
  DevBuf o;
  if (o.alloc(order * sizeof(double))) return 1;
  htlr::launch_cheb_nodes(lo, hi, order, o.d(), 0);
  CUDA_TRY(cudaMemcpy(out_host, o.ptr, order * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

int htlr_lagrange_matrix(const double* pts_host, int64_t npts, const double* nodes_host, int32_t order,
                         double* out_host) {
  if ((!pts_host && npts) || !nodes_host || !out_host) return fail(-1, "null argument");
  if (order < 1 || order > 64) return fail(-1, "order must be in [1, 64]");
  DevBuf dp, dn, o;
  if (upload(dp, pts_host, npts * sizeof(double)) || upload(dn, nodes_host, order * sizeof(double)) ||
      o.alloc(std::max<int64_t>(1, npts * order) * sizeof(double)))
    return 1;
  htlr::launch_lagrange(dp.d(), npts, dn.d(), order, o.d(), 0);
  CUDA_TRY(cudaMemcpy(out_host, o.ptr, npts * order * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

int htlr_kernel_pairs(int32_t kernel, double sigma, double scale, int32_t d, const double* x_host, int64_t m1,
                      const double* y_host, int64_t m2, double* out_host) {
  if (!out_host || (!x_host && m1) || (!y_host && m2)) return fail(-1, "null argument");
  if (d < 1 || d > 3) return fail(-1, "dimension must be 1..3 for device kernel pairs");
  if (kernel < 0 || kernel > 2) return fail(-1, "unknown kernel kind");
  htlr::KernelParams kp;
  kp.kind = kernel;
  kp.denom = (2.0 * sigma) * sigma;
  kp.scale = scale;
  DevBuf dx, dy, o, flag;
  if (upload(dx, x_host, m1 * d * sizeof(double)) || upload(dy, y_host, m2 * d * sizeof(double)) ||
      o.alloc(std::max<int64_t>(1, m1 * m2) * sizeof(double)) || flag.alloc(sizeof(int)))
    return 1;
  CUDA_TRY(cudaMemset(flag.ptr, 0, sizeof(int)));
  htlr::launch_pairs(kp, d, dx.d(), m1, dy.d(), m2, o.d(), (int*)flag.ptr, 0);
  int hit = 0;
  CUDA_TRY(cudaMemcpy(&hit, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost));
  if (hit) return fail(-1, "SLP kernel evaluated on the diagonal");
  CUDA_TRY(cudaMemcpy(out_host, o.ptr, m1 * m2 * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

int htlr_kernel_pairs_masked(int32_t kernel, double sigma, double scale, int32_t d, const double* x_host, int64_t m,
                             const double* diag_host, double* out_host) {
  if (!out_host || !diag_host || (!x_host && m)) return fail(-1, "null argument");
  if (d < 1 || d > 3) return fail(-1, "dimension must be 1..3 for device kernel pairs");
  if (kernel < 0 || kernel > 2) return fail(-1, "unknown kernel kind");
  htlr::KernelParams kp;
  kp.kind = kernel;
  kp.denom = (2.0 * sigma) * sigma;
  kp.scale = scale;
  DevBuf dx, o, flag;
  if (upload(dx, x_host, m * d * sizeof(double)) || o.alloc(std::max<int64_t>(1, m * m) * sizeof(double)) ||
      flag.alloc(sizeof(int)))
    return 1;
  CUDA_TRY(cudaMemset(flag.ptr, 0, sizeof(int)));
  // coincident pairs (the diagonal, and any repeated point) are flagged and
  // zeroed by the pair kernel instead of evaluating the singular kernel there
  htlr::launch_pairs(kp, d, dx.d(), m, dx.d(), m, o.d(), (int*)flag.ptr, 0);
  CUDA_TRY(cudaMemcpy(out_host, o.ptr, m * m * sizeof(double), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < m; ++i) out_host[i * m + i] = diag_host[i];
  return 0;
}

static int tensor_rc(cudaError_t e) {
  return e == cudaSuccess ? 0 : fail(1, std::string("tensor op: ") + cudaGetErrorString(e));
}

int htlr_mode_product(const double* t, int64_t a, int64_t k, int64_t b, const double* m, int64_t rows, double* out) {
  if ((!t && a * k * b) || (!m && rows * k) || (!out && a * rows * b)) return fail(-1, "null argument");
  if (a < 0 || k < 0 || b < 0 || rows < 0) return fail(-1, "negative extent");
  return tensor_rc(htlr::tensor_mode_product(t, a, k, b, m, rows, out));
}

int htlr_gemm(const double* a, const double* b, int64_t m, int64_t k, int64_t n, double* c) {
  if ((!a && m * k) || (!b && k * n) || (!c && m * n)) return fail(-1, "null argument");
  if (m < 0 || k < 0 || n < 0) return fail(-1, "negative extent");
  return tensor_rc(htlr::tensor_gemm(a, b, m, k, n, c));
}

int htlr_kron(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc, double* out) {
  if ((!a && ar * ac) || (!b && br * bc) || (!out && ar * ac * br * bc)) return fail(-1, "null argument");
  return tensor_rc(htlr::tensor_kron(a, ar, ac, b, br, bc, out));
}

int htlr_qr(const double* a, int64_t rows, int64_t cols, double* q, double* r) {
  if (!a || !q || !r) return fail(-1, "null argument");
  if (rows < cols) return fail(-1, "qr requires rows >= cols, got shape (" + std::to_string(rows) + ", " +
                                       std::to_string(cols) + ")");
  return tensor_rc(htlr::tensor_qr(a, rows, cols, q, r));
}

int64_t htlr_last_launch_count(const htlr_plan* pl) { return pl ? pl->last_launches : -1; }

int htlr_diag_value(htlr_plan* pl, double* out) {
  if (!pl || !out) return fail(-1, "null argument");
  if (!pl->constructed) return fail(-1, "plan not constructed");
  CUDA_TRY(cudaSetDevice(pl->device));
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(out, pl->diag.ptr, sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

// Mapped grid export: the regenerated block with raw factors (target: Lagrange
// factor at the mapped points; source: cell widths x factor), same operator as
// the reference-style Q/R representation.
static int export_block_mapped(htlr_plan* pl, const htlr::LeafRec& lf, double* out, int64_t cap, double* factors,
                               int64_t factor_cap, int32_t* shapes) {
  const int d = pl->d, p = pl->p;
  const Level& lv = pl->levels[lf.level];
  DevBuf tmp, dout;
  if (lf.kind == 0) {
    const int s = lv.side, P = ipow(p, d);
    if ((int64_t)P * P > cap) return fail(-1, "block buffer too small");
    if (!factors || factor_cap < (int64_t)2 * d * s * p) return fail(-1, "factor buffer too small");
    std::vector<double> nodes((size_t)lv.m * p), L((size_t)lv.m * s * p), WL((size_t)lv.m * s * p);
    CUDA_TRY(cudaMemcpy(nodes.data(), lv.nodes.ptr, nodes.size() * 8, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(L.data(), lv.Lm.ptr, L.size() * 8, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(WL.data(), lv.WLm.ptr, WL.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<double> ntns(2 * 3 * p, 0.0);
    for (int a = 0; a < d; ++a)
      for (int t = 0; t < p; ++t) {
        ntns[a * p + t] = nodes[(size_t)lf.tc[a] * p + t];
        ntns[3 * p + a * p + t] = nodes[(size_t)lf.sc[a] * p + t];
      }
    if (upload(tmp, ntns.data(), ntns.size() * 8) || dout.alloc((size_t)P * P * 8)) return 1;
    htlr::launch_mapped_core_export(pl->kp, d, p, tmp.d(), tmp.d() + 3 * p, dout.d(), 0);
    CUDA_TRY(cudaMemcpy(out, dout.ptr, (size_t)P * P * 8, cudaMemcpyDeviceToHost));
    for (int a = 0; a < d; ++a) {
      std::memcpy(factors + (int64_t)a * s * p, &L[(size_t)lf.tc[a] * s * p], (size_t)s * p * 8);
      std::memcpy(factors + (int64_t)(d + a) * s * p, &WL[(size_t)lf.sc[a] * s * p], (size_t)s * p * 8);
    }
    shapes[0] = 0;
    shapes[1] = ipow(s, d);
    shapes[2] = ipow(s, d);
    shapes[3] = 2 * d * s * p;
    return 0;
  }
  const int sL = pl->sL, P = ipow(sL, d);
  if ((int64_t)P * P > cap) return fail(-1, "block buffer too small");
  std::vector<double> geo(3 * 3 * sL, 0.0);   // xt, ys, ws
  for (int a = 0; a < d; ++a)
    for (int i = 0; i < sL; ++i) {
      geo[a * sL + i] = pl->mx[(size_t)lf.tc[a] * sL + i];
      geo[3 * sL + a * sL + i] = pl->mx[(size_t)lf.sc[a] * sL + i];
      geo[6 * sL + a * sL + i] = pl->mc[(size_t)lf.sc[a] * sL + i];
    }
  bool self = true;
  for (int a = 0; a < d; ++a) self = self && lf.tc[a] == lf.sc[a];
  if (upload(tmp, geo.data(), geo.size() * 8) || dout.alloc((size_t)P * P * 8)) return 1;
  htlr::launch_mapped_near_export(pl->kp, d, sL, tmp.d(), tmp.d() + 3 * sL, tmp.d() + 6 * sL, self ? 1 : 0,
                                  dout.d(), 0);
  CUDA_TRY(cudaMemcpy(out, dout.ptr, (size_t)P * P * 8, cudaMemcpyDeviceToHost));
  if (self) {
    std::vector<double> dv((size_t)pl->N), av;
    CUDA_TRY(cudaMemcpy(dv.data(), pl->dvec.ptr, dv.size() * 8, cudaMemcpyDeviceToHost));
    if (pl->has_coeff) {
      av.resize((size_t)pl->N);
      CUDA_TRY(cudaMemcpy(av.data(), pl->coeff.ptr, av.size() * 8, cudaMemcpyDeviceToHost));
    }
    for (int k = 0; k < P; ++k) {
      int x = k % sL, y = (k / sL) % sL, z = k / (sL * sL);
      int64_t g = (int64_t)(lf.tc[0] * sL + x) + (int64_t)pl->n * (lf.tc[1] * sL + y);
      if (d == 3) g += (int64_t)pl->n * pl->n * (lf.tc[2] * sL + z);
      out[(int64_t)k * P + k] = dv[g] + (pl->has_coeff ? av[g] : pl->desc.coeff_const);
    }
  }
  shapes[0] = 1;
  shapes[1] = P;
  shapes[2] = P;
  shapes[3] = 0;
  return 0;
}

// Separable plan export: the Kronecker product of the pass's device-built 1-D
// factors (the operator the apply kernel uses), in the dense path's formats.
static int export_block_sep(htlr_plan* pl, const htlr::LeafRec& lf, double* out, int64_t cap, double* factors,
                            int64_t factor_cap, int32_t* shapes) {
  const int d = pl->d, p = pl->p, s = htlr::kSepP;
  const Level& lv = pl->levels[lf.level];
  const Pass* ps = nullptr;
  for (auto& q : pl->passes)
    if (lf.kind == 0 ? (!q.to_y && q.level == lf.level) : q.to_y) ps = &q;
  if (!ps && lf.kind == 0) ps = &pl->passes[pl->leaf_pass];   // leaf-level cores live in the leaf pass
  const int NO = ps->sep_NO, OR = (NO - 1) / 2;
  std::vector<double> tab((size_t)2 * NO * htlr::kSepSlot);
  CUDA_TRY(cudaMemcpy(tab.data(), ps->sep_tab.ptr, tab.size() * sizeof(double), cudaMemcpyDeviceToHost));
  const double* M[3];
  const int kind = lf.kind == 0 ? 0 : 1;
  for (int a = 0; a < d; ++a) {
    const int o = lf.sc[a] - lf.tc[a];
    if (std::abs(o) > OR) return fail(2, "leaf offset outside the separable tables");
    M[a] = tab.data() + (int64_t)(kind * NO + o + OR) * htlr::kSepSlot + 192;
  }
  const int P = s * s * s;
  if ((int64_t)P * P > cap) return fail(-1, "block buffer too small");
  const double scale = pl->kp.scale;
  auto entry = [&](int m, int k) {
    return (scale * M[0][(m % s) * s + k % s]) * M[1][((m / s) % s) * s + (k / s) % s] *
           M[2][(m / (s * s)) * s + k / (s * s)];
  };
  shapes[0] = lf.kind;
  shapes[1] = P;
  shapes[2] = P;
  shapes[3] = 0;
  if (lf.kind == 0) {
    for (int k = 0; k < P; ++k)
      for (int m = 0; m < P; ++m) out[m + (int64_t)P * k] = entry(m, k);
    if (lv.side != p) {
      std::vector<double> q((size_t)lv.side * p);
      CUDA_TRY(cudaMemcpy(q.data(), lv.Q.ptr, q.size() * sizeof(double), cudaMemcpyDeviceToHost));
      const int64_t need = (int64_t)2 * d * lv.side * p;
      if (!factors || factor_cap < need) return fail(-1, "factor buffer too small");
      for (int f = 0; f < 2 * d; ++f) std::memcpy(factors + (int64_t)f * lv.side * p, q.data(), q.size() * sizeof(double));
      shapes[3] = (int32_t)need;
      shapes[1] = ipow(lv.side, d);
      shapes[2] = ipow(lv.side, d);
    }
    return 0;
  }
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) out[(int64_t)i * P + j] = entry(i, j);
  bool self = true;
  for (int a = 0; a < d; ++a)
    if (lf.tc[a] != lf.sc[a]) self = false;
  if (self) {
    double dv = 0.0;
    CUDA_TRY(cudaMemcpy(&dv, pl->diag.ptr, sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<double> a(P, pl->desc.coeff_const);
    if (pl->has_coeff) {
      std::vector<double> all((size_t)pl->N);
      CUDA_TRY(cudaMemcpy(all.data(), pl->coeff.ptr, all.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (int k = 0; k < P; ++k) {
        const int x = k % s, y = (k / s) % s, z = k / (s * s);
        a[k] = all[(int64_t)(lf.tc[0] * s + x) + (int64_t)pl->n * (lf.tc[1] * s + y) +
                   (int64_t)pl->n * pl->n * (lf.tc[2] * s + z)];
      }
    }
    for (int i = 0; i < P; ++i) out[(int64_t)i * P + i] = dv * pl->hd + a[i];
  }
  return 0;
}

int htlr_formulation(const htlr_plan* pl) {
  if (!pl) return fail(-1, "null plan");
  if (!pl->constructed) return fail(-1, "plan not constructed");
  return pl->mapped ? 2 : pl->sep ? 1 : 0;
}

int htlr_leaf_pass(const htlr_plan* pl) {
  if (!pl) return fail(-1, "null plan");
  if (!pl->constructed) return fail(-1, "plan not constructed");
  if (!pl->sep || pl->mapped) return 0;
  const Pass& lp = pl->passes[pl->leaf_pass];
  return lp.band ? 3 : lp.sep_nblocks > 0 ? 2 : 1;
}

int htlr_export_block(htlr_plan* pl, int64_t leaf_id, double* core_or_dense, int64_t cap, double* factors,
                      int64_t factor_cap, int32_t* shapes) {
  if (!pl || !core_or_dense || !shapes) return fail(-1, "null argument");
  if (!pl->constructed) return fail(-1, "plan not constructed");
  if (int rc = ensure_leaves(pl)) return rc;
  if (leaf_id < 0 || leaf_id >= (int64_t)pl->tree.leaves.size()) return fail(-1, "leaf id out of range");
  CUDA_TRY(cudaSetDevice(pl->device));
  CUDA_TRY(cudaDeviceSynchronize());
  const auto& lf = pl->tree.leaves[leaf_id];
  if (pl->mapped) return export_block_mapped(pl, lf, core_or_dense, cap, factors, factor_cap, shapes);
  const int d = pl->d, p = pl->p;
  const Level& lv = pl->levels[lf.level];
  // separable plans regenerate the block from the 1-D factors (no table id;
  // analytic levels have no offset tables)
  if (pl->sep) return export_block_sep(pl, lf, core_or_dense, cap, factors, factor_cap, shapes);
  const OffsetTable& tab = lf.kind == 0 ? lv.adm : pl->near;
  const int64_t key = pack_offset(lf.tc, lf.sc, d, lv.m);
  const int id = tab.dense.empty() ? tab.id.at(key) : tab.dense[key] - 1;
  if (id < 0) return fail(2, "leaf offset missing from the plan's tables");
  const Pass* ps = nullptr;
  int mat = id;
  if (lf.kind == 0) {
    for (auto& q : pl->passes)
      if (!q.to_y && q.level == lf.level) ps = &q;
    if (!ps) {
      ps = &pl->passes[pl->leaf_pass];
      mat = pl->near_mats + id;
    }
  } else {
    ps = &pl->passes[pl->leaf_pass];
  }
  std::vector<double> tiled((size_t)ps->mat_stride);
  CUDA_TRY(cudaMemcpy(tiled.data(), ps->table.d() + (int64_t)mat * ps->mat_stride, tiled.size() * sizeof(double),
                      cudaMemcpyDeviceToHost));
  const int P = ps->P;
  if ((int64_t)P * P > cap) return fail(-1, "block buffer too small");
  shapes[0] = lf.kind;
  shapes[1] = P;
  shapes[2] = P;
  shapes[3] = 0;
  if (lf.kind == 0) {
    // core tensor, F-order with target modes first: element (m, k) at m + P*k
    for (int k = 0; k < P; ++k)
      for (int m = 0; m < P; ++m)
        core_or_dense[m + (int64_t)P * k] = tiled[htlr::tiled_offset(m, k, ps->MT, ps->K_pad)];
    if (pl->lowrank) {
      // LowRankBlock(u, g, v): g = core as a P x P matrix (row-major), u = v =
      // dense Kronecker factor (identity where the side equals p)
      const int64_t S = ipow(lv.side, d);
      std::vector<double> g((size_t)P * P);
      for (int k = 0; k < P; ++k)
        for (int m = 0; m < P; ++m) g[(size_t)m * P + k] = core_or_dense[m + (int64_t)P * k];
      std::memcpy(core_or_dense, g.data(), g.size() * sizeof(double));
      if (!factors || factor_cap < 2 * S * P) return fail(-1, "factor buffer too small");
      if (lv.Kron.ptr) {
        CUDA_TRY(cudaMemcpy(factors, lv.Kron.ptr, (size_t)(S * P) * sizeof(double), cudaMemcpyDeviceToHost));
      } else {
        for (int64_t e = 0; e < S * P; ++e) factors[e] = (e / P == e % P) ? 1.0 : 0.0;
      }
      std::memcpy(factors + S * P, factors, (size_t)(S * P) * sizeof(double));
      shapes[0] = 2;
      shapes[1] = (int32_t)S;
      shapes[2] = (int32_t)S;
      shapes[3] = (int32_t)(2 * S * P);
      return 0;
    }
    if (lv.side != p) {
      std::vector<double> q((size_t)lv.side * p);
      CUDA_TRY(cudaMemcpy(q.data(), lv.Q.ptr, q.size() * sizeof(double), cudaMemcpyDeviceToHost));
      int64_t need = (int64_t)2 * d * lv.side * p;
      if (!factors || factor_cap < need) return fail(-1, "factor buffer too small");
      for (int f = 0; f < 2 * d; ++f)
        std::memcpy(factors + (int64_t)f * lv.side * p, q.data(), q.size() * sizeof(double));
      shapes[3] = (int32_t)need;
      shapes[1] = ipow(lv.side, d);
      shapes[2] = ipow(lv.side, d);
    }
  } else {
    // dense rows x cols, row-major, with a(x_i) on the tau == sigma diagonal
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < P; ++j)
        core_or_dense[(int64_t)i * P + j] = tiled[htlr::tiled_offset(i, j, ps->MT, ps->K_pad)];
    bool self = true;
    for (int a = 0; a < d; ++a)
      if (lf.tc[a] != lf.sc[a]) self = false;
    if (self) {
      std::vector<double> a(P, pl->desc.coeff_const);
      if (pl->has_coeff) {
        std::vector<double> all((size_t)pl->N);
        CUDA_TRY(cudaMemcpy(all.data(), pl->coeff.ptr, all.size() * sizeof(double), cudaMemcpyDeviceToHost));
        const int s = pl->sL;
        for (int k = 0; k < P; ++k) {
          int x = k % s, y = (k / s) % s, z = k / (s * s);
          int64_t g = (int64_t)(lf.tc[0] * s + x) + (int64_t)pl->n * (lf.tc[1] * s + y);
          if (d == 3) g += (int64_t)pl->n * pl->n * (lf.tc[2] * s + z);
          a[k] = all[g];
        }
      }
      for (int i = 0; i < P; ++i) core_or_dense[(int64_t)i * P + i] += a[i];
    }
  }
  return 0;
}

int htlr_storage(const htlr_plan* pl, int64_t out[5]) {
  if (!pl || !out) return fail(-1, "null argument");
  if (!pl->lists_built) return fail(-1, "lists not built");
  const int d = pl->d, p = pl->p;
  const int64_t PL = ipow(pl->sL, d);
  int64_t dense = pl->num_near * PL * PL, fac = 0, core = 0;
  for (const auto& lv : pl->levels) {
    core += lv.num_adm * (int64_t)ipow(p, 2 * d);
    if (pl->lowrank)   // LowRankBlock u and v: s^d x p^d each (blocks.py:294)
      fac += lv.num_adm * (int64_t)2 * ipow(lv.side, d) * ipow(p, d);
    else if (lv.side != p)
      fac += lv.num_adm * (int64_t)2 * d * lv.side * p;
  }
  out[0] = dense;
  out[1] = fac;
  out[2] = core;
  out[3] = dense + fac + core;
  out[4] = pl->device_scalars;
  return 0;
}

}  // extern "C"
