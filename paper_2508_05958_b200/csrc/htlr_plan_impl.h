// Internal header of the plan's translation units (not part of the C ABI):
// the plan object and its host-side records, shared by
//   htlr_plan.cu    plan lifetime, interaction lists, shard setters, construct
//   htlr_matvec.cu  matvec scheduling (streams, graphs, host pipelines, shards)
//   htlr_capi.cu    the remaining C-ABI entry points (profiling, exact rows,
//                   per-block exports, tensor helpers, storage)
#pragma once
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

namespace htlr_impl {

extern thread_local std::string g_last_error;   // htlr_plan.cu

inline int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(1, std::string(#expr) + ": " + cudaGetErrorString(_e));              \
  } while (0)

inline int ipow(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}
inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

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

inline int64_t pack_offset(const int* tc, const int* sc, int d, int m) {
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

}  // namespace htlr_impl
using namespace htlr_impl;


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


// y-x sweep of the banded passes as two line kernels (all SMs) instead of the
// plane kernel (one SM per z-point plane): z-slab shards, whose slab has few
// planes (on one GPU the plane kernel is faster: 108 vs 136 us, config 4)
inline bool band_xy_lines(const htlr_plan* pl) { return pl->zslab; }
// HTLR_FDIRECT=0: the leaf pass writes Y and the downward pass follows it
// (the formulation the parity tests cross-check the direct-f one against)
inline bool fdirect_enabled() {
  const char* e = getenv("HTLR_FDIRECT");
  return !(e && e[0] == '0');
}


// functions shared between the translation units
namespace htlr_impl {
void gauss01(int q, std::vector<double>& x, std::vector<double>& w);
int make_tasks(Pass& ps, int R, std::vector<htlr::GemmTask>& out);
}  // namespace htlr_impl
// (C linkage like their definitions inside the extern "C" blocks; hidden: not part of the ABI)
#pragma GCC visibility push(hidden)
extern "C" {
bool cube_params(const htlr_plan* pl, double* const* W, htlr::CubeLevels& cl);
int ensure_workspace(htlr_plan* pl, int R);
double band_flops_of(int level, bool leaf, int64_t nt, double* z_share = nullptr);
int upload(DevBuf& buf, const void* src, size_t bytes);
int ensure_leaves(const htlr_plan* cpl);
void drop_graphs(htlr_plan* pl);
}
#pragma GCC visibility pop
