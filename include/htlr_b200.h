/*
 * htlr_b200.h -- C ABI of the B200-native HTLR hot path.
 *
 * Drop-in boundary for the reference package `htlr`
 * (/root/reference/pkg/src/htlr).  The reference exposes an in-process
 * Python API only; these entry points are what its Python layer would bind
 * (ctypes / cffi) to replace, as one unit, the pair
 *     construct(cfg, grid, threads)   operators.py:121-126
 *     matvec(op, u)                   operators.py:159-161
 * together with the tree/list builders they call
 *     build_cluster_tree              grids.py:210-234
 *     build_block_cluster_tree        grids.py:268-296
 * and the accounting the reference reports
 *     storage_report / operation_counts  operators.py:175-209.
 * INTEGRATION.md shows the binding stub.
 *
 * Conventions
 *   - Plain C types only; device buffers are raw pointers owned by the caller
 *     (typically torch tensors' data_ptr()); `stream` is a cudaStream_t passed
 *     as void*.  The plan owns every internal device buffer (lists, factors,
 *     deduplicated cores / near blocks, workspaces).
 *   - Vectors use the reference's grid linearisation (first index fastest,
 *     tensor.py:4-8).  A block of R right-hand sides is row-major [N][R].
 *   - Status codes: 0 ok; negative = invalid argument (the Python layer
 *     raises ValueError, as the reference does); positive = CUDA failure
 *     (RuntimeError).  htlr_last_error() returns a thread-local message.
 *   - A plan is not thread-safe; different plans may be used concurrently.
 *   - There is no CPU fallback: every numeric step runs in sm_100a kernels.
 */
#ifndef HTLR_B200_H
#define HTLR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct htlr_plan htlr_plan;

/* kernels.py:33-103.  `scale` multiplies the reference formula, so the
 * BASELINE kernels are  -log r = 2*pi*SLP2D,  1/r = 4*pi*SLP3D,
 * exp(-r^2/s^2) = GAUSSIAN with sigma = s/sqrt(2). */
enum htlr_kernel_kind { HTLR_KERNEL_GAUSSIAN = 0, HTLR_KERNEL_SLP2D = 1, HTLR_KERNEL_SLP3D = 2 };

/* grids.py:130-165 */
enum htlr_rule_kind { HTLR_RULE_WEAK = 0, HTLR_RULE_STRONG = 1 };

/* leaf kinds in exported lists (grids.py:377-378) */
enum htlr_leaf_kind { HTLR_LEAF_ADMISSIBLE = 0, HTLR_LEAF_INADMISSIBLE = 1 };

typedef struct htlr_desc {
  int32_t d;                  /* 2 or 3 (UniformGrid, grids.py:26-27)          */
  int32_t n;                  /* points per side, h = 1/n                      */
  int32_t leaf_side_max;      /* BuildConfig.leaf_side (operators.py:43)        */
  int32_t rank;               /* BuildConfig.rank = Chebyshev order p           */
  int32_t rule;               /* htlr_rule_kind                                 */
  double eta;                 /* AdmissibilityRule.eta (strong only)            */
  int32_t kernel;             /* htlr_kernel_kind                               */
  double sigma;               /* KernelSpec.sigma (gaussian)                    */
  double scale;               /* multiplies the reference kernel formula        */
  int32_t quad_q;             /* QuadratureConfig.q (kernels.py:187)            */
  int32_t corner_subdivision; /* 1: singular corner-subdivided rule, i.e.
                               * !smooth_at_diagonal && QuadratureConfig.
                               * corner_subdivision (kernels.py:263-265)       */
  double coeff_const;         /* CoefficientFn.constant(c); see htlr_set_coeff  */
  int32_t grid_kind;          /* 0 UniformGrid (grids.py:18-50); 1 mapped
                               * quasi-uniform tensor grid of BASELINE config
                               * 5: x_i = phi((i+1/2)/n), cells [phi(i/n),
                               * phi((i+1)/n)], phi(t) = t + A sin(2 pi t)/(2 pi) */
  double amplitude;           /* A (mapped grid only)                          */
} htlr_desc;

/* Create a plan on `device` (-1: host-only plan that can build and export
 * the trees/lists and the storage accounting, but does no device work);
 * validates the descriptor like the reference's
 * constructors (UniformGrid, _leaf_side, BuildConfig).  Replaces the argument
 * checking of grids.py:23-27,196-207 and operators.py:49-59. */
int htlr_plan_create(const htlr_desc* desc, int device, htlr_plan** out);
int htlr_plan_destroy(htlr_plan* plan);

/* Cluster tree + block cluster tree, bit-exact with grids.py:210-296 (host
 * C++, -ffp-contract=off), flattened into per-level device CSR / offset
 * tables.  Replaces build_cluster_tree + build_block_cluster_tree. */
int htlr_build_lists(htlr_plan* plan);

/* Tree summary: depth, leaf side, leaf counts (operation_counts,
 * operators.py:200-209).  Any pointer may be NULL. */
int htlr_tree_info(const htlr_plan* plan, int32_t* depth, int32_t* leaf_side,
                   int64_t* num_leaves, int64_t* num_admissible, int64_t* num_inadmissible);

/* DFS leaf list (BlockClusterTree.leaves, grids.py:268-296) as int32 rows
 * [leaf_id, kind, level, tau lo/hi per dim, sigma lo/hi per dim]:
 * num_leaves x (3 + 4d) values.  `cap` = capacity of `rows` in int32s. */
int htlr_export_lists(const htlr_plan* plan, int32_t* rows, int64_t cap);

/* Per-point coefficient a(x_i) (CoefficientFn evaluated by the caller on the
 * grid points, kernels.py:162-175); host array of N doubles, F-order.  If
 * never called, coeff_const is used. */
int htlr_set_coeff(htlr_plan* plan, const double* a_host);

/* Construction on the device: diagonal cell quadrature (kernels.py:195-265),
 * per-level Lagrange factors + Householder QR (chebyshev.py:52-66,
 * tensor.py:107-115), Chebyshev kernel sampling + R folding of every unique
 * (level, offset) core (chebyshev.py:69-85, blocks.py:126-164), and the
 * unique near-field blocks (blocks.py:190-227).  Replaces _build_payloads
 * (operators.py:102-118).  Stream-ordered. */
int htlr_construct(htlr_plan* plan, void* stream);

/* f = A u for R right-hand sides (operators.py:138-161 applied column-wise):
 * u, f are DEVICE pointers to row-major [N][nrhs] doubles.  Stream-ordered,
 * asynchronous.  Replaces matvec / _hierarchical_matvec. */
int htlr_matvec(htlr_plan* plan, const double* u, double* f, int64_t nrhs, void* stream);

/* H-matrix baseline (construct_hmatrix / hmatrix_matvec, operators.py:129-135,
 * 164-165; LowRankBlock blocks.py:76-86,167-187,262-264): the admissible
 * blocks' factors are applied as dense kron(Q,..,Q) (s^d x p^d) matrices
 * instead of mode products; same cores, same operator.  Call before
 * htlr_construct; uniform grids only.  Exported admissible blocks then have
 * kind 2 (u = v = dense factor, g = core matrix). */
int htlr_set_lowrank(htlr_plan* plan, int32_t on);

/* ---- multi-GPU: shard the target boxes by cluster subtrees --------------
 * Clusters are numbered in Morton order with the reference's child order, so
 * every subtree is a contiguous id range on every level.  With `world` (a
 * power of two) shards, shard `rank` owns the contiguous range
 * [rank, rank+1) * M_l / world of the M_l clusters of each level l: its
 * target rows, its leaf boxes and its source clusters' upward data.
 * Call htlr_set_shard before htlr_build_lists / htlr_construct. */
int htlr_set_shard(htlr_plan* plan, int32_t rank, int32_t world);
/* z-slab shards of a banded separable plan (3-D Gaussian, eta = 1, p = leaf
 * side = 8; BASELINE config 4), set after htlr_construct on an unsharded plan:
 * shard `rank` of `world` owns the leaf boxes with z in
 * [rank, rank+1) * 2^L / world.  Every shard holds the whole input u; the
 * local phase adds the own boxes' upward contributions into the W_l exchange
 * buffers, which the caller then SUM-reduces across shards (all-reduce, see
 * htlr_exchange_kind); the remote phase runs the banded passes over the z
 * range of each level that holds the own boxes (the z sweep reads the halo
 * from u itself, so there is no other exchange), the downward pass, and
 * writes the f rows of the own boxes -- a contiguous block of the F-order f.
 * world = 1 restores the whole plan.  No reference counterpart. */
int htlr_set_zslab(htlr_plan* plan, int32_t rank, int32_t world);
/* How the exchange buffers are combined across shards: 0 all-gather (shard
 * r's chunk is the r-th 1/world of each buffer), 1 sum (all-reduce). */
int htlr_exchange_kind(const htlr_plan* plan);
/* Owned leaf-box range (Morton ids), owned (target, source) pairs and their
 * GEMM flops per right-hand side. */
int htlr_shard_info(const htlr_plan* plan, int64_t* own_leaf_lo, int64_t* own_leaf_hi,
                    int64_t* own_pairs, double* own_flops);
/* The exchange step: buffers every shard must all-gather between the local
 * and the remote phase -- the leaf-box-major input ub and the upward
 * coefficients W_l of each compressed level.  Each is cluster-major in Morton
 * order, so shard r's part is the contiguous r-th 1/world of its bytes.
 * exchange_info reports the count and total bytes per buffer for `nrhs`;
 * bind_exchange hands the plan caller-owned device buffers of those sizes
 * (e.g. torch tensors all-gathered with NCCL by the caller). */
int htlr_exchange_info(const htlr_plan* plan, int64_t nrhs, int64_t* count, int64_t* bytes, int64_t cap);
int htlr_bind_exchange(htlr_plan* plan, int64_t nrhs, void* const* ptrs, int64_t count);
/* local: permute + upward of the own clusters into the exchange buffers;
 * remote: GEMMs of the own targets and the fused downward pass, writing the
 * f rows of the own leaf boxes (other rows untouched).  htlr_matvec is
 * local + remote for an unsharded plan. */
int htlr_matvec_local(htlr_plan* plan, const double* u, int64_t nrhs, void* stream);
int htlr_matvec_remote(htlr_plan* plan, const double* u, double* f, int64_t nrhs, void* stream);
/* The remote phase in two halves: contract (GEMMs / regenerated blocks into
 * the accumulators H_l, Y) and expand (downward pass into f).  A sharded plan
 * on a mapped grid with the symmetric regeneration evaluates every unordered
 * block pair once, so its column sums land in other shards' rows: it
 * accumulates into full-size buffers that the caller binds (bind_reduce, sizes
 * from reduce_info; cluster-major, shard r's rows = the r-th 1/world of the
 * bytes) and must sum-reduce-scatter between contract and expand.
 * reduce_info reports count 0 for every other plan; htlr_matvec_remote then
 * equals contract + expand (and refuses a plan that needs the reduction).
 * No reference counterpart: the reference has no parallel matvec. */
int htlr_reduce_info(const htlr_plan* plan, int64_t nrhs, int64_t* count, int64_t* bytes, int64_t cap);
int htlr_bind_reduce(htlr_plan* plan, int64_t nrhs, void* const* ptrs, int64_t count);
int htlr_matvec_contract(htlr_plan* plan, const double* u, int64_t nrhs, void* stream);
int htlr_matvec_expand(htlr_plan* plan, const double* u, double* f, int64_t nrhs, void* stream);

/* The remote phase split around the exchange, so the all-gather overlaps
 * device work: _begin zeroes the accumulators and (separable plans) applies
 * the blocks whose sources this shard owns -- it reads only the own chunk of
 * the exchange buffers; _finish, after the exchange, applies the rest and runs
 * the downward pass.  begin + finish == htlr_matvec_remote (not for the
 * mapped symmetric plans, which use contract / reduce / expand). */
int htlr_matvec_remote_begin(htlr_plan* plan, const double* u, int64_t nrhs, void* stream);
int htlr_matvec_remote_finish(htlr_plan* plan, const double* u, double* f, int64_t nrhs, void* stream);

/* Diagonal cell average used by the inadmissible tau == sigma blocks
 * (operators.py:95-99).  Synchronises. */
int htlr_diag_value(htlr_plan* plan, double* out);

/* Payload of one DFS leaf, as the reference stores it (blocks.py:33-73):
 *   admissible: core (p^(2d), F-order, target modes first) into `core_or_dense`,
 *               per dim u then v factors (s x p, row-major) into `factors`
 *               (dims whose box side equals p store nothing: factor None);
 *   inadmissible: dense |tau| x |sigma| row-major into `core_or_dense`.
 * shapes[0] = kind, shapes[1] = rows, shapes[2] = cols, shapes[3] = number of
 * factor scalars written.  Synchronises. */
int htlr_export_block(htlr_plan* plan, int64_t leaf_id, double* core_or_dense, int64_t cap,
                      double* factors, int64_t factor_cap, int32_t* shapes);

/* f = A u with u and f in page-locked HOST memory (the reference's matvec
 * takes host numpy arrays, operators.py:159-161): the plan copies u in and f
 * out on the stream itself.  For separable plans the copies are overlapped
 * with the device work (z-slabs of the vectors, two streams, one CUDA graph
 * per (nrhs, u, f)); otherwise H2D, htlr_matvec, D2H.  Asynchronous on
 * `stream`; negative if a vector is not page-locked (cudaHostAlloc /
 * cudaHostRegister / pinned torch tensors) or the plan is sharded. */
int htlr_matvec_host(htlr_plan* plan, const double* u_host, double* f_host, int64_t nrhs, void* stream);

/* How the constructed plan applies its blocks: 0 = dense deduplicated cores
 * and near blocks (fp64 tensor-core GEMM passes); 1 = separable cores (a
 * tensor-product kernel -- the Gaussian -- on a uniform 3-D grid with
 * p = leaf side = 8: every block is the Kronecker product of three 8 x 8
 * per-axis factors, applied as mode products; HTLR_SEPARABLE=0 forces 0);
 * 2 = regenerated cores (mapped grid).  Same operator in every case
 * (blocks.py:126-227); negative on error. */
int htlr_formulation(const htlr_plan* plan);

/* Leaf-level pass of a separable plan: 0 = not separable (dense GEMM or
 * regenerated passes), 1 = per-warp pair runs, 2 = cooperative per-parent
 * CTAs, 3 = banded line sweeps (eta = 1 strong admissibility: the leaf lists'
 * product-set structure, checked against the lists at construction).  All
 * apply the reference's blocks (blocks.py:126-227); negative on error. */
int htlr_leaf_pass(const htlr_plan* plan);

/* storage_report equivalent (operators.py:175-197): scalars the reference
 * would store: [dense, factor, core, total]; plus what this plan stores
 * on the device after deduplication in out[4]. */
int htlr_storage(const htlr_plan* plan, int64_t out[5]);

/* Diagonal cell average of a translation-invariant kernel over a width-h
 * cell (diagonal_entry, kernels.py:252-265), computed by the device
 * quadrature kernel on `device`; corner_subdivision as in htlr_desc.
 * Synchronous. */
int htlr_cell_average(int32_t kernel, double sigma, double scale, int32_t d, double h, int32_t q,
                      int32_t corner_subdivision, int device, double* out);

/* CUDA-graph replay of htlr_matvec (default on): the first call with a given
 * (nrhs, u, f) captures the launch sequence, later calls replay it. */
int htlr_set_graphs(htlr_plan* plan, int32_t on);

/* Exact rows of the Nystrom system (exact_row_evaluator, oracles.py:65-100):
 * out[r] = sum_{j != i} k(x_i, x_j) w_j u_j + (diag_i + a_i) u_i for
 * i = rows[r]; rows, u, out are device pointers (u of N doubles, F-order).
 * Needs only htlr_plan_create (+ htlr_set_coeff).  Synchronises. */
int htlr_exact_rows(htlr_plan* plan, const int64_t* rows, int64_t nrows, const double* u, double* out,
                    void* stream);

/* Quasi-uniform (triangle mesh) front end, SURVEY 8(f) f3 (quasi.py):
 * areas[c] = |triangle t  intersect  cell (i, j)| of the uniform m_side x
 * m_side grid for candidate c = (t, i, j) (Sutherland-Hodgman clipping +
 * shoelace, quasi.py:123-171); tri_xy = F x 6 doubles (x0 y0 x1 y1 x2 y2);
 * all device pointers; stream-ordered. */
int htlr_overlap_areas(const double* tri_xy, const int32_t* cand, int64_t ncand, int32_t m_side, double* areas,
                       void* stream);
/* y = A x for a CSR matrix (the transfer matrices S and T, quasi.py:174-261);
 * device pointers; stream-ordered. */
int htlr_csr_spmv(const int64_t* rowptr, const int32_t* cols, const double* vals, int64_t nrows, const double* x,
                  double* y, void* stream);

/* Building blocks of the public API, computed on the current device from
 * host arrays (synchronous): Chebyshev nodes (cheb_points, chebyshev.py:31-38),
 * Lagrange factor matrix npts x order (factor_matrix, chebyshev.py:52-66),
 * kernel values m1 x m2 for d-dimensional point sets (pairwise,
 * kernels.py:113-117; -1 "SLP kernel evaluated on the diagonal" on r = 0). */
int htlr_cheb_nodes(double lo, double hi, int32_t order, double* out_host);
int htlr_lagrange_matrix(const double* pts_host, int64_t npts, const double* nodes_host, int32_t order,
                         double* out_host);
int htlr_kernel_pairs(int32_t kernel, double sigma, double scale, int32_t d, const double* x_host, int64_t m1,
                      const double* y_host, int64_t m2, double* out_host);
/* kernels.py:137-149 pairwise_masked_diagonal for one point set (row i and
 * column i the same point): every coincident pair is kept off the singular
 * evaluator and entry (i, i) is replaced by diag[i]. */
int htlr_kernel_pairs_masked(int32_t kernel, double sigma, double scale, int32_t d, const double* x_host, int64_t m,
                             const double* diag_host, double* out_host);
/* Per-block tensor building blocks of htlr.tensor / htlr.blocks, computed on
 * the current device; host arrays, row-major:
 *   mode_product: out[a][r][b] = sum_k m[r][k] t[a][k][b]  (tensor.py:35-52 with
 *                 the contracted mode's leading / trailing extents a, b);
 *   gemm:         c = a (m x k) . b (k x n)               (contract, tensor.py:55-86);
 *   kron:         numpy.kron(a, b)                       (blocks.py:166-187);
 *   qr:           thin Householder QR, rows >= cols, LAPACK dgeqr2 / dorg2r
 *                 sign conventions (tensor.py:107-115). */
int htlr_mode_product(const double* t, int64_t a, int64_t k, int64_t b, const double* m, int64_t rows, double* out);
int htlr_gemm(const double* a, const double* b, int64_t m, int64_t k, int64_t n, double* c);
int htlr_kron(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc, double* out);
int htlr_qr(const double* a, int64_t rows, int64_t cols, double* q, double* r);

/* Per-launch profiling of htlr_matvec: when enabled, every kernel launch of
 * a matvec is bracketed by CUDA events on the launching stream.
 * htlr_profile_read returns, for the last matvec, one entry per launch:
 * kind (0 permute, 1 upward, 2 level GEMM, 3 leaf GEMM, 4 downward), tree
 * level, device milliseconds, algorithmic flops and algorithmic bytes.
 * Any output pointer may be NULL; synchronises on the last event. */
int htlr_profile_enable(htlr_plan* plan, int32_t on);
int htlr_profile_read(htlr_plan* plan, int32_t* kinds, int32_t* levels, double* ms, double* flops,
                      double* bytes, int64_t cap, int64_t* count);

/* Number of CUDA kernel launches issued by the last htlr_matvec call. */
int64_t htlr_last_launch_count(const htlr_plan* plan);

const char* htlr_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HTLR_B200_H */
