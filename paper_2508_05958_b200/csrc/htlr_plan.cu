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
#include "htlr_plan_impl.h"

namespace htlr_impl {
thread_local std::string g_last_error;
}

namespace htlr_impl {

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

}  // namespace htlr_impl

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
double band_flops_of(int level, bool leaf, int64_t nt, double* z_share) {
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
int ensure_leaves(const htlr_plan* cpl) {
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

int upload(DevBuf& buf, const void* src, size_t bytes) {
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
bool cube_params(const htlr_plan* pl, double* const* W, htlr::CubeLevels& cl) {
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


int ensure_workspace(htlr_plan* pl, int R) {
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

}  // extern "C"
