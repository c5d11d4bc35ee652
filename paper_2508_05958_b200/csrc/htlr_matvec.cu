// Matvec scheduling of the B200 HTLR plan (operators.py:138-161): the phases
// of one matvec on their streams, CUDA graphs keyed by the caller's vectors,
// the host-vector pipelines and the sharded entry points.
#include "htlr_plan_impl.h"

extern "C" {

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
  pl->f_red = nullptr;
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
// 0.1286 / 0.1284 ms; with the direct-f order 8 / 20 / 32 / 40 / 48 / 64 / 80:
// 0.1311 / 0.1331 / 0.1351 / 0.1290 / 0.1229 / 0.1250 / 0.1311 ms, flat from 48
// to 62: the z sweep's 4096 half-line units take three rounds of its 16 warps
// per SM on any grid of 86 to 127 SMs)
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
  pl->f_red = nullptr;
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
  // a profiled matvec runs the same two kernels, serialised on the one stream
  const bool prof_serial = pl->profiling && !fork && (stages & 1) && !own_only && !rest_only && !pl->leaf_pending &&
                           !pipe_za && pl->sep && pl->passes[pl->leaf_pass].band;
  if ((leaf_z_done || prof_serial) && (stages & 2) && !cx.pipe && pl->shard_world == 1 && !pl->zslab &&
      !band_xy_lines(pl) && fdirect_enabled()) {
    const Pass& lq = pl->passes[pl->leaf_pass];
    const int nbx = 1 << lq.level;
    const bool planes = htlr::band_lines_supported(lq.level) && lq.band_lo[0] == 0 && lq.band_lo[1] == 0 &&
                        lq.band_hi[0] == nbx && lq.band_hi[1] == nbx && lq.band_lo[2] == 0 && lq.band_hi[2] == nbx;
    if (planes && lq.P == htlr::kSepP * htlr::kSepP * htlr::kSepP && cube_params(pl, nullptr, fcl)) {
      // a third stream, forked behind the upward pass: the zeroing of f and
      // the cooperative (non-banded) level passes run beside the banded ones
      if (fork) {
        if (!pl->fz_ev) CUDA_TRY(cudaEventCreateWithFlags(&pl->fz_ev, cudaEventDisableTiming));
        for (auto& ev : pl->fd_ev)
          if (!ev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        if (!pl->leaf_stream) CUDA_TRY(cudaStreamCreateWithFlags(&pl->leaf_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventRecord(pl->fd_ev[0], pl->side_stream));
        CUDA_TRY(cudaStreamWaitEvent(pl->leaf_stream, pl->fd_ev[0], 0));
        CUDA_TRY(cudaMemsetAsync(f, 0, (size_t)pl->N * R * sizeof(double), pl->leaf_stream));
        CUDA_TRY(cudaEventRecord(pl->fz_ev, pl->leaf_stream));
      } else {
        CUDA_TRY(cudaMemsetAsync(f, 0, (size_t)pl->N * R * sizeof(double), cx.st));
      }
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
    if (fdirect && fork && !ps.to_y && !ps.band) sst = pl->leaf_stream;
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
        if (ps.to_y && fdirect && fork) CUDA_TRY(cudaStreamWaitEvent(sst, pl->fz_ev, 0));
        pl->f_red = (ps.to_y && fdirect) ? f : nullptr;   // never stale: an error return may have skipped the reset below
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
    if (fork) {
      CUDA_TRY(cudaEventRecord(pl->fd_ev[1], pl->leaf_stream));
      CUDA_TRY(cudaStreamWaitEvent(pl->side_stream, pl->fd_ev[1], 0));
    }
    const int64_t fb0 = pl->own_lo[pl->L], fnb = pl->own_hi[pl->L] - fb0;
    // work: the expansion's three mode products per leaf box; bytes: f summed (+ u read with a coefficient)
    const double sl = pl->sL;
    const double macs = sl * p * p * p + sl * sl * p * p + sl * sl * sl * p;
    if (cx.prof_begin(4, pl->L, 2.0 * macs * fnb * R, R8 * 2.0 * (double)pl->N)) return 1;
    htlr::launch_downward_cube(fcl, pl->L, R, fb0, fnb, fork ? pl->side_stream : cx.st, u, f, nullptr,
                               pl->has_coeff ? pl->coeff.d() : nullptr, pl->desc.coeff_const, pl->n, 0, 1 << 30, true);
    if (cx.prof_end()) return 1;
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

void drop_graphs(htlr_plan* pl) {
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

}  // extern "C"
