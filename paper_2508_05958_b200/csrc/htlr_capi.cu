// The remaining C-ABI entry points (include/htlr_b200.h): cell averages,
// per-launch profiling, exact rows, device building blocks of the reference's
// chebyshev / tensor / kernels modules, per-block exports, storage.
#include "htlr_plan_impl.h"

extern "C" {

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

