// Cluster tree + block cluster tree, bit-exact with the reference.
//
// Reference: /root/reference/pkg/src/htlr/grids.py
//   _leaf_side               :196-207   exact halving to the threshold
//   build_cluster_tree       :210-234   midpoint split, children in
//                                       np.ndindex order (last dim fastest)
//   domain_of                :237-242   [lo*h, hi*h], h = 1.0/n
//   DomainBox                :110-127   diameter_sq / distance_sq / overlap
//   is_admissible            :153-165   strong: diam <= eta*eta*dist*(1+1e-12)
//   build_block_cluster_tree :268-296   DFS, sigma children outer, tau inner
//
// Every level of the reference tree is uniform (all boxes at level l have
// side n >> l, guaranteed by the exact halving), so a cluster is identified by
// its integer coordinates at its level; children of c are 2c + combo.
// This file must be compiled with -ffp-contract=off: the predicate is
// evaluated with separate IEEE multiplies and adds in Python's order.
#include "htlr_lists.h"

#include <algorithm>
#include <atomic>
#include <thread>

#include <algorithm>
#include <cmath>
#include <cstdio>

namespace htlr {

int compute_leaf_side(int n, int leaf_side_max, int* side, std::string& err) {
  if (leaf_side_max < 1) {
    err = "leaf threshold must be positive";
    return -1;
  }
  int s = n;
  while (s > leaf_side_max) {
    if (s % 2) {
      char buf[160];
      snprintf(buf, sizeof buf,
               "grid side %d cannot be halved evenly down to the leaf threshold %d", n,
               leaf_side_max);
      err = buf;
      return -1;
    }
    s /= 2;
  }
  *side = s;
  return 0;
}

namespace {

// Python: float(sum((b - a) ** 2 for a, b in intervals)); the int start 0
// makes the first term exact, then sequential float adds.
double diameter_sq(int d, const double* lo, const double* hi) {
  double total = 0.0;
  for (int a = 0; a < d; ++a) {
    double e = hi[a] - lo[a];
    double sq = e * e;   // pow(x, 2.0) is correctly rounded == x*x
    total = (a == 0) ? sq : total + sq;
  }
  return total;
}

double distance_sq(int d, const double* lo1, const double* hi1, const double* lo2,
                   const double* hi2) {
  double total = 0.0;
  for (int a = 0; a < d; ++a) {
    double g1 = lo1[a] - hi2[a];
    double g2 = lo2[a] - hi1[a];
    double gap = g1;
    if (g2 > gap) gap = g2;
    if (0.0 > gap) gap = 0.0;
    double sq = gap * gap;
    total = total + sq;
  }
  return total;
}

double overlap_volume(int d, const double* lo1, const double* hi1, const double* lo2,
                      const double* hi2) {
  double vol = 1.0;
  for (int a = 0; a < d; ++a) {
    double mn = hi1[a] < hi2[a] ? hi1[a] : hi2[a];
    double mx = lo1[a] > lo2[a] ? lo1[a] : lo2[a];
    double length = mn - mx;
    if (length <= 0.0) return 0.0;
    vol = vol * length;
  }
  return vol;
}

}  // namespace

bool admissible_boxes(const TreeSpec& spec, const int* tlo, const int* thi, const int* slo,
                      const int* shi) {
  const double h = 1.0 / (double)spec.n;
  double a1[3], b1[3], a2[3], b2[3];
  const bool mapped = !spec.bounds.empty();
  for (int a = 0; a < spec.d; ++a) {
    a1[a] = mapped ? spec.bounds[tlo[a]] : (double)tlo[a] * h;
    b1[a] = mapped ? spec.bounds[thi[a]] : (double)thi[a] * h;
    a2[a] = mapped ? spec.bounds[slo[a]] : (double)slo[a] * h;
    b2[a] = mapped ? spec.bounds[shi[a]] : (double)shi[a] * h;
  }
  if (spec.rule == 0) return overlap_volume(spec.d, a1, b1, a2, b2) == 0.0;
  double dist = distance_sq(spec.d, a1, b1, a2, b2);
  double dt = diameter_sq(spec.d, a1, b1);
  double ds = diameter_sq(spec.d, a2, b2);
  double diam = dt >= ds ? dt : ds;   // Python max() keeps the first on ties
  double rhs = spec.eta * spec.eta;
  rhs = rhs * dist;
  rhs = rhs * (1.0 + 1e-12);
  return diam <= rhs;
}

namespace {

struct Builder {
  const TreeSpec& spec;
  const Tree& tree;
  std::vector<LeafRec>* out;   // append here, or ...
  LeafRec* dst = nullptr;      // ... write here (exact size known), or only count
  size_t count = 0;
  int combos[8][3];
  int ncombo;
  // split > 0: stop the recursion at that level and record the pending
  // subtree (kind -1) instead, in DFS position
  int split = -1;
  int truncate = -1;              // >= 0: inadmissible pairs of that level are dropped, not refined
  size_t n_adm = 0, n_near = 0;   // pushed leaves by kind
  // Uniform grid with n a power of two: h = 2^-k, so every box bound, gap,
  // square and sum in the predicate is exact in double and the predicate is a
  // function of (level, |offset| per axis) alone -- evaluated once per such
  // key by build_tree (with the reference's arithmetic, on the pair (0, o))
  // and looked up here.  -1: no such pair on the level.
  static constexpr int kMemo = kOffsetMemo;
  const int8_t* memo = nullptr;

  Builder(const TreeSpec& s, const Tree& t, std::vector<LeafRec>* o, const int8_t* m = nullptr)
      : spec(s), tree(t), out(o), memo(m) {
    // np.ndindex(*([2] * d)): last dimension varies fastest
    ncombo = 1 << spec.d;
    for (int i = 0; i < ncombo; ++i) {
      for (int a = 0; a < spec.d; ++a) {
        int shift = spec.d - 1 - a;
        combos[i][a] = (i >> shift) & 1;
      }
    }
  }

  bool admissible(const int* tc, const int* sc, int level) {
    if (memo) {
      int o[3] = {0, 0, 0};
      bool fits = true;
      for (int a = 0; a < spec.d; ++a) {
        o[a] = tc[a] > sc[a] ? tc[a] - sc[a] : sc[a] - tc[a];
        fits = fits && o[a] < kMemo;
      }
      if (fits) {
        const int8_t v = memo[(((size_t)level * kMemo + o[0]) * kMemo + o[1]) * kMemo + o[2]];
        if (v >= 0) return v != 0;
      }
    }
    const int side = tree.side(level);
    int tlo[3], thi[3], slo[3], shi[3];
    for (int a = 0; a < spec.d; ++a) {
      tlo[a] = tc[a] * side;
      thi[a] = tlo[a] + side;
      slo[a] = sc[a] * side;
      shi[a] = slo[a] + side;
    }
    return admissible_boxes(spec, tlo, thi, slo, shi);
  }

  void visit(const int* tc, const int* sc, int level) {
    if (admissible(tc, sc, level)) {
      push(0, level, tc, sc);
      return;
    }
    if (level == tree.depth) {   // both leaves (lock-step refinement)
      push(1, level, tc, sc);
      return;
    }
    if (level == truncate) return;
    if (level == split) {
      push(-1, level, tc, sc);
      return;
    }
    int tk[3], sk[3];
    for (int si = 0; si < ncombo; ++si) {
      for (int a = 0; a < spec.d; ++a) sk[a] = 2 * sc[a] + combos[si][a];
      for (int ti = 0; ti < ncombo; ++ti) {
        for (int a = 0; a < spec.d; ++a) tk[a] = 2 * tc[a] + combos[ti][a];
        visit(tk, sk, level + 1);
      }
    }
  }

  // the children of a pending subtree (its own node was visited already)
  void expand(const LeafRec& r) {
    int tk[3], sk[3];
    for (int si = 0; si < ncombo; ++si) {
      for (int a = 0; a < spec.d; ++a) sk[a] = 2 * r.sc[a] + combos[si][a];
      for (int ti = 0; ti < ncombo; ++ti) {
        for (int a = 0; a < spec.d; ++a) tk[a] = 2 * r.tc[a] + combos[ti][a];
        visit(tk, sk, r.level + 1);
      }
    }
  }

  void push(int kind, int level, const int* tc, const int* sc) {
    if (kind == 0)
      ++n_adm;
    else if (kind == 1)
      ++n_near;
    if (!out && !dst) {
      ++count;
      return;
    }
    LeafRec r;
    r.kind = kind;
    r.level = level;
    for (int a = 0; a < 3; ++a) {
      r.tc[a] = a < spec.d ? tc[a] : 0;
      r.sc[a] = a < spec.d ? sc[a] : 0;
    }
    if (dst)
      dst[count++] = r;
    else
      out->push_back(r);
  }
};

}  // namespace

double mapped_phi(double t, double amplitude) {
  const double two_pi = 2.0 * 3.141592653589793;
  double arg = two_pi * t;
  double v = amplitude * std::sin(arg);
  v = v / two_pi;
  return t + v;
}

void mapped_tables(int n, double amplitude, std::vector<double>& bounds, std::vector<double>& coords,
                   std::vector<double>& widths) {
  bounds.resize(n + 1);
  coords.resize(n);
  widths.resize(n);
  for (int i = 0; i <= n; ++i) bounds[i] = mapped_phi((double)i / (double)n, amplitude);
  for (int i = 0; i < n; ++i) {
    coords[i] = mapped_phi(((double)i + 0.5) / (double)n, amplitude);
    widths[i] = bounds[i + 1] - bounds[i];
  }
}

std::vector<int8_t> offset_memo(const TreeSpec& spec, int depth) {
  std::vector<int8_t> memo;
  if (!spec.bounds.empty() || spec.n < 1 || (spec.n & (spec.n - 1)) != 0) return memo;
  constexpr int K = kOffsetMemo;
  memo.assign((size_t)(depth + 1) * K * K * K, -1);
  for (int l = 0; l <= depth; ++l) {
    const int m = 1 << l, sd = spec.n >> l;
    const int kz = spec.d == 3 ? K : 1;
    for (int ox = 0; ox < K && ox < m; ++ox)
      for (int oy = 0; oy < K && oy < m; ++oy)
        for (int oz = 0; oz < kz && oz < m; ++oz) {
          const int o[3] = {ox, oy, oz};
          int tlo[3], thi[3], slo[3], shi[3];
          for (int a = 0; a < spec.d; ++a) {
            tlo[a] = 0;
            thi[a] = sd;
            slo[a] = o[a] * sd;
            shi[a] = slo[a] + sd;
          }
          memo[(((size_t)l * K + ox) * K + oy) * K + oz] = admissible_boxes(spec, tlo, thi, slo, shi) ? 1 : 0;
        }
  }
  return memo;
}

int build_tree(const TreeSpec& spec, Tree& out, std::string& err, int max_level) {
  if (spec.d != 2 && spec.d != 3) {
    err = "only d = 2 and d = 3 are supported";
    return -1;
  }
  if (spec.n < 1) {
    err = "n must be positive";
    return -1;
  }
  if (spec.rule == 1 && !(spec.eta > 0)) {
    err = "strong admissibility needs eta > 0";
    return -1;
  }
  int side = 0;
  if (compute_leaf_side(spec.n, spec.leaf_side_max, &side, err)) return -1;
  out = Tree();
  out.spec = spec;
  out.leaf_side = side;
  int depth = 0;
  for (int s = spec.n; s > side; s /= 2) ++depth;
  out.depth = depth;
  // DFS down to a split level sequentially (the recursion's order), then the
  // pending subtrees in parallel, concatenated in DFS position: the same
  // leaf list as one sequential recursion
  const std::vector<int8_t> memo = offset_memo(spec, depth);
  const int8_t* mp = memo.empty() ? nullptr : memo.data();
  std::vector<LeafRec> top;
  Builder b(spec, out, &top, mp);
  b.split = depth >= 3 ? 2 : (depth >= 2 ? 1 : -1);
  if (max_level >= 0 && max_level < depth) {
    b.truncate = max_level;
    out.truncated = true;
  }
  int root[3] = {0, 0, 0};
  b.visit(root, root, 0);
  std::vector<size_t> pend;
  for (size_t i = 0; i < top.size(); ++i)
    if (top[i].kind < 0) pend.push_back(i);
  // two parallel passes over the pending subtrees: count their leaves, then
  // write them straight into their slots of the final array (no per-subtree
  // vectors: their growth and the concatenation cost more than the walk)
  std::vector<size_t> cnt(pend.size(), 0);
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const unsigned nthreads = (unsigned)std::max<size_t>(1, std::min<size_t>(hw, pend.size()));
  auto parallel = [&](auto&& body) {
    std::atomic<size_t> next{0};
    auto work = [&]() {
      for (size_t k = next++; k < pend.size(); k = next++) body(k);
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nthreads; ++t) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
  };
  std::vector<size_t> cadm(pend.size(), 0), cnear(pend.size(), 0);
  parallel([&](size_t k) {
    Builder w(spec, out, nullptr, mp);
    w.truncate = b.truncate;
    w.expand(top[pend[k]]);
    cnt[k] = w.count;
    cadm[k] = w.n_adm;
    cnear[k] = w.n_near;
  });
  std::vector<size_t> pos(top.size() + 1, 0);
  {
    size_t k = 0, acc = 0;
    for (size_t i = 0; i < top.size(); ++i) {
      pos[i] = acc;
      acc += top[i].kind >= 0 ? 1 : cnt[k++];
    }
    pos[top.size()] = acc;
  }
  out.leaves.resize(pos[top.size()]);
  for (size_t i = 0; i < top.size(); ++i)
    if (top[i].kind >= 0) out.leaves[pos[i]] = top[i];
  parallel([&](size_t k) {
    Builder w(spec, out, nullptr, mp);
    w.truncate = b.truncate;
    w.dst = out.leaves.data() + pos[pend[k]];
    w.expand(top[pend[k]]);
  });
  for (const auto& r : top) {
    if (r.kind == 0)
      ++out.num_adm;
    else if (r.kind == 1)
      ++out.num_near;
  }
  for (size_t k = 0; k < pend.size(); ++k) {
    out.num_adm += (int64_t)cadm[k];
    out.num_near += (int64_t)cnear[k];
  }
  return 0;
}

}  // namespace htlr
