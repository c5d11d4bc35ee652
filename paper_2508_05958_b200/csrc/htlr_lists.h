// Host-side cluster tree / block cluster tree for the B200 HTLR plan.
//
// Restates grids.py:196-296 of the reference with IEEE-double arithmetic in
// the reference's evaluation order (compiled with -ffp-contract=off), so the
// DFS leaf list is bit-identical to BlockClusterTree.leaves.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace htlr {

struct TreeSpec {
  int d = 3;
  int n = 0;
  int leaf_side_max = 0;
  int rule = 1;        // 0 weak, 1 strong
  double eta = 1.0;
  // mapped tensor grid (BASELINE config 5): cell boundaries phi(i/n),
  // i = 0..n, used for the domain boxes; empty = uniform grid (i*h)
  std::vector<double> bounds;
};

// phi(t) = t + A sin(2 pi t) / (2 pi), evaluated in the same operation order
// as the oracle's Python expression (oracle/htlr_oracle.py MappedGeometry).
double mapped_phi(double t, double amplitude);
void mapped_tables(int n, double amplitude, std::vector<double>& bounds, std::vector<double>& coords,
                   std::vector<double>& widths);

// One admissible or inadmissible leaf, in cluster coordinates of its level.
struct LeafRec {
  LeafRec() {}         // no value-initialisation: the leaf array is sized first, then written in parallel
  int32_t kind;        // 0 admissible, 1 inadmissible
  int32_t level;
  int32_t tc[3];       // target cluster coords (box lo = tc * side(level))
  int32_t sc[3];       // source cluster coords
};

struct Tree {
  TreeSpec spec;
  int leaf_side = 0;   // side of the leaf boxes (grids.py:196-207)
  int depth = 0;       // number of halvings
  std::vector<LeafRec> leaves;   // DFS order == reference leaf_id order
  int64_t num_adm = 0, num_near = 0;
  bool truncated = false;        // built with max_level: pairs below it are not listed

  int side(int level) const { return spec.n >> level; }
  int clusters_per_dim(int level) const { return 1 << level; }
};

// Returns 0 on success, negative with `err` set on invalid input.
int compute_leaf_side(int n, int leaf_side_max, int* side, std::string& err);
// max_level >= 0: stop at that level -- its inadmissible pairs are dropped
// instead of refined, so only the admissible leaves of levels <= max_level
// are listed (plans that apply the deeper levels as banded sweeps; the full
// list is built when an export asks for it).
int build_tree(const TreeSpec& spec, Tree& out, std::string& err, int max_level = -1);

// Uniform grid with n a power of two: the admissibility predicate per
// (level, |offset| per axis), [level][ox][oy][oz] with kOffsetMemo entries per
// axis: 1 admissible, 0 not, -1 no such pair on the level.  Empty for other
// grids (the predicate is then not exactly translation invariant).
constexpr int kOffsetMemo = 16;
std::vector<int8_t> offset_memo(const TreeSpec& spec, int depth);

// Reference admissibility predicate on index boxes (grids.py:110-127,153-165).
bool admissible_boxes(const TreeSpec& spec, const int* tlo, const int* thi,
                      const int* slo, const int* shi);

}  // namespace htlr
