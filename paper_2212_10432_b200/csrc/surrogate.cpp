// Search-engine cost model (NEXT-3): the paper's second search level, "a machine-learning
// model [XGBoost] predicts the performance of fine-grained parameter settings, and the
// predicted best are run" (P:369 step 3), here as a small gradient-boosted
// regression-tree ensemble fitted on the candidates already timed in the same search.
//
// Features of an Operator Graph (graph_features): per operator name the number of
// occurrences over the whole (branch-expanded) graph, then per numeric parameter class the
// mean of log2(value) over its occurrences (0 when absent), then the number of leaves.  The
// target is log(time); squared loss; depth-limited trees with exhaustive split search (the
// training sets are tens to a few hundred candidates, so exact search is cheap).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>

#include "internal.h"

namespace as {

namespace {

const char* const kOps[] = {"ROW_DIV",        "COL_DIV",        "SORT",           "SORT_SUB",
                            "BIN",            "DIA_DECOM",      "DENSE_DECOM",    "COMPRESS",
                            "BMTB_ROW_BLOCK", "BMW_ROW_BLOCK",  "BMT_ROW_BLOCK",  "BMTB_NNZ_BLOCK",
                            "BMW_NNZ_BLOCK",  "BMT_NNZ_BLOCK",  "BMT_PAD",        "SORT_BMTB",
                            "THREAD_TOTAL_RED", "THREAD_BITMAP_RED_G", "WARP_TOTAL_RED", "WARP_BITMAP_RED",
                            "WARP_SEG_ADD_RED", "SHMEM_TOTAL_RED", "SHMEM_OFFSET_RED", "SET_RESOURCE"};
constexpr int kNOps = sizeof(kOps) / sizeof(kOps[0]);
// numeric parameter classes: (op name or "" for any, key)
struct PClass {
  const char* op;
  const char* key;
};
const PClass kPar[] = {{"BMT_ROW_BLOCK", "rows"}, {"BMT_NNZ_BLOCK", "nnz"},  {"BMW_ROW_BLOCK", "rows"},
                       {"BMW_NNZ_BLOCK", "nnz"},  {"BMTB_ROW_BLOCK", "rows"}, {"BMTB_NNZ_BLOCK", "nnz"},
                       {"SET_RESOURCE", "tpb"},   {"SET_RESOURCE", "grid"},   {"SET_RESOURCE", "stages"}, {"SET_RESOURCE", "xcache"},
                       {"SET_RESOURCE", "stream"},
                       {"BMT_PAD", "vec"},        {"DIA_DECOM", "theta"},     {"DIA_DECOM", "max"},
                       {"DENSE_DECOM", "b"},      {"DENSE_DECOM", "theta"},   {"SORT_SUB", "g"}};
constexpr int kNPar = sizeof(kPar) / sizeof(kPar[0]);

void walk(const Seq& g, std::vector<double>& cnt, std::vector<double>& sum, std::vector<double>& num,
          double& leaves) {
  bool branched = false;
  for (const Op& op : g) {
    for (int i = 0; i < kNOps; ++i)
      if (op.name == kOps[i]) cnt[i] += 1;
    for (int i = 0; i < kNPar; ++i) {
      if (op.name != kPar[i].op) continue;
      for (const auto& kv : op.params) {
        if (kv.first != kPar[i].key) continue;
        const double v = kv.second.k == Value::FLOAT ? kv.second.f : (double)kv.second.i;
        sum[i] += std::log2(1.0 + std::max(0.0, v));
        num[i] += 1;
      }
    }
    for (const Seq& b : op.br) {
      walk(b, cnt, sum, num, leaves);
      branched = true;
    }
  }
  if (!branched) leaves += 1;
}

struct Node {
  int feat = -1;       // -1: leaf
  double thr = 0, val = 0;
  int lo = -1, hi = -1;
};

struct Tree {
  std::vector<Node> nodes;
  double predict(const double* x) const {
    int i = 0;
    while (nodes[i].feat >= 0) i = x[nodes[i].feat] <= nodes[i].thr ? nodes[i].lo : nodes[i].hi;
    return nodes[i].val;
  }
};

// Least-squares regression tree on rows idx of X (n x d, row-major) with residuals r.
int grow(Tree& t, const std::vector<double>& X, size_t d, const std::vector<double>& r, std::vector<size_t> idx,
         int depth, int max_depth, size_t min_leaf) {
  Node nd;
  double s = 0;
  for (size_t i : idx) s += r[i];
  nd.val = idx.empty() ? 0.0 : s / (double)idx.size();
  const int me = (int)t.nodes.size();
  t.nodes.push_back(nd);
  if (depth >= max_depth || idx.size() < 2 * min_leaf) return me;
  double best_gain = 1e-12, best_thr = 0;
  int best_f = -1;
  const double n = (double)idx.size(), tot = s;
  std::vector<std::pair<double, double>> col(idx.size());
  for (size_t f = 0; f < d; ++f) {
    for (size_t k = 0; k < idx.size(); ++k) col[k] = {X[idx[k] * d + f], r[idx[k]]};
    std::sort(col.begin(), col.end());
    double ls = 0;
    for (size_t k = 0; k + 1 < col.size(); ++k) {
      ls += col[k].second;
      if (col[k].first == col[k + 1].first) continue;
      const double nl = (double)(k + 1), nr = n - nl;
      if (nl < (double)min_leaf || nr < (double)min_leaf) continue;
      // SSE reduction of the split = ls^2/nl + rs^2/nr - tot^2/n
      const double gain = ls * ls / nl + (tot - ls) * (tot - ls) / nr - tot * tot / n;
      if (gain > best_gain) {
        best_gain = gain;
        best_f = (int)f;
        best_thr = 0.5 * (col[k].first + col[k + 1].first);
      }
    }
  }
  if (best_f < 0) return me;
  std::vector<size_t> li, hi;
  for (size_t i : idx) (X[i * d + best_f] <= best_thr ? li : hi).push_back(i);
  const int l = grow(t, X, d, r, std::move(li), depth + 1, max_depth, min_leaf);
  const int h = grow(t, X, d, r, std::move(hi), depth + 1, max_depth, min_leaf);
  t.nodes[me].feat = best_f;
  t.nodes[me].thr = best_thr;
  t.nodes[me].lo = l;
  t.nodes[me].hi = h;
  return me;
}

}  // namespace

size_t graph_feature_count() { return (size_t)kNOps + kNPar + 1; }

std::vector<double> graph_features(const Seq& g) {
  std::vector<double> cnt(kNOps, 0.0), sum(kNPar, 0.0), num(kNPar, 0.0);
  double leaves = 0;
  walk(g, cnt, sum, num, leaves);
  std::vector<double> f = cnt;
  for (int i = 0; i < kNPar; ++i) f.push_back(num[i] > 0 ? sum[i] / num[i] : 0.0);
  f.push_back(leaves);
  return f;
}

// Gradient-boosted trees: F_0 = mean(y); F_k = F_{k-1} + lr * tree_k(residuals).
void surrogate_fit_predict(const double* X, const double* y, size_t n, size_t d, const double* Xq, size_t nq,
                           double* out, int rounds, int max_depth, double lr) {
  const double base = n ? std::accumulate(y, y + n, 0.0) / (double)n : 0.0;
  std::vector<double> Xv(X, X + n * d), F(n, base), r(n);
  std::vector<Tree> trees;
  std::vector<size_t> all(n);
  std::iota(all.begin(), all.end(), 0);
  const size_t min_leaf = n >= 16 ? 2 : 1;
  for (int k = 0; k < rounds && n >= 2; ++k) {
    for (size_t i = 0; i < n; ++i) r[i] = y[i] - F[i];
    Tree t;
    grow(t, Xv, d, r, all, 0, max_depth, min_leaf);
    for (size_t i = 0; i < n; ++i) F[i] += lr * t.predict(&Xv[i * d]);
    trees.push_back(std::move(t));
  }
  for (size_t q = 0; q < nq; ++q) {
    double v = base;
    for (const Tree& t : trees) v += lr * t.predict(Xq + q * d);
    out[q] = v;
  }
}

}  // namespace as

using namespace as;

extern "C" {

as_status_t as_graph_features(as_graph_t g, double* out, size_t* n) {
  return guard([&] {
    if (!g || !n) fail(AS_ERR_INVALID_ARG, "NULL argument");
    const size_t need = graph_feature_count();
    if (!out) {
      *n = need;
      return;
    }
    if (*n < need) {
      *n = need;
      fail(AS_ERR_INVALID_ARG, "feature buffer too small");
    }
    std::vector<double> f = graph_features(g->g);
    std::memcpy(out, f.data(), need * sizeof(double));
    *n = need;
  });
}

as_status_t as_surrogate_fit_predict(const double* X, const double* y, size_t n, size_t d, const double* Xq,
                                     size_t nq, double* out) {
  return guard([&] {
    if ((n && (!X || !y)) || (nq && (!Xq || !out)) || d == 0) fail(AS_ERR_INVALID_ARG, "NULL argument or d == 0");
    surrogate_fit_predict(X, y, n, d, Xq, nq, out, 60, 3, 0.2);
  });
}

}  // extern "C"
