// Model-Driven Format Compression (NEXT-2; §V-D): replace an index array of the
// format by a closed-form model plus a few patches, so that the kernel computes the value
// instead of loading it ("transforming array type data (in memory) to models and replacing
// memory access with calculation").  Hypotheses (linear, step, periodic linear),
// one closed form model(i) = b + k1*(i / w) + k2*(i % w):
//   linear    w = 1                      candidates from the element pairs (0,1), (n/2, n/2+1), (n-2, n-1)
//   periodic  w in 2, 4, ..., 256 (< n)  b = a[0], k2 = a[1] - a[0], k1 = a[w] - a[0]
//   step      w = first run length (< n) b = a[0], k2 = 0, k1 = a[w] - a[0]
// Exact fitting with patches ("a small number of errors can be tolerated by adding if
// statements"), at most `budget` (<= 8); fewest patches wins, earlier candidate on ties
// (linear, periodic, step: SPEC S:337-340).
#include <array>
#include <cstring>

#include "internal.h"

namespace as {

namespace {

// patches of one candidate, or -1 when more than budget
int count_patches(const std::vector<int64_t>& a, int64_t b, int64_t k1, int64_t k2, int64_t w, int budget,
                  IdxModel* keep) {
  int np = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    const int64_t ii = (int64_t)i;
    if (b + k1 * (ii / w) + k2 * (ii % w) == a[i]) continue;
    if (np >= budget) return -1;
    if (keep) {
      keep->pi[np] = ii;
      keep->pv[np] = a[i];
    }
    ++np;
  }
  return np;
}

}  // namespace

bool fit_array_model(const std::vector<int64_t>& a, int budget, IdxModel* out) {
  const int64_t n = (int64_t)a.size();
  if (n < 2 || budget < 0) return false;
  budget = std::min(budget, kMaxPatches);
  struct Cand {
    int kind;
    int64_t b, k1, k2, w;
  };
  std::vector<Cand> cands;
  for (int64_t j : {int64_t(0), n / 2, n - 2})
    if (j >= 0 && j + 1 < n) {
      const int64_t k = a[j + 1] - a[j];
      cands.push_back({1, a[j] - k * j, k, 0, 1});
    }
  for (int64_t w = 2; w <= 256 && w < n; w *= 2) cands.push_back({2, a[0], a[w] - a[0], a[1] - a[0], w});
  int64_t run = 1;
  while (run < n && a[run] == a[0]) ++run;
  if (run < n) cands.push_back({3, a[0], a[run] - a[0], 0, run});
  int best = -1, best_np = budget + 1;
  for (size_t c = 0; c < cands.size(); ++c) {
    const int np = count_patches(a, cands[c].b, cands[c].k1, cands[c].k2, cands[c].w, budget, nullptr);
    if (np >= 0 && np < best_np) {
      best = (int)c;
      best_np = np;
    }
  }
  if (best < 0) return false;
  IdxModel m;
  m.kind = cands[best].kind;
  m.b = cands[best].b;
  m.k1 = cands[best].k1;
  m.k2 = cands[best].k2;
  m.w = cands[best].w;
  m.np = count_patches(a, m.b, m.k1, m.k2, m.w, budget, &m);
  *out = m;
  return true;
}

// Necessary condition for fit_array_model(a) on a long array seen through its first
// elements `pre` (>= 258 of them) and a[n/2], a[n/2+1], a[n-2], a[n-1]: the same candidates,
// patches counted on the prefix only (a lower bound of the full count).  false => no model
// fits, so the caller can skip reading the whole array (device builds of 10^7-entry arrays).
bool model_may_fit(const std::vector<int64_t>& pre, int64_t n, int64_t am0, int64_t am1, int64_t al0, int64_t al1,
                   int budget) {
  const int64_t np = (int64_t)pre.size();
  if (np < 258 || np >= n) return true;
  budget = std::min(budget, kMaxPatches);
  std::vector<std::array<int64_t, 4>> cands;  // b, k1, k2, w
  cands.push_back({pre[0] - (pre[1] - pre[0]) * 0, pre[1] - pre[0], 0, 1});
  const int64_t jm = n / 2;
  cands.push_back({am0 - (am1 - am0) * jm, am1 - am0, 0, 1});
  cands.push_back({al0 - (al1 - al0) * (n - 2), al1 - al0, 0, 1});
  for (int64_t w = 2; w <= 256 && w < n; w *= 2) cands.push_back({pre[0], pre[w] - pre[0], pre[1] - pre[0], w});
  int64_t run = 1;
  while (run < np && pre[run] == pre[0]) ++run;
  if (run == np) return true;  // the step candidate needs more of the array
  cands.push_back({pre[0], pre[run] - pre[0], 0, run});
  for (auto& c : cands)
    if (count_patches(pre, c[0], c[1], c[2], c[3], budget, nullptr) >= 0) return true;
  return false;
}

}  // namespace as

using namespace as;

extern "C" {

as_status_t as_fit_array_model(const int64_t* a, size_t n, int budget, int64_t* out) {
  return guard([&] {
    if ((n && !a) || !out) fail(AS_ERR_INVALID_ARG, "NULL argument");
    if (budget < 0 || budget > kMaxPatches) fail(AS_ERR_INVALID_ARG, "budget must be in [0, 8]");
    IdxModel m;
    // the device build's shortcut: a prefix probe rejects most non-model arrays (model_may_fit)
    if (n > 8192 && !model_may_fit(std::vector<int64_t>(a, a + 4096), (int64_t)n, a[n / 2], a[n / 2 + 1], a[n - 2],
                                   a[n - 1], budget))
      fail(AS_ERR_NOT_FOUND, "no model within the patch budget");
    if (!fit_array_model(std::vector<int64_t>(a, a + n), budget, &m)) fail(AS_ERR_NOT_FOUND, "no model within the patch budget");
    out[0] = m.kind;
    out[1] = m.b;
    out[2] = m.k1;
    out[3] = m.k2;
    out[4] = m.w;
    out[5] = m.np;
    for (int j = 0; j < m.np; ++j) {
      out[6 + 2 * j] = m.pi[j];
      out[7 + 2 * j] = m.pv[j];
    }
  });
}

}  // extern "C"
