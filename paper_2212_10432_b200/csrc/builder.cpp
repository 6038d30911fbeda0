// Designer + Format construction: executes an Operator Graph on the Matrix Metadata Set
// ("Designer would execute the complete graph by executing its operators in orders, which
// include logic to modify Matrix Metadata Set"; §V-A), extracts the arrays the
// kernel reads (§V-B) and lowers the implementing stage onto the sm_100a kernel
// family (§V-C: distribution = mapping stage, reduction = implementing stage).
//
// Readings: A6 empty rows, A7-A9 SORT/SORT_SUB/BIN, A10-A11
// ROW/COL_DIV, A12 DIA_DECOM, A13 DENSE_DECOM, A14 COMPRESS, A15 block cutting, A16 P1
// checks, A17 implicit arrays, A18 BMT_PAD, A19 SORT_BMTB, A20 bitmaps, A22 writer rule.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <unordered_map>

#include "internal.h"

namespace as {

namespace {

struct BState {
  std::vector<int64_t> rows;                   // global rows, current order
  std::shared_ptr<std::vector<uint8_t>> mask;  // per canonical entry; null = all present
  bool contiguous = true;                      // rows r0..r1-1 ascending, unpermuted
};

inline bool live(const BState& st, int64_t e) { return !st.mask || (*st.mask)[e]; }

std::vector<int64_t> row_lengths(const Matrix& A, const BState& st) {
  std::vector<int64_t> L(st.rows.size());
  parallel_for((int64_t)st.rows.size(), [&](int64_t a, int64_t e) {
    for (int64_t i = a; i < e; ++i) {
      int64_t r = st.rows[i];
      if (!st.mask) {
        L[i] = A.row_ptr[r + 1] - A.row_ptr[r];
      } else {
        int64_t c = 0;
        for (int64_t k = A.row_ptr[r]; k < A.row_ptr[r + 1]; ++k) c += (*st.mask)[k];
        L[i] = c;
      }
    }
  });
  return L;
}

// Stable permutation by descending length within [a, e) of idx (A7).
void stable_desc(std::vector<int64_t>& idx, const std::vector<int64_t>& len, size_t a, size_t e) {
  std::stable_sort(idx.begin() + a, idx.begin() + e, [&](int64_t x, int64_t y) { return len[x] > len[y]; });
}

// AS_TRACE=1: phase timings of the builder on stderr (developer aid)
void trace(const char* phase) {
  static const bool on = std::getenv("AS_TRACE") != nullptr;
  static auto last = std::chrono::steady_clock::now();
  auto now = std::chrono::steady_clock::now();
  if (on) std::fprintf(stderr, "[as_plan] %-24s %8.3f s\n", phase, std::chrono::duration<double>(now - last).count());
  nvtxMarkA(phase);  // builder phase boundary on the NVTX timeline
  last = now;
}

int64_t row_of(const std::vector<int64_t>& rp, int64_t e) {
  return (int64_t)(std::upper_bound(rp.begin(), rp.end(), e) - rp.begin()) - 1;
}

struct Builder {
  const Matrix& A;
  HostPlan& hp;
  Builder(const Matrix& a, HostPlan& h) : A(a), hp(h) {}

  void run(const Seq& s, BState st) {
    for (size_t k = 0; k < s.size(); ++k) {
      const Op& op = s[k];
      const std::string& nm = op.name;
      if (nm == "ROW_DIV") {
        auto& cuts = op.getl("cuts");
        int64_t mb = (int64_t)st.rows.size();
        if (cuts.back() >= mb) fail(AS_ERR_PLAN_INFEASIBLE, "ROW_DIV cut " + std::to_string(cuts.back()) + " >= rows " + std::to_string(mb));
        std::vector<int64_t> b = {0};
        b.insert(b.end(), cuts.begin(), cuts.end());
        b.push_back(mb);
        for (size_t i = 0; i < op.br.size(); ++i) {
          BState sub;
          sub.rows.assign(st.rows.begin() + b[i], st.rows.begin() + b[i + 1]);
          sub.mask = st.mask;
          sub.contiguous = st.contiguous;
          run(op.br[i], std::move(sub));
        }
        return;
      }
      if (nm == "COL_DIV") {
        auto& cuts = op.getl("cuts");
        if (cuts.back() >= A.n) fail(AS_ERR_PLAN_INFEASIBLE, "COL_DIV cut >= n");
        std::vector<int64_t> b = {0};
        b.insert(b.end(), cuts.begin(), cuts.end());
        b.push_back(A.n);
        for (size_t i = 0; i < op.br.size(); ++i) {
          auto mk = std::make_shared<std::vector<uint8_t>>(A.nnz());
          auto& M = *mk;
          int64_t lo = b[i], hi = b[i + 1];
          parallel_for(A.nnz(), [&](int64_t a, int64_t e) {
            for (int64_t j = a; j < e; ++j) M[j] = (A.col[j] >= lo && A.col[j] < hi) && live(st, j);
          });
          BState sub{st.rows, mk, st.contiguous};
          run(op.br[i], std::move(sub));
        }
        return;
      }
      if (nm == "SORT" || nm == "SORT_SUB") {
        auto L = row_lengths(A, st);
        std::vector<int64_t> idx(st.rows.size());
        std::iota(idx.begin(), idx.end(), 0);
        size_t g = nm == "SORT" ? idx.size() : (size_t)op.geti("g");
        if (g == 0) g = 1;
        for (size_t a = 0; a < idx.size(); a += g) stable_desc(idx, L, a, std::min(idx.size(), a + g));
        std::vector<int64_t> rows(idx.size());
        for (size_t i = 0; i < idx.size(); ++i) rows[i] = st.rows[idx[i]];
        st.rows.swap(rows);
        st.contiguous = false;
        continue;
      }
      if (nm == "BIN") {
        auto& t = op.getl("t");
        auto L = row_lengths(A, st);
        for (size_t bi = 0; bi < op.br.size(); ++bi) {
          int64_t lo = bi == 0 ? 0 : t[bi - 1];
          int64_t hi = bi < t.size() ? t[bi] : INT64_MAX;
          BState sub;
          sub.mask = st.mask;
          sub.contiguous = false;
          for (size_t i = 0; i < L.size(); ++i)
            if (L[i] > lo && L[i] <= hi) sub.rows.push_back(st.rows[i]);
          run(op.br[bi], std::move(sub));
        }
        return;
      }
      if (nm == "HYB_DECOM") {
        // HYB decomposition (NEXT-4; the operator P:583 names as missing): the first w live
        // nonzeros of every row form branch 0 (the ELL part), the rest branch 1 (the COO
        // part); both are ordinary sub-graphs and their partial sums meet in y.
        const int64_t w = op.geti("w");
        auto m0 = std::make_shared<std::vector<uint8_t>>(A.nnz(), 0);
        auto m1 = std::make_shared<std::vector<uint8_t>>(A.nnz(), 0);
        parallel_for((int64_t)st.rows.size(), [&](int64_t a, int64_t e) {
          for (int64_t i = a; i < e; ++i) {
            const int64_t r = st.rows[i];
            int64_t k = 0;
            for (int64_t j = A.row_ptr[r]; j < A.row_ptr[r + 1]; ++j)
              if (live(st, j)) ((k++ < w) ? (*m0)[j] : (*m1)[j]) = 1;
          }
        });
        run(op.br[0], BState{st.rows, m0, st.contiguous});
        run(op.br[1], BState{st.rows, m1, st.contiguous});
        return;
      }
      if (nm == "DIA_DECOM") {
        dia_decom(op, st);
        return;
      }
      if (nm == "DENSE_DECOM") {
        dense_decom(op, st);
        return;
      }
      if (nm == "COMPRESS") {
        compress_and_map(st, s, k + 1);
        return;
      }
      fail(AS_ERR_INVALID_ARG, "unexpected operator " + nm);
    }
  }

  void residual(const Op& op, BState st) {
    if (op.br.size() == 2) {
      run(op.br[1], std::move(st));
      return;
    }
    auto L = row_lengths(A, st);
    for (auto x : L)
      if (x) fail(AS_ERR_PLAN_INFEASIBLE, op.name + ": residual is non-empty but the graph gives it no branch");
  }

  // ---------------------------------------------------------------- DIA_DECOM (A12)
  void dia_decom(const Op& op, const BState& st) {
    if (!st.contiguous) fail(AS_ERR_PLAN_INFEASIBLE, "DIA_DECOM needs contiguous unpermuted rows");
    double theta = op.getf("theta");
    int64_t dmax = op.geti("max");
    int64_t mb = (int64_t)st.rows.size();
    int64_t r0 = mb ? st.rows[0] : 0;
    int64_t omin = -(r0 + mb - 1), span = A.n + mb - 1;  // offsets o in [omin, n-1-r0]
    std::vector<int64_t> cnt(mb ? (size_t)span : 0, 0);
    for (int64_t i = 0; i < mb; ++i) {
      int64_t r = r0 + i;
      for (int64_t e = A.row_ptr[r]; e < A.row_ptr[r + 1]; ++e)
        if (live(st, e)) cnt[(size_t)(A.col[e] - r - omin)]++;
    }
    std::vector<int64_t> sel;
    for (size_t j = 0; j < cnt.size(); ++j) {
      if (!cnt[j]) continue;
      int64_t o = (int64_t)j + omin;
      // len_o = #band rows r with 0 <= r + o < n
      int64_t lo = std::max(r0, -o), hi = std::min(r0 + mb, A.n - o);
      int64_t len = std::max<int64_t>(0, hi - lo);
      if ((double)cnt[j] >= theta * (double)len) sel.push_back(o);
    }
    if ((int64_t)sel.size() > dmax) {
      std::sort(sel.begin(), sel.end(), [&](int64_t a, int64_t b) {
        int64_t ca = cnt[a - omin], cb = cnt[b - omin];
        if (ca != cb) return ca > cb;
        if (std::llabs(a) != std::llabs(b)) return std::llabs(a) < std::llabs(b);
        return a < b;
      });
      sel.resize(dmax);
    }
    std::sort(sel.begin(), sel.end());
    int64_t D = (int64_t)sel.size();
    HostPart P;
    P.kind = "dia";
    P.r0 = r0;
    P.mb = D ? mb : 0;
    P.dia_off = sel;
    P.dia_val.assign((size_t)(D * mb), 0.0);
    auto mk = std::make_shared<std::vector<uint8_t>>(A.nnz());
    auto& M = *mk;
    for (int64_t e = 0; e < A.nnz(); ++e) M[e] = live(st, e);
    std::vector<int64_t> dpos(cnt.size(), -1);
    for (int64_t d = 0; d < D; ++d) dpos[(size_t)(sel[d] - omin)] = d;
    for (int64_t i = 0; i < mb && D; ++i) {
      int64_t r = r0 + i;
      for (int64_t e = A.row_ptr[r]; e < A.row_ptr[r + 1]; ++e) {
        if (!M[e]) continue;
        int64_t d = dpos[(size_t)(A.col[e] - r - omin)];
        if (d >= 0) {
          P.dia_val[(size_t)(d * mb + i)] = A.val[e];
          M[e] = 0;
        }
      }
    }
    if (D) {
      P.origin.resize(mb);
      std::iota(P.origin.begin(), P.origin.end(), r0);
      P.excl = P.origin;
    }
    P.fam = FAM_DIA;
    P.fam_name = "dia";
    if (op.br[0].size() > 1) {
      P.tpb = (int)op.br[0][1].geti("tpb");
      P.grid = (int)op.br[0][1].geti("grid");
      P.stages = (int)op.br[0][1].geti("stages");
      P.stream = (int)op.br[0][1].geti("stream");
    }
    hp.parts.push_back(std::move(P));
    residual(op, BState{st.rows, mk, true});
  }

  // ---------------------------------------------------------------- DENSE_DECOM (A13)
  void dense_decom(const Op& op, const BState& st) {
    if (!st.contiguous) fail(AS_ERR_PLAN_INFEASIBLE, "DENSE_DECOM needs contiguous unpermuted rows");
    int64_t b = op.geti("b");
    double theta = op.getf("theta");
    int64_t mb = (int64_t)st.rows.size();
    int64_t r0 = mb ? st.rows[0] : 0, r1 = r0 + mb;
    // per tile row I (b rows): the column tiles J of its live nonzeros, sorted; a tile is
    // selected when it holds >= theta*b^2 of them.  Tile rows are independent -> parallel.
    const int64_t I0 = mb ? r0 / b : 0, nI = mb ? (r1 - 1) / b - I0 + 1 : 0;
    const double need = theta * (double)(b * b);
    std::vector<std::vector<int64_t>> sel((size_t)nI);
    parallel_for(
        nI,
        [&](int64_t ia, int64_t ie) {
          std::vector<int64_t> js;
          for (int64_t ii = ia; ii < ie; ++ii) {
            const int64_t I = I0 + ii;
            js.clear();
            for (int64_t r = std::max(I * b, r0); r < std::min(I * b + b, r1); ++r)
              for (int64_t e = A.row_ptr[r]; e < A.row_ptr[r + 1]; ++e)
                if (live(st, e)) js.push_back(A.col[e] / b);
            std::sort(js.begin(), js.end());
            for (size_t u = 0; u < js.size();) {
              size_t v = u;
              while (v < js.size() && js[v] == js[u]) ++v;
              if ((double)(v - u) >= need) sel[(size_t)ii].push_back(js[u]);
              u = v;
            }
          }
        },
        256);
    HostPart P;
    P.kind = "dense";
    P.b = b;
    P.r0 = r0;
    P.mb = mb;
    std::vector<int64_t> tile_of_row((size_t)nI + 1, 0);  // first tile index of tile row ii
    for (int64_t ii = 0; ii < nI; ++ii) {
      tile_of_row[(size_t)ii + 1] = tile_of_row[(size_t)ii] + (int64_t)sel[(size_t)ii].size();
      if (sel[(size_t)ii].empty()) continue;
      P.tile_row_id.push_back(I0 + ii);
      P.tile_row_ptr.push_back(tile_of_row[(size_t)ii]);
      for (int64_t J : sel[(size_t)ii]) P.tile_col.push_back(J);
    }
    const int64_t T = tile_of_row[(size_t)nI];
    P.tile_row_ptr.push_back(T);
    P.tile_val.assign((size_t)(T * b * b), 0.0);
    auto mk = std::make_shared<std::vector<uint8_t>>(A.nnz());
    auto& M = *mk;
    parallel_for(A.nnz(), [&](int64_t a0, int64_t e0) {
      for (int64_t e = a0; e < e0; ++e) M[e] = live(st, e);
    });
    if (T) {
      parallel_for(
          nI,
          [&](int64_t ia, int64_t ie) {
            for (int64_t ii = ia; ii < ie; ++ii) {
              const std::vector<int64_t>& js = sel[(size_t)ii];
              if (js.empty()) continue;
              const int64_t I = I0 + ii;
              for (int64_t r = std::max(I * b, r0); r < std::min(I * b + b, r1); ++r)
                for (int64_t e = A.row_ptr[r]; e < A.row_ptr[r + 1]; ++e) {
                  if (!M[e]) continue;
                  const int64_t J = A.col[e] / b;
                  auto it = std::lower_bound(js.begin(), js.end(), J);
                  if (it == js.end() || *it != J) continue;
                  const int64_t t = tile_of_row[(size_t)ii] + (it - js.begin());
                  const int64_t i = r - I * b, j = A.col[e] - J * b;
                  P.tile_val[(size_t)(t * b * b + j * b + i)] = A.val[e];
                  M[e] = 0;
                }
            }
          },
          256);
      for (int64_t I : P.tile_row_id)
        for (int64_t r = I * b; r < I * b + b; ++r)
          if (r >= r0 && r < r1) P.excl.push_back(r);
    }
    P.origin = P.excl;
    P.fam = FAM_DENSE;
    P.fam_name = "dense";
    if (op.br[0].size() > 1) {
      P.tpb = (int)op.br[0][1].geti("tpb");
      P.grid = (int)op.br[0][1].geti("grid");
      P.stages = (int)op.br[0][1].geti("stages");
      P.stream = (int)op.br[0][1].geti("stream");
    }
    hp.parts.push_back(std::move(P));
    residual(op, BState{st.rows, mk, true});
  }

  // ---------------------------------------------------------------- COMPRESS + mapping
  void compress_and_map(const BState& st, const Seq& s, size_t from) {
    HostPart P;
    P.kind = "csr";
    // COMPRESS (A14): rows in the current order, empty rows compacted (A6)
    auto L = row_lengths(A, st);
    for (size_t i = 0; i < st.rows.size(); ++i)
      if (L[i]) P.origin.push_back(st.rows[i]);
    int64_t mp = (int64_t)P.origin.size();
    P.row_ptr.assign(mp + 1, 0);
    {
      int64_t j = 0;
      for (size_t i = 0; i < st.rows.size(); ++i)
        if (L[i]) {
          P.row_ptr[j + 1] = P.row_ptr[j] + L[i];
          ++j;
        }
    }
    int64_t nnz = P.row_ptr[mp];
    P.col.resize(nnz);
    P.val.resize(nnz);
    parallel_for(mp, [&](int64_t a, int64_t e) {
      for (int64_t i = a; i < e; ++i) {
        int64_t r = P.origin[i], o = P.row_ptr[i];
        for (int64_t k = A.row_ptr[r]; k < A.row_ptr[r + 1]; ++k)
          if (live(st, k)) {
            P.col[o] = A.col[k];
            P.val[o] = A.val[k];
            ++o;
          }
      }
    });

    trace("compress");
    // collect the mapping / implementing operators
    std::vector<int> order;
    const Op* pad = nullptr;
    for (size_t k = from; k < s.size(); ++k) {
      const Op& op = s[k];
      const std::string& nm = op.name;
      if (nm.size() > 6 && nm.substr(nm.size() - 6) == "_BLOCK") {
        int l = nm.rfind("BMTB_", 0) == 0 ? 0 : nm.rfind("BMW_", 0) == 0 ? 1 : 2;
        P.lv[l].present = true;
        P.lv[l].nnz = nm.find("_NNZ_") != std::string::npos;
        P.lv[l].size = op.params[0].second.i;
        order.push_back(l);
      } else if (nm == "BMT_PAD") {
        pad = &op;
      } else if (nm == "SORT_BMTB") {
        P.sort_bmtb = true;
      } else if (nm == "SET_RESOURCE") {
        P.tpb = (int)op.geti("tpb");
        P.grid = (int)op.geti("grid");
        P.stages = (int)op.geti("stages");
        P.xcache = op.geti("xcache");
        P.stream = (int)op.geti("stream");
      } else if (nm == "THREAD_TOTAL_RED") P.red[2] = RED_TOTAL;
      else if (nm == "THREAD_BITMAP_RED_G") P.red[2] = RED_BITMAP;
      else if (nm == "WARP_TOTAL_RED") P.red[1] = RED_TOTAL;
      else if (nm == "WARP_BITMAP_RED") P.red[1] = RED_BITMAP;
      else if (nm == "WARP_SEG_ADD_RED") P.red[1] = RED_SEG;
      else if (nm == "SHMEM_TOTAL_RED") P.red[0] = RED_TOTAL;
      else if (nm == "SHMEM_OFFSET_RED") P.red[0] = RED_OFFSET;
    }

    // block cutting (A15): children restart at each parent; ROW children group row fragments
    std::vector<int64_t> parent = {0, nnz};
    if (nnz == 0) parent = {0};
    for (int l : order) {
      Level& lv = P.lv[l];
      lv.start = cut(P.row_ptr, parent, lv.nnz, lv.size);
      if (l == 0 && P.sort_bmtb) sort_bmtb(P);
      parent = lv.start;
    }
    trace("cut+sort_bmtb");
    for (int l : order) first_rows(P.row_ptr, P.lv[l]);
    trace("first_rows");

    // P1 (A16): X_TOTAL_RED needs every level-X block inside one row
    for (int l = 0; l < 3; ++l) {
      if (P.red[l] != RED_TOTAL) continue;
      Level& lv = P.lv[l];
      // a block [a, e) lies in one row iff its last element is before the next row start
      for (int64_t t = 0; t < lv.count(); ++t)
        if (lv.start[t + 1] > P.row_ptr[lv.first_row[t] + 1])
          fail(AS_ERR_PLAN_INFEASIBLE, std::string("P1: ") + (l == 0 ? "SHMEM" : l == 1 ? "WARP" : "THREAD") +
                                           "_TOTAL_RED but a block spans rows");
    }

    // bitmaps (A20)
    if (P.red[2] == RED_BITMAP && P.lv[2].nnz) {
      Level& bt = P.lv[2];
      P.bm_words = (int)((bt.size + 31) / 32);
      P.bitmap.assign((size_t)(bt.count() * P.bm_words), 0u);
      parallel_for(mp, [&](int64_t ra, int64_t re) {
        int64_t t = ra < mp ? std::upper_bound(bt.start.begin(), bt.start.end(), P.row_ptr[ra]) - bt.start.begin() - 1 : 0;
        for (int64_t r = ra; r < re; ++r) {
          int64_t h = P.row_ptr[r];
          while (bt.start[t + 1] <= h) ++t;
          int64_t j = h - bt.start[t];
          __atomic_fetch_or(&P.bitmap[(size_t)(t * P.bm_words + j / 32)], 1u << (j % 32), __ATOMIC_RELAXED);
        }
      });
    }

    trace("p1+bitmap");
    if (pad) build_pad(P, *pad);
    trace("pad");

    // writer units: blocks of the highest level carrying a reduction (A21/A22)
    int top = -1;
    for (int l = 2; l >= 0; --l)
      if (P.red[l] != RED_NONE) top = l;  // smallest index = coarsest level
    std::vector<int64_t> unit_start;
    if (top >= 0) unit_start = P.lv[top].start;
    {
      int64_t u = 0;
      for (int64_t r = 0; r < mp; ++r) {
        int64_t a = P.row_ptr[r], e = P.row_ptr[r + 1];
        bool ex;
        if (top < 0) {
          ex = (e - a) == 1;
        } else {
          while (unit_start[u + 1] <= a) ++u;
          ex = e <= unit_start[u + 1];
        }
        (ex ? P.excl : P.atom).push_back(P.origin[r]);
      }
    }
    trace("writer_units");
    lower(P);
    hp.parts.push_back(std::move(P));
  }

  static std::vector<int64_t> cut(const std::vector<int64_t>& rp, const std::vector<int64_t>& parent, bool nnz,
                                  int64_t size) {
    std::vector<int64_t> out;
    int64_t np = (int64_t)parent.size() - 1;
    int64_t r = 0;
    for (int64_t p = 0; p < np; ++p) {
      int64_t a = parent[p], e = parent[p + 1];
      if (nnz) {
        for (int64_t x = a; x < e; x += size) out.push_back(x);
      } else {
        // fragments = rows intersecting [a, e)
        while (rp[r + 1] <= a) ++r;
        int64_t cntf = 0;
        for (int64_t q = r; q + 1 < (int64_t)rp.size() && rp[q] < e; ++q) {
          if (rp[q + 1] <= a) continue;
          if (cntf % size == 0) out.push_back(std::max(rp[q], a));
          ++cntf;
        }
      }
    }
    out.push_back(parent.back());
    return out;
  }

  static void first_rows(const std::vector<int64_t>& rp, Level& lv) {
    lv.first_row.resize(lv.count());
    int64_t r = 0;
    for (int64_t t = 0; t < lv.count(); ++t) {
      while (rp[r + 1] <= lv.start[t]) ++r;
      lv.first_row[t] = r;
    }
  }

  // SORT_BMTB (A19): stable descending sort of the (whole) rows inside each BMTB
  void sort_bmtb(HostPart& P) {
    Level& bt = P.lv[0];
    int64_t mp = (int64_t)P.origin.size();
    std::vector<int64_t> len(mp), perm(mp);
    for (int64_t r = 0; r < mp; ++r) len[r] = P.row_ptr[r + 1] - P.row_ptr[r];
    std::iota(perm.begin(), perm.end(), 0);
    parallel_for(
        bt.count(),
        [&](int64_t b0, int64_t b1) {
          for (int64_t b = b0; b < b1; ++b) {
            int64_t ra = row_of(P.row_ptr, bt.start[b]), re = row_of(P.row_ptr, bt.start[b + 1] - 1) + 1;
            stable_desc(perm, len, ra, re);
          }
        },
        1 << 10);
    std::vector<int64_t> org(mp), rp(mp + 1, 0);
    std::vector<int32_t> col(P.col.size());
    std::vector<double> val(P.val.size());
    for (int64_t i = 0; i < mp; ++i) {
      org[i] = P.origin[perm[i]];
      rp[i + 1] = rp[i] + len[perm[i]];
    }
    parallel_for(mp, [&](int64_t a, int64_t e) {
      for (int64_t i = a; i < e; ++i) {
        int64_t r = perm[i];
        std::copy(P.col.begin() + P.row_ptr[r], P.col.begin() + P.row_ptr[r + 1], col.begin() + rp[i]);
        std::copy(P.val.begin() + P.row_ptr[r], P.val.begin() + P.row_ptr[r + 1], val.begin() + rp[i]);
      }
    });
    P.origin.swap(org);
    P.row_ptr.swap(rp);
    P.col.swap(col);
    P.val.swap(val);
  }

  // BMT_PAD (A18): slot-major interleaved in units of vec; pad col = last real col
  void build_pad(HostPart& P, const Op& op) {
    const std::string& sc = op.gets("scope");
    P.pad = true;
    P.pad_scope = sc == "GLOBAL" ? -1 : sc == "BMTB" ? 0 : 1;
    int64_t vec = op.geti("vec");
    if (vec == 0) vec = hp.dt == AS_R64F ? 2 : 4;
    P.vec = (int)vec;
    Level& bt = P.lv[2];
    std::vector<int64_t> groups = P.pad_scope < 0 ? std::vector<int64_t>{0, bt.start.back()} : P.lv[P.pad_scope].start;
    int64_t ng = (int64_t)groups.size() - 1;
    int64_t t = 0, base = 0;
    P.grp_first_bmt.clear();
    for (int64_t g = 0; g < ng; ++g) {
      int64_t t0 = t;
      int64_t W = 0;
      while (t < bt.count() && bt.start[t] >= groups[g] && bt.start[t + 1] <= groups[g + 1]) {
        W = std::max(W, bt.start[t + 1] - bt.start[t]);
        ++t;
      }
      W = (W + vec - 1) / vec * vec;
      P.grp_first_bmt.push_back(t0);
      P.grp_base.push_back(base);
      P.pad_width.push_back(W);
      base += (t - t0) * W;
    }
    P.grp_first_bmt.push_back(t);
    // P4b: the padded layout may not exceed 4x the nonzeros (+1M slots); an
    // ELL over a power-law matrix would otherwise need max_len x rows slots.
    const int64_t nnz = bt.start.empty() ? 0 : bt.start.back();
    if (base > 4 * nnz + (int64_t(1) << 20))
      fail(AS_ERR_PLAN_INFEASIBLE, "P4b: BMT_PAD would store " + std::to_string(base) + " slots for " +
                                       std::to_string(nnz) + " nonzeros (padding rate above 4x)");
    P.pad_col.assign((size_t)base, 0);
    P.pad_val.assign((size_t)base, 0.0);
    // fill: groups are independent; GLOBAL scope (one group) splits over its BMTs
    auto fill = [&](int64_t g, int64_t ta, int64_t te) {
      int64_t t0 = P.grp_first_bmt[g], nt = P.grp_first_bmt[g + 1] - t0, W = P.pad_width[g];
      for (int64_t tt = ta; tt < te; ++tt) {
        int64_t a = bt.start[tt], e = bt.start[tt + 1], lt = tt - t0;
        for (int64_t j = 0; j < W; ++j) {
          int64_t slot = P.grp_base[g] + (j / vec) * nt * vec + lt * vec + (j % vec);
          if (a + j < e) {
            P.pad_col[slot] = P.col[a + j];
            P.pad_val[slot] = P.val[a + j];
          } else {
            P.pad_col[slot] = P.col[e - 1];
          }
        }
      }
    };
    if (ng == 1) {
      parallel_for(P.grp_first_bmt[1], [&](int64_t a, int64_t e) { fill(0, a, e); }, 1 << 12);
    } else {
      parallel_for(
          ng,
          [&](int64_t a, int64_t e) {
            for (int64_t g = a; g < e; ++g) fill(g, P.grp_first_bmt[g], P.grp_first_bmt[g + 1]);
          },
          1 << 8);
    }
  }

  // Implementing stage -> kernel family; anything else is infeasible here.
  void lower(HostPart& P) {
    Level *B = &P.lv[0], *W = &P.lv[1], *T = &P.lv[2];
    Red rb = P.red[0], rw = P.red[1], rt = P.red[2];
    auto no = [](const Level* l) { return !l->present; };
    if (T->present && !T->nnz && (no(W) || !W->nnz) && (no(B) || !B->nnz) && rt != RED_NONE && rw == RED_NONE &&
        rb == RED_NONE) {
      P.fam = FAM_THREAD_ROW;
      P.fam_name = P.pad ? "thread_row_pad" : "thread_row";
    } else if (T->present && T->nnz && no(W) && rt == RED_BITMAP && rw == RED_NONE && rb == RED_NONE) {
      P.fam = FAM_NNZ_THREAD;
      P.fam_name = "nnz_thread_bitmap";
    } else if (T->present && T->nnz && W->present && rt == RED_BITMAP && (rw == RED_SEG || rw == RED_BITMAP) &&
               rb == RED_NONE) {
      P.fam = FAM_NNZ_WARP;
      P.fam_name = rw == RED_SEG ? "nnz_warp_seg" : "nnz_warp_bitmap";
    } else if (W->present && rw == RED_TOTAL && (no(T) || (T->nnz && rt == RED_TOTAL)) && rb == RED_NONE) {
      P.fam = FAM_WARP_ROW;
      P.fam_name = "warp_row";
    } else if (B->present && rb == RED_TOTAL && no(W) && no(T)) {
      P.fam = FAM_BLOCK_TOTAL;
      P.fam_name = "block_total";
    } else if (B->present && rb == RED_OFFSET && no(W) && no(T)) {
      P.fam = FAM_BLOCK_OFFSET;
      P.fam_name = "block_offset";
    } else {
      P.fam = FAM_COMPOSE;
    }
    // BMT_PAD is read by the THREAD_ROW and NNZ families and by the composed kernel
    if (P.pad && P.fam != FAM_THREAD_ROW && P.fam != FAM_NNZ_THREAD && P.fam != FAM_NNZ_WARP) P.fam = FAM_COMPOSE;
    if (P.fam == FAM_COMPOSE) {
      // the Kernel Builder's per-level fragments: name = levels + reductions
      static const char* rn[] = {"", "total", "bitmap", "seg", "offset"};
      P.fam_name = "compose";
      const char* ln[] = {"b", "w", "t"};
      for (int l = 0; l < 3; ++l)
        if (P.lv[l].present || P.red[l] != RED_NONE)
          P.fam_name += std::string("_") + ln[l] + (P.red[l] != RED_NONE ? rn[P.red[l]] : "");
      if (P.pad) P.fam_name += "_pad";
    }
  }
};

// A22 writer rule (see oracle/builder_ref.writer_rule for the same reading).
void writer_rule(HostPlan& hp) {
  std::vector<int64_t> live;
  for (size_t i = 0; i < hp.parts.size(); ++i)
    if (!hp.parts[i].excl.empty() || !hp.parts[i].atom.empty()) live.push_back((int64_t)i);
  std::stable_sort(live.begin(), live.end(),
                   [&](int64_t a, int64_t b) { return hp.parts[a].excl.size() > hp.parts[b].excl.size(); });
  // R-conc: the main stream is the stream of the first part in launch order; parts naming
  // another stream run beside it into a scratch vector of their own (mode 3), added into y
  // after the streams join -- so the rule below runs over the main-stream parts only, and
  // rows of side parts that no main part writes join the pre-pass (y <- beta*y first)
  const int main_stream = live.empty() ? 0 : hp.parts[live[0]].stream;
  std::vector<uint8_t> written(hp.m, 0), pre(hp.m, 0);
  for (int64_t i : live) {
    HostPart& p = hp.parts[i];
    if (p.stream != main_stream) continue;
    bool all_first = true;
    for (int64_t r : p.excl)
      if (written[r]) {
        all_first = false;
        break;
      }
    p.mode = all_first ? 0 : 1;
    if (!all_first)
      for (int64_t r : p.excl)
        if (!written[r]) pre[r] = 1;
    for (int64_t r : p.atom)
      if (!written[r]) pre[r] = 1;
    for (int64_t r : p.excl) written[r] = 1;
    for (int64_t r : p.atom) written[r] = 1;
  }
  for (int64_t i : live) {
    HostPart& p = hp.parts[i];
    if (p.stream == main_stream) continue;
    p.mode = 3;
    for (int64_t r : p.excl)
      if (!written[r]) pre[r] = 1;
    for (int64_t r : p.atom)
      if (!written[r]) pre[r] = 1;
  }
  for (int64_t r = 0; r < hp.m; ++r)
    if (pre[r] || !written[r]) hp.prepass.push_back(r);
  hp.launch_order = live;
}

}  // namespace

HostPlan build_plan(const Matrix& A, const Seq& g) {
  HostPlan hp;
  hp.m = A.m;
  hp.n = A.n;
  hp.dt = A.dt;
  Builder b(A, hp);
  BState st;
  st.rows.resize(A.m);
  std::iota(st.rows.begin(), st.rows.end(), 0);
  b.run(g, std::move(st));
  writer_rule(hp);
  std::vector<uint8_t> seen(A.n, 0);
  parallel_for(A.nnz(), [&](int64_t a, int64_t e) {
    for (int64_t i = a; i < e; ++i) __atomic_store_n(&seen[A.col[i]], (uint8_t)1, __ATOMIC_RELAXED);
  });
  hp.distinct_cols = std::accumulate(seen.begin(), seen.end(), (int64_t)0);
  return hp;
}

// ------------------------------------------------------------------ export (logical arrays)
namespace {
template <class T>
void put(std::map<std::string, std::pair<std::vector<uint8_t>, int>>& out, const std::string& k, const std::vector<T>& v) {
  std::vector<uint8_t> b(v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(b.data(), v.data(), b.size());
  out[k] = {std::move(b), 0};
}
std::vector<int64_t> i64(const std::vector<int32_t>& v) { return std::vector<int64_t>(v.begin(), v.end()); }

void put_vals(std::map<std::string, std::pair<std::vector<uint8_t>, int>>& out, const std::string& k,
              const std::vector<double>& v, as_dtype_t dt) {
  if (dt == AS_R64F) return put(out, k, v);
  std::vector<float> f(v.begin(), v.end());
  put(out, k, f);
}

std::map<std::string, std::pair<std::vector<uint8_t>, int>> export_all(const HostPlan& hp) {
  std::map<std::string, std::pair<std::vector<uint8_t>, int>> out;
  static const char* lname[3] = {"bmtb", "bmw", "bmt"};
  for (size_t i = 0; i < hp.parts.size(); ++i) {
    const HostPart& p = hp.parts[i];
    std::string pre = "p" + std::to_string(i) + ".";
    if (p.kind == "csr") {
      put(out, pre + "origin_rows", p.origin);
      put(out, pre + "row_ptr", p.row_ptr);
      put(out, pre + "col", i64(p.col));
      put_vals(out, pre + "val", p.val, hp.dt);
      for (int l = 0; l < 3; ++l) {
        if (!p.lv[l].present) continue;
        put(out, pre + lname[l] + ".nz_ptr", p.lv[l].start);
        put(out, pre + lname[l] + ".first_row", p.lv[l].first_row);
      }
      if (!p.bitmap.empty() || (p.red[2] == RED_BITMAP && p.lv[2].nnz)) put(out, pre + "bmt.bitmap", p.bitmap);
      if (p.pad) {
        put(out, pre + "pad.width", p.pad_width);
        std::vector<int64_t> pb = p.grp_base;  // padded slot offset of every group + total slots
        pb.push_back((int64_t)p.pad_col.size());
        put(out, pre + "pad.base", pb);
        put(out, pre + "pad.col", i64(p.pad_col));
        put_vals(out, pre + "pad.val", p.pad_val, hp.dt);
      }
      if (p.red[0] == RED_OFFSET) {
        std::vector<int64_t> ptr = {0}, offs;
        const Level& bt = p.lv[0];
        for (int64_t b = 0; b < bt.count(); ++b) {
          int64_t a = bt.start[b], e = bt.start[b + 1];
          for (int64_t r = bt.first_row[b]; r < (int64_t)p.origin.size() && p.row_ptr[r] < e; ++r)
            offs.push_back(std::max(p.row_ptr[r], a) - a);
          offs.push_back(e - a);
          ptr.push_back((int64_t)offs.size());
        }
        put(out, pre + "bmtb.reduce_ptr", ptr);
        put(out, pre + "bmtb.reduce_row_offsets", offs);
      }
    } else if (p.kind == "dia") {
      put(out, pre + "dia.off", p.dia_off);
      put_vals(out, pre + "dia.val", p.dia_val, hp.dt);
      put(out, pre + "origin_rows", p.origin);
    } else {
      put(out, pre + "tile.row_id", p.tile_row_id);
      std::vector<int64_t> rp = p.tile_row_ptr;
      put(out, pre + "tile.row_ptr", rp);
      put(out, pre + "tile.col", p.tile_col);
      put_vals(out, pre + "tile.val", p.tile_val, hp.dt);
      put(out, pre + "origin_rows", p.origin);
    }
  }
  put(out, "launch_order", hp.launch_order);
  std::vector<int64_t> mode;
  for (auto& p : hp.parts) mode.push_back(p.mode);
  put(out, "mode", mode);
  put(out, "prepass", hp.prepass);
  return out;
}
}  // namespace

bool export_key(const HostPlan& hp, const std::string& key, void* dst, size_t* bytes) {
  auto all = export_all(hp);
  auto it = all.find(key);
  if (it == all.end()) return false;
  *bytes = it->second.first.size();
  if (dst && *bytes) std::memcpy(dst, it->second.first.data(), *bytes);
  return true;
}

std::vector<std::string> export_keys(const HostPlan& hp) {
  std::vector<std::string> k;
  for (auto& kv : export_all(hp)) k.push_back(kv.first);
  return k;
}

}  // namespace as
