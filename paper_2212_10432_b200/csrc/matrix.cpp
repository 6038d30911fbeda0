// a1 Ingest: COO / CSR / Matrix Market -> canonical CSR on the host, row statistics,
// ROW_DIV bands and nnz-balanced multi-GPU cuts.
//
//   input format: Matrix Market (P:2), COO as the universal source  — reading A3
//   duplicates rejected (reading A4), empty rows accepted (reading A6, P:408 footnote)
//   statistics: avg = nnz/n, population row variance, irregular > 100
//   cuts: reading A35
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>

#include "internal.h"

namespace as {

namespace {
void check_dims(int64_t m, int64_t n) {
  if (m < 0 || n < 0 || m >= (int64_t(1) << 31) - 1 || n >= (int64_t(1) << 31) - 1)
    fail(AS_ERR_INVALID_ARG, "m and n must be in [0, 2^31-1)");
}

double load_val(const void* val, as_dtype_t dt, int64_t i) {
  return dt == AS_R64F ? ((const double*)val)[i] : (double)((const float*)val)[i];
}
}  // namespace

// COO -> canonical CSR: counting sort by row, then sort columns inside each row.
Matrix matrix_from_coo(int64_t m, int64_t n, int64_t nnz, const int64_t* row, const int64_t* col,
                       const void* val, as_dtype_t dt, int base) {
  check_dims(m, n);
  if (nnz < 0 || (nnz > 0 && (!row || !col || !val))) fail(AS_ERR_INVALID_ARG, "null triplet arrays");
  if (base != 0 && base != 1) fail(AS_ERR_INVALID_ARG, "index_base must be 0 or 1");
  if (dt != AS_R32F && dt != AS_R64F) fail(AS_ERR_DTYPE, "dtype must be AS_R32F or AS_R64F");
  Matrix A;
  A.m = m;
  A.n = n;
  A.dt = dt;
  A.row_ptr.assign(m + 1, 0);
  for (int64_t i = 0; i < nnz; ++i) {
    int64_t r = row[i] - base, c = col[i] - base;
    if (r < 0 || r >= m || c < 0 || c >= n)
      fail(AS_ERR_INDEX_OUT_OF_RANGE, "triplet " + std::to_string(i) + " (" + std::to_string(row[i]) + "," +
                                          std::to_string(col[i]) + ") outside " + std::to_string(m) + "x" + std::to_string(n));
    A.row_ptr[r + 1]++;
  }
  for (int64_t r = 0; r < m; ++r) A.row_ptr[r + 1] += A.row_ptr[r];
  // fast path: already sorted by (row, col)
  bool sorted = true;
  for (int64_t i = 1; i < nnz && sorted; ++i)
    if (row[i] < row[i - 1] || (row[i] == row[i - 1] && col[i] <= col[i - 1])) sorted = false;
  A.col.resize(nnz);
  A.val.resize(nnz);
  if (sorted) {
    parallel_for(nnz, [&](int64_t a, int64_t e) {
      for (int64_t i = a; i < e; ++i) {
        A.col[i] = (int32_t)(col[i] - base);
        A.val[i] = load_val(val, dt, i);
      }
    });
    return A;
  }
  std::vector<int64_t> pos(A.row_ptr.begin(), A.row_ptr.end() - 1);
  for (int64_t i = 0; i < nnz; ++i) {
    int64_t r = row[i] - base;
    int64_t p = pos[r]++;
    A.col[p] = (int32_t)(col[i] - base);
    A.val[p] = load_val(val, dt, i);
  }
  std::vector<std::pair<int32_t, double>> tmp;
  for (int64_t r = 0; r < m; ++r) {
    int64_t a = A.row_ptr[r], e = A.row_ptr[r + 1];
    tmp.clear();
    for (int64_t i = a; i < e; ++i) tmp.push_back({A.col[i], A.val[i]});
    std::stable_sort(tmp.begin(), tmp.end(), [](auto& x, auto& y) { return x.first < y.first; });
    for (int64_t i = a; i < e; ++i) {
      A.col[i] = tmp[i - a].first;
      A.val[i] = tmp[i - a].second;
      if (i > a && A.col[i] == A.col[i - 1])
        fail(AS_ERR_DUPLICATE, "duplicate entry (" + std::to_string(r + base) + "," + std::to_string(A.col[i] + base) + ")");
    }
  }
  return A;
}

Matrix matrix_from_csr(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const void* val,
                       as_dtype_t dt) {
  check_dims(m, n);
  if (!row_ptr || (row_ptr[m] > 0 && (!col || !val))) fail(AS_ERR_INVALID_ARG, "null CSR arrays");
  if (dt != AS_R32F && dt != AS_R64F) fail(AS_ERR_DTYPE, "dtype must be AS_R32F or AS_R64F");
  if (row_ptr[0] != 0) fail(AS_ERR_INVALID_ARG, "row_ptr[0] must be 0");
  for (int64_t r = 0; r < m; ++r)
    if (row_ptr[r + 1] < row_ptr[r]) fail(AS_ERR_INVALID_ARG, "row_ptr not monotone");
  Matrix A;
  A.m = m;
  A.n = n;
  A.dt = dt;
  A.row_ptr.assign(row_ptr, row_ptr + m + 1);
  int64_t nnz = row_ptr[m];
  A.col.assign(col, col + nnz);
  A.val.resize(nnz);
  std::vector<int> bad(1, 0);
  parallel_for(m, [&](int64_t a, int64_t e) {
    for (int64_t r = a; r < e; ++r) {
      for (int64_t i = row_ptr[r]; i < row_ptr[r + 1]; ++i) {
        if (col[i] < 0 || col[i] >= n) bad[0] = 1;
        if (i > row_ptr[r] && col[i] <= col[i - 1]) bad[0] = bad[0] ? bad[0] : 2;
        A.val[i] = load_val(val, dt, i);
      }
    }
  });
  if (bad[0] == 1) fail(AS_ERR_INDEX_OUT_OF_RANGE, "column index outside the matrix");
  if (bad[0] == 2) fail(AS_ERR_DUPLICATE, "columns must be strictly ascending within a row");
  return A;
}

Matrix matrix_from_mtx(const char* path, as_dtype_t dt) {
  std::ifstream f(path);
  if (!f) fail(AS_ERR_INVALID_ARG, std::string("cannot open ") + path);
  std::string line;
  if (!std::getline(f, line)) fail(AS_ERR_MALFORMED, "empty file");
  std::string lower = line;
  std::transform(lower.begin(), lower.end(), lower.begin(), ::tolower);
  std::istringstream hs(lower);
  std::string banner, obj, fmt, field, sym;
  hs >> banner >> obj >> fmt >> field >> sym;
  if (banner != "%%matrixmarket" || obj != "matrix" || fmt != "coordinate")
    fail(AS_ERR_MALFORMED, "only '%%MatrixMarket matrix coordinate' is supported");
  if ((field != "real" && field != "integer" && field != "pattern") || (sym != "general" && sym != "symmetric"))
    fail(AS_ERR_MALFORMED, "unsupported field/symmetry " + field + "/" + sym);
  while (std::getline(f, line))
    if (!line.empty() && line[0] != '%' && line.find_first_not_of(" \t\r") != std::string::npos) break;
  int64_t m = -1, n = -1, nnz = -1;
  {
    std::istringstream ss(line);
    if (!(ss >> m >> n >> nnz)) fail(AS_ERR_MALFORMED, "size line must be 'm n nnz'");
  }
  std::vector<int64_t> R, C;
  std::vector<double> V;
  int64_t count = 0;
  while (std::getline(f, line)) {
    if (line.empty() || line[0] == '%' || line.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::istringstream ss(line);
    int64_t r, c;
    double v = 1.0;
    if (!(ss >> r >> c)) fail(AS_ERR_MALFORMED, "bad entry line");
    if (field != "pattern" && !(ss >> v)) fail(AS_ERR_MALFORMED, "bad entry value");
    ++count;
    if (r < 1 || r > m || c < 1 || c > n) fail(AS_ERR_INDEX_OUT_OF_RANGE, "(" + std::to_string(r) + "," + std::to_string(c) + ")");
    R.push_back(r - 1);
    C.push_back(c - 1);
    V.push_back(v);
    if (sym == "symmetric" && r != c) {
      R.push_back(c - 1);
      C.push_back(r - 1);
      V.push_back(v);
    }
  }
  if (count != nnz) fail(AS_ERR_MALFORMED, "entry count does not match the size line");
  std::vector<float> Vf;
  const void* vp = V.data();
  if (dt == AS_R32F) {
    Vf.assign(V.begin(), V.end());
    vp = Vf.data();
  }
  return matrix_from_coo(m, n, (int64_t)R.size(), R.data(), C.data(), vp, dt, 0);
}

as_stats_t matrix_stats(const Matrix& A) {
  as_stats_t s{};
  s.m = A.m;
  s.n = A.n;
  s.nnz = A.nnz();
  s.min_row_len = A.m ? INT64_MAX : 0;
  for (int64_t r = 0; r < A.m; ++r) {
    int64_t L = A.row_ptr[r + 1] - A.row_ptr[r];
    s.max_row_len = std::max(s.max_row_len, L);
    s.min_row_len = std::min(s.min_row_len, L);
    s.empty_rows += L == 0;
  }
  s.avg_row_len = A.m ? (double)s.nnz / (double)A.m : 0.0;
  double acc = 0.0;
  for (int64_t r = 0; r < A.m; ++r) {
    double d = (double)(A.row_ptr[r + 1] - A.row_ptr[r]) - s.avg_row_len;
    acc += d * d;
  }
  s.row_len_variance = A.m ? acc / (double)A.m : 0.0;
  s.irregular = s.row_len_variance > 100.0;
  return s;
}

Matrix matrix_row_slice(const Matrix& A, int64_t r0, int64_t r1) {
  if (r0 < 0 || r1 < r0 || r1 > A.m) fail(AS_ERR_INVALID_ARG, "row slice out of range");
  Matrix B;
  B.m = r1 - r0;
  B.n = A.n;
  B.dt = A.dt;
  int64_t a = A.row_ptr[r0], e = A.row_ptr[r1];
  B.row_ptr.resize(B.m + 1);
  for (int64_t r = 0; r <= B.m; ++r) B.row_ptr[r] = A.row_ptr[r0 + r] - a;
  B.col.assign(A.col.begin() + a, A.col.begin() + e);
  B.val.assign(A.val.begin() + a, A.val.begin() + e);
  return B;
}

// A35: cut_r = argmin_i |P*row_ptr[i] - r*nnz| (ties -> smaller i), non-decreasing.
std::vector<int64_t> row_cuts(const std::vector<int64_t>& rp, int world) {
  if (world < 1) fail(AS_ERR_INVALID_ARG, "world >= 1");
  int64_t m = (int64_t)rp.size() - 1, nnz = rp[m];
  std::vector<int64_t> cuts(world + 1, 0);
  cuts[world] = m;
  for (int r = 1; r < world; ++r) {
    // rp is non-decreasing: the minimiser is next to the first i with P*rp[i] >= r*nnz
    __int128 target = (__int128)r * nnz;
    int64_t lo = 0, hi = m;  // first i with P*rp[i] >= target
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if ((__int128)world * rp[mid] >= target) hi = mid;
      else lo = mid + 1;
    }
    int64_t best = lo;
    auto dist = [&](int64_t i) {
      __int128 d = (__int128)world * rp[i] - target;
      return d < 0 ? -d : d;
    };
    // the first index attaining the minimal distance (ties -> smaller i)
    int64_t i = lo;
    if (i > m) i = m;
    best = i;
    // walk left over equal row_ptr values and the predecessor
    if (i > 0 && dist(i - 1) <= dist(i)) {
      int64_t j = i - 1;
      while (j > 0 && dist(j - 1) <= dist(j)) --j;
      best = j;
    } else {
      while (best > 0 && dist(best - 1) == dist(best)) --best;
    }
    cuts[r] = std::max(best, cuts[r - 1]);
  }
  return cuts;
}

}  // namespace as
