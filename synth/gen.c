/* Seeded synthetic matrix generators for the large BASELINE configs (C3, C4, C5).
 *
 * Input generation only: no SpMV and no format building.  Shared by the CUDA-path tests,
 * the oracle tests and bench.py through synth/__init__.py.  Randomness is Philox4x32-10
 * keyed by (seed, stream) with the element / draw index as the counter, so results do not
 * depend on the thread count.  Output is CSR (row_ptr int64[m+1], col int32[nnz]) with
 * strictly ascending columns in every row; values are drawn afterwards from the entry index.
 *
 * Recipes:
 *   C3 R-MAT (a,b,c,d), labels permuted, self loops and duplicates dropped, first
 *      occurrences in draw order kept until nnz - n off-diagonal entries, diagonal added.
 *   C4 n_tiles dense b x b tiles (distinct tile rows, uniform tile column) + diagonal +
 *      uniform scattered entries outside tiles and diagonal, deduplicated, topped up in
 *      rounds until exactly nnz.
 *   C5 row lengths 0.9*U{4..16} + 0.1*U{17..123}, capped by the band window, adjusted by
 *      +-1 along an affine permutation of the rows until the sum is nnz; each row = the
 *      diagonal + distinct uniform columns in [i-band, i+band] (rejection sampling).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ Philox4x32-10 */
static inline void philox(uint64_t seed, uint32_t stream, uint64_t ctr_lo, uint32_t ctr_hi, uint32_t out[4]) {
  uint32_t c0 = (uint32_t)ctr_lo, c1 = (uint32_t)(ctr_lo >> 32), c2 = ctr_hi, c3 = stream;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32) ^ 0x5bd1e995u;
  for (int i = 0; i < 10; ++i) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}
static inline uint32_t rnd32(uint64_t seed, uint32_t stream, uint64_t i, uint32_t sub) {
  uint32_t o[4];
  philox(seed, stream, i, sub >> 2, o);
  return o[sub & 3];
}
static inline uint64_t rnd_below(uint64_t seed, uint32_t stream, uint64_t i, uint32_t sub, uint64_t n) {
  uint32_t o[4];
  philox(seed, stream, i, sub, o);
  uint64_t v = ((uint64_t)o[0] << 32) | o[1];
  return n ? v % n : 0;
}

/* ------------------------------------------------------------------ threading */
typedef struct { void (*fn)(void*, int64_t, int64_t); void* ctx; int64_t a, e; } task_t;
static void* task_run(void* p) { task_t* t = (task_t*)p; t->fn(t->ctx, t->a, t->e); return NULL; }
static void par(int nth, int64_t n, void (*fn)(void*, int64_t, int64_t), void* ctx) {
  if (nth < 1) nth = 1;
  if (nth > 256) nth = 256;
  if (n < 4096) nth = 1;
  pthread_t th[256];
  task_t t[256];
  for (int i = 0; i < nth; ++i) {
    t[i] = (task_t){fn, ctx, n * i / nth, n * (i + 1) / nth};
    if (i) pthread_create(&th[i], NULL, task_run, &t[i]);
  }
  task_run(&t[0]);
  for (int i = 1; i < nth; ++i) pthread_join(th[i], NULL);
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : x > y;
}
typedef struct { uint64_t key, idx; } kv_t;
static int cmp_kv(const void* a, const void* b) {
  const kv_t *x = (const kv_t*)a, *y = (const kv_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : x->idx > y->idx;
}

/* Sort kv pairs by (key, idx) with a parallel bucket sort over the key range [0, kmax). */
typedef struct { kv_t* dst; int64_t* off; } bs_t;
static void bs_sort_buckets(void* p, int64_t a, int64_t e) {
  bs_t* s = (bs_t*)p;
  for (int64_t b = a; b < e; ++b) qsort(s->dst + s->off[b], (size_t)(s->off[b + 1] - s->off[b]), sizeof(kv_t), cmp_kv);
}
static inline int64_t bucket_of(uint64_t key, uint64_t width, int nb) {
  uint64_t b = key / width;
  return b >= (uint64_t)nb ? nb - 1 : (int64_t)b;
}
/* keys are expected in [0, kmax) except sentinels (UINT64_MAX), which land in the last bucket */
static void sort_kv(kv_t* v, int64_t n, uint64_t kmax, int nth) {
  if (n <= 1) return;
  int nb = nth * 16;
  if (nb > 4096) nb = 4096;
  int64_t* cnt = (int64_t*)calloc((size_t)nb + 1, sizeof(int64_t));
  uint64_t width = kmax / (uint64_t)nb + 1;
  for (int64_t i = 0; i < n; ++i) cnt[bucket_of(v[i].key, width, nb) + 1]++;
  for (int b = 0; b < nb; ++b) cnt[b + 1] += cnt[b];
  kv_t* tmp = (kv_t*)malloc((size_t)n * sizeof(kv_t));
  int64_t* pos = (int64_t*)malloc((size_t)nb * sizeof(int64_t));
  memcpy(pos, cnt, (size_t)nb * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) tmp[pos[bucket_of(v[i].key, width, nb)]++] = v[i];
  bs_t s = {tmp, cnt};
  par(nth, nb, bs_sort_buckets, &s);
  memcpy(v, tmp, (size_t)n * sizeof(kv_t));
  free(tmp);
  free(pos);
  free(cnt);
}

/* ------------------------------------------------------------------ values */
typedef struct { uint64_t seed; int int_mode; int f32; void* val; int64_t i0; } val_t;
static void fill_vals(void* p, int64_t a, int64_t e) {
  val_t* s = (val_t*)p;
  for (int64_t k = a; k < e; ++k) {
    const int64_t i = s->i0 + k; /* global nonzero index: the Philox counter */
    double v;
    if (s->int_mode) {
      uint32_t u = rnd32(s->seed, 3, (uint64_t)i, 0);
      int mag = 1 + (int)(u % 4u);
      v = ((u >> 8) & 1) ? -mag : mag;
    } else {
      uint32_t o[4];
      philox(s->seed, 4, (uint64_t)i, 0, o);
      uint64_t bits = ((uint64_t)(o[0] >> 5) << 26) | (o[1] >> 6);
      v = (double)bits * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
    }
    if (s->f32) ((float*)s->val)[k] = (float)v;
    else ((double*)s->val)[k] = v;
  }
}
/* values for nnz entries: U[-1,1) (real) or {-4..4}\{0} (int_mode); f32 selects float */
int synth_values(uint64_t seed, int64_t nnz, int int_mode, int f32, void* val, int nth) {
  val_t s = {seed, int_mode, f32, val, 0};
  par(nth, nnz, fill_vals, &s);
  return 0;
}
/* values of the nonzeros [i0, i0 + n) only (a rank's ROW_DIV band): identical to the
 * corresponding slice of synth_values */
int synth_values_range(uint64_t seed, int64_t i0, int64_t n, int int_mode, int f32, void* val, int nth) {
  val_t s = {seed, int_mode, f32, val, i0};
  par(nth, n, fill_vals, &s);
  return 0;
}

/* ------------------------------------------------------------------ C5 band-irregular */
typedef struct { int64_t m, band; uint64_t seed; int64_t* L; const int64_t* rp; int32_t* col; int64_t r0; } c5_t;
static void c5_len(void* p, int64_t a, int64_t e) {
  c5_t* s = (c5_t*)p;
  for (int64_t i = a; i < e; ++i) {
    uint32_t o[4];
    philox(s->seed, 0, (uint64_t)i, 0, o);
    int64_t L = (o[0] < 3865470566u) ? 4 + (int64_t)(o[1] % 13u) : 17 + (int64_t)(o[1] % 107u); /* 0.9*2^32 */
    int64_t lo = i - s->band < 0 ? 0 : i - s->band, hi = i + s->band > s->m - 1 ? s->m - 1 : i + s->band;
    int64_t cap = hi - lo + 1;
    s->L[i] = L < cap ? L : cap;
  }
}
static void c5_cols(void* p, int64_t a, int64_t e) {
  c5_t* s = (c5_t*)p;
  int32_t buf[4096];
  for (int64_t i = s->r0 + a; i < s->r0 + e; ++i) {
    int64_t lo = i - s->band < 0 ? 0 : i - s->band, hi = i + s->band > s->m - 1 ? s->m - 1 : i + s->band;
    int64_t width = hi - lo; /* window without the diagonal */
    int64_t need = s->rp[i + 1] - s->rp[i] - 1, got = 0;
    uint32_t sub = 0;
    buf[got++] = (int32_t)i;
    while (got < need + 1) {
      int64_t c = lo + (int64_t)(rnd_below(s->seed, 10, (uint64_t)i, sub++, (uint64_t)width));
      if (c >= i) ++c;
      int dup = 0;
      for (int64_t k = 0; k < got; ++k)
        if (buf[k] == c) { dup = 1; break; }
      if (!dup) buf[got++] = (int32_t)c;
    }
    qsort(buf, (size_t)got, sizeof(int32_t), cmp_i32);
    memcpy(s->col + (s->rp[i] - s->rp[s->r0]), buf, (size_t)got * sizeof(int32_t));
  }
}
static int64_t gcd64(int64_t a, int64_t b) { while (b) { int64_t t = a % b; a = b; b = t; } return a; }

/* row lengths of C5 (drawn per row, then the seeded round-robin +-1 adjustment to nnz):
 * row_ptr[m+1] (out) */
int synth_c5_rowptr(int64_t m, int64_t nnz, int64_t band, uint64_t seed, int64_t* row_ptr, int nth) {
  int64_t* L = (int64_t*)malloc((size_t)m * sizeof(int64_t));
  c5_t s = {m, band, seed, L, row_ptr, NULL, 0};
  par(nth, m, c5_len, &s);
  int64_t tot = 0;
  for (int64_t i = 0; i < m; ++i) tot += L[i];
  int64_t diff = nnz - tot;
  int64_t a = (int64_t)(rnd_below(seed, 2, 0, 0, (uint64_t)m) | 1), b = (int64_t)rnd_below(seed, 2, 1, 0, (uint64_t)m);
  while (gcd64(a, m) != 1) a += 2;
  int64_t k = 0, stall = 0;
  while (diff != 0 && stall < 2 * m) {
    int64_t i = (int64_t)(((__int128)a * k + b) % m);
    ++k;
    int64_t lo = i - band < 0 ? 0 : i - band, hi = i + band > m - 1 ? m - 1 : i + band;
    if (diff > 0 && L[i] < hi - lo + 1) { L[i]++; diff--; stall = 0; }
    else if (diff < 0 && L[i] > 1) { L[i]--; diff++; stall = 0; }
    else stall++;
  }
  if (diff != 0) { free(L); return -1; }
  row_ptr[0] = 0;
  for (int64_t i = 0; i < m; ++i) row_ptr[i + 1] = row_ptr[i] + L[i];
  free(L);
  return 0;
}
/* columns of rows [r0, r1) given the full row_ptr: col[row_ptr[r1] - row_ptr[r0]] (out).
 * Per-row counter-based draws, so a band equals the same rows of the whole matrix. */
int synth_c5_band(int64_t m, int64_t band, uint64_t seed, const int64_t* row_ptr, int64_t r0, int64_t r1,
                  int32_t* col, int nth) {
  c5_t s = {m, band, seed, NULL, row_ptr, col, r0};
  par(nth, r1 - r0, c5_cols, &s);
  return 0;
}
/* rows m, total nnz, band half-width; row_ptr[m+1] (out), col[nnz] (out) */
int synth_c5(int64_t m, int64_t nnz, int64_t band, uint64_t seed, int64_t* row_ptr, int32_t* col, int nth) {
  if (synth_c5_rowptr(m, nnz, band, seed, row_ptr, nth)) return -1;
  return synth_c5_band(m, band, seed, row_ptr, 0, m, col, nth);
}

/* ------------------------------------------------------------------ C4 block-dense */
typedef struct {
  int64_t m, b, nt; uint64_t seed; const int32_t* tile_of; /* tile col per tile row, -1 if none */
  kv_t* kv; int64_t d0; const int64_t* srp; const kv_t* skv; int64_t* rp; int32_t* col; int count_only;
} c4_t;
static void c4_draw(void* p, int64_t a, int64_t e) {
  c4_t* s = (c4_t*)p;
  for (int64_t i = a; i < e; ++i) {
    uint64_t d = (uint64_t)(s->d0 + i);
    for (uint32_t sub = 0;; ++sub) { /* rejection: redraw on tile / diagonal hits */
      uint32_t o[4];
      philox(s->seed, 5, d, sub, o);
      int64_t r = (int64_t)((((uint64_t)o[0] << 32) | o[1]) % (uint64_t)s->m);
      int64_t c = (int64_t)((((uint64_t)o[2] << 32) | o[3]) % (uint64_t)s->m);
      int32_t J = s->tile_of[r / s->b];
      if (c == r || (J >= 0 && c / s->b == J)) continue;
      s->kv[i].key = (uint64_t)r * (uint64_t)s->m + (uint64_t)c;
      s->kv[i].idx = d;
      break;
    }
  }
}
static void c4_rows(void* p, int64_t a, int64_t e) {
  c4_t* s = (c4_t*)p;
  int32_t buf[8192];
  for (int64_t r = a; r < e; ++r) {
    int64_t n = 0;
    int32_t J = s->tile_of[r / s->b];
    int diag_in_tile = J >= 0 && r / s->b == J;
    if (J >= 0)
      for (int64_t j = 0; j < s->b; ++j) buf[n++] = (int32_t)(J * s->b + j);
    if (!diag_in_tile) buf[n++] = (int32_t)r;
    for (int64_t k = s->srp[r]; k < s->srp[r + 1]; ++k) buf[n++] = (int32_t)(s->skv[k].key % (uint64_t)s->m);
    if (s->count_only) { s->rp[r + 1] = n; continue; }
    qsort(buf, (size_t)n, sizeof(int32_t), cmp_i32);
    memcpy(s->col + s->rp[r], buf, (size_t)n * sizeof(int32_t));
  }
}
/* tiles_out[2*n_tiles] = (I, J) sorted; row_ptr[m+1]; col[nnz] */
int synth_c4(int64_t m, int64_t b, int64_t n_tiles, int64_t nnz, uint64_t seed, int64_t* tiles_out,
             int64_t* row_ptr, int32_t* col, int nth) {
  int64_t nt = m / b;
  int32_t* perm = (int32_t*)malloc((size_t)nt * sizeof(int32_t));
  for (int64_t i = 0; i < nt; ++i) perm[i] = (int32_t)i;
  for (int64_t i = 0; i < n_tiles; ++i) { /* partial Fisher-Yates */
    int64_t j = i + (int64_t)rnd_below(seed, 0, (uint64_t)i, 0, (uint64_t)(nt - i));
    int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  qsort(perm, (size_t)n_tiles, sizeof(int32_t), cmp_i32);
  int32_t* tile_of = (int32_t*)malloc((size_t)nt * sizeof(int32_t));
  for (int64_t i = 0; i < nt; ++i) tile_of[i] = -1;
  int64_t base = m;
  for (int64_t t = 0; t < n_tiles; ++t) {
    int64_t I = perm[t], J = (int64_t)rnd_below(seed, 1, (uint64_t)t, 0, (uint64_t)nt);
    tile_of[I] = (int32_t)J;
    tiles_out[2 * t] = I;
    tiles_out[2 * t + 1] = J;
    base += b * b - (I == J ? b : 0);
  }
  free(perm);
  int64_t need = nnz - base;
  if (need < 0) { free(tile_of); return -1; }
  kv_t* kv = (kv_t*)malloc((size_t)(need + 16) * sizeof(kv_t));
  int64_t have = 0, drawn = 0;
  c4_t s = {m, b, nt, seed, tile_of, NULL, 0, NULL, NULL, row_ptr, col, 0};
  while (have < need) { /* draw exactly the deficit, dedup (keep first draw), repeat */
    int64_t deficit = need - have;
    s.kv = kv + have;
    s.d0 = drawn;
    par(nth, deficit, c4_draw, &s);
    drawn += deficit;
    have += deficit;
    sort_kv(kv, have, (uint64_t)m * (uint64_t)m, nth);
    int64_t w = 0;
    for (int64_t i = 0; i < have; ++i)
      if (i == 0 || kv[i].key != kv[w - 1].key) kv[w++] = kv[i];
    have = w;
  }
  /* scatter row pointers */
  int64_t* srp = (int64_t*)calloc((size_t)m + 1, sizeof(int64_t));
  for (int64_t i = 0; i < have; ++i) srp[kv[i].key / (uint64_t)m + 1]++;
  for (int64_t r = 0; r < m; ++r) srp[r + 1] += srp[r];
  s.srp = srp;
  s.skv = kv;
  s.count_only = 1;
  row_ptr[0] = 0;
  par(nth, m, c4_rows, &s);
  for (int64_t r = 0; r < m; ++r) row_ptr[r + 1] += row_ptr[r];
  s.count_only = 0;
  par(nth, m, c4_rows, &s);
  free(srp);
  free(kv);
  free(tile_of);
  return row_ptr[m] == nnz ? 0 : -2;
}

/* ------------------------------------------------------------------ C3 R-MAT */
typedef struct { int scale; uint64_t seed; const int32_t* perm; kv_t* kv; int64_t d0; uint32_t ta, tab, tabc; } c3_t;
static void c3_draw(void* p, int64_t a, int64_t e) {
  c3_t* s = (c3_t*)p;
  for (int64_t i = a; i < e; ++i) {
    uint64_t d = (uint64_t)(s->d0 + i);
    uint64_t r = 0, c = 0;
    for (int l = 0; l < s->scale; l += 4) {
      uint32_t o[4];
      philox(s->seed, 6, d, (uint32_t)(l >> 2), o);
      for (int q = 0; q < 4 && l + q < s->scale; ++q) {
        uint32_t u = o[q];
        uint64_t rb = u >= s->tab, cb = (u >= s->ta && u < s->tab) || u >= s->tabc;
        r = (r << 1) | rb;
        c = (c << 1) | cb;
      }
    }
    r = (uint64_t)s->perm[r];
    c = (uint64_t)s->perm[c];
    s->kv[i].key = r == c ? UINT64_MAX : (r << s->scale) | c;
    s->kv[i].idx = d;
  }
}
/* k-th smallest (0-based) of distinct values, in place (Hoare quickselect, median of 3) */
static uint64_t select_kth(uint64_t* a, int64_t n, int64_t k) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    uint64_t x = a[lo], y = a[(lo + hi) / 2], z = a[hi];
    uint64_t piv = x < y ? (y < z ? y : (x < z ? z : x)) : (x < z ? x : (y < z ? z : y));
    int64_t i = lo, j = hi;
    while (i <= j) {
      while (a[i] < piv) ++i;
      while (a[j] > piv) --j;
      if (i <= j) { uint64_t t = a[i]; a[i] = a[j]; a[j] = t; ++i; --j; }
    }
    if (k <= j) hi = j;
    else if (k >= i) lo = i;
    else return a[k];
  }
  return a[k];
}
/* n = 2^scale rows, nnz total (incl. diagonal); a, b, c in [0,1) (d = 1-a-b-c) */
int synth_c3(int scale, int64_t nnz, double pa, double pb, double pc, uint64_t seed, int64_t* row_ptr, int32_t* col,
             int nth) {
  int64_t n = (int64_t)1 << scale;
  int32_t* perm = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
  for (int64_t i = n - 1; i > 0; --i) {
    int64_t j = (int64_t)rnd_below(seed, 7, (uint64_t)i, 0, (uint64_t)(i + 1));
    int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  int64_t target = nnz - n;
  int64_t cap = target + target / 3 + (1 << 20);
  kv_t* kv = (kv_t*)malloc((size_t)cap * sizeof(kv_t));
  c3_t s = {scale, seed, perm, NULL, 0, (uint32_t)(pa * 4294967296.0), (uint32_t)((pa + pb) * 4294967296.0),
            (uint32_t)((pa + pb + pc) * 4294967296.0)};
  int64_t have = 0, drawn = 0;
  while (have < target) {
    int64_t batch = (target - have) + (target - have) / 4 + 1024;
    if (have + batch > cap) {
      cap = have + batch;
      kv = (kv_t*)realloc(kv, (size_t)cap * sizeof(kv_t));
    }
    s.kv = kv + have;
    s.d0 = drawn;
    par(nth, batch, c3_draw, &s);
    drawn += batch;
    have += batch;
    sort_kv(kv, have, (uint64_t)n << scale, nth);  /* by key, then draw index */
    int64_t w = 0;
    for (int64_t i = 0; i < have; ++i) {
      if (kv[i].key == UINT64_MAX) break; /* self loops sort last */
      if (w == 0 || kv[i].key != kv[w - 1].key) kv[w++] = kv[i];
    }
    have = w;
  }
  if (have > target) { /* keep the first `target` distinct edges in draw order */
    uint64_t* ix = (uint64_t*)malloc((size_t)have * sizeof(uint64_t));
    for (int64_t i = 0; i < have; ++i) ix[i] = kv[i].idx;
    uint64_t thr = select_kth(ix, have, target - 1); /* target-th smallest draw index */
    free(ix);
    int64_t w = 0;
    for (int64_t i = 0; i < have; ++i)
      if (kv[i].idx <= thr) kv[w++] = kv[i];
    have = w;
  }
  /* CSR with the diagonal */
  memset(row_ptr, 0, (size_t)(n + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < have; ++i) row_ptr[(kv[i].key >> scale) + 1]++;
  for (int64_t r = 0; r < n; ++r) row_ptr[r + 1] += row_ptr[r] + 1;
  int64_t k = 0;
  for (int64_t r = 0; r < n; ++r) {
    int64_t o = row_ptr[r];
    int diag_done = 0;
    while (k < have && (int64_t)(kv[k].key >> scale) == r) {
      int64_t c = (int64_t)(kv[k].key & (uint64_t)(n - 1));
      if (!diag_done && c > r) { col[o++] = (int32_t)r; diag_done = 1; }
      col[o++] = (int32_t)c;
      ++k;
    }
    if (!diag_done) col[o++] = (int32_t)r;
  }
  free(kv);
  free(perm);
  return row_ptr[n] == nnz ? 0 : -2;
}
