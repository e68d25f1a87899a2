/*
 * wvlt_oracle.c -- CPU restatement of the reference construction algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1702_07578_b200/)
 * links, loads or calls this file.  It is used by tests/ as the parity
 * checker, by __graft_entry__.smoke() as the checker, and by bench.py as the
 * CPU baseline ("port" of the reference's own CPU path).
 *
 * It follows pkg/src/wvlt of the reference line by line in behaviour (not in
 * code): every function cites the reference file:line it restates.  Parity of
 * this restatement is pinned against golden vectors produced by the reference
 * itself (tests/golden/make_golden.py, tests/test_oracle_golden.py).
 *
 * Conventions (reference _kernels.py:8-13): symbols widened to uint64 before
 * shifting, counts/positions int64, bit vector words uint64 LSB-first.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define KIND_WT 0
#define KIND_WM 1
#define SLICE_ALIGNMENT 512 /* construct.py:42 */

static inline uint64_t sym_at(const void* text, int sb, int64_t i) {
  switch (sb) {
    case 1: return ((const uint8_t*)text)[i];
    case 2: return ((const uint16_t*)text)[i];
    case 4: return ((const uint32_t*)text)[i];
    default: return ((const uint64_t*)text)[i];
  }
}

static inline void sym_put(void* out, int sb, int64_t i, uint64_t v) {
  switch (sb) {
    case 1: ((uint8_t*)out)[i] = (uint8_t)v; break;
    case 2: ((uint16_t*)out)[i] = (uint16_t)v; break;
    case 4: ((uint32_t*)out)[i] = (uint32_t)v; break;
    default: ((uint64_t*)out)[i] = v; break;
  }
}

/* bitperm.code_width, bitperm.py:18-22 */
int oracle_code_width(int64_t sigma) {
  if (sigma <= 1) return 0;
  uint64_t v = (uint64_t)(sigma - 1);
  int w = 0;
  while (v) { ++w; v >>= 1; }
  return w;
}

/* bitperm.reverse_bits, bitperm.py:39-47 */
static inline uint64_t rev_bits(uint64_t v, int width) {
  uint64_t r = 0;
  for (int i = 0; i < width; ++i) { r = (r << 1) | (v & 1); v >>= 1; }
  return r;
}

/* _kernels.hist_and_msb_bits, _kernels.py:23-36 */
static void hist_and_msb_bits(const void* text, int sb, int64_t lo, int64_t hi, int64_t* hist, uint64_t* words,
                              int width) {
  const uint64_t msb = (uint64_t)(width - 1);
  for (int64_t i = lo; i < hi; ++i) {
    const uint64_t v = sym_at(text, sb, i);
    hist[v] += 1;
    if ((v >> msb) & 1u) {
      const int64_t j = i - lo;
      words[j >> 6] |= 1ull << (j & 63);
    }
  }
}

/* _kernels.fold_pairs, _kernels.py:45-49 */
static void fold_pairs(int64_t* hist, int64_t m) {
  for (int64_t i = 0; i < m; ++i) hist[i] = hist[2 * i] + hist[2 * i + 1];
}

/* _kernels.starts_identity / starts_ordered, _kernels.py:52-72; the order is
 * the bit-reversal permutation rho_m (bitperm.py:50-62) computed on the fly */
static void starts(const int64_t* hist, int64_t* out, int ell, int wm) {
  const int64_t m = 1ll << ell;
  int64_t run = 0;
  for (int64_t r = 0; r < m; ++r) {
    const int64_t q = wm ? (int64_t)rev_bits((uint64_t)r, ell) : r;
    out[q] = run;
    run += hist[q];
  }
}

/* _kernels.sort_level_pass, _kernels.py:163-176 */
static void sort_level_pass(const void* text, int sb, int64_t n, int prefix_shift, int bit_shift, int64_t* cursors,
                            uint64_t* words) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t v = sym_at(text, sb, i);
    const uint64_t q = prefix_shift >= 64 ? 0 : (v >> prefix_shift);
    const int64_t pos = cursors[q]++;
    if ((v >> bit_shift) & 1u) words[pos >> 6] |= 1ull << (pos & 63);
  }
}

/* construct.build_by_prefix_counting + _sequential_levels(fused=True),
 * construct.py:242-319.  level_words: width * ceil(n/64) words (overwritten),
 * zeros: width entries, hist (optional): 2^width entries of the full histogram. */
int oracle_build_pc(const void* text, int sb, int64_t n, int64_t sigma, int kind, uint64_t* level_words,
                    int64_t* zeros, int64_t* hist_out) {
  const int width = oracle_code_width(sigma);
  const int64_t nwords = (n + 63) >> 6;
  if (width == 0) {
    if (hist_out) hist_out[0] = n;
    return 0;
  }
  memset(level_words, 0, (size_t)width * nwords * 8);
  for (int l = 0; l < width; ++l) zeros[l] = 0;
  const int64_t nb = 1ll << width;
  int64_t* hist = (int64_t*)calloc((size_t)nb, 8);
  int64_t* borders = (int64_t*)malloc((size_t)nb * 8);
  if (!hist || !borders) { free(hist); free(borders); return -1; }
  hist_and_msb_bits(text, sb, 0, n, hist, level_words, width);
  if (hist_out) memcpy(hist_out, hist, (size_t)nb * 8);
  for (int ell = width - 1; ell >= 1; --ell) {
    const int64_t m = 1ll << ell;
    int64_t ev = 0; /* construct._evensum, construct.py:238-239 */
    for (int64_t i = 0; i < 2 * m; i += 2) ev += hist[i];
    zeros[ell] = ev;
    fold_pairs(hist, m);
    starts(hist, borders, ell, kind == KIND_WM);
    sort_level_pass(text, sb, n, width - ell, width - 1 - ell, borders, level_words + (int64_t)ell * nwords);
  }
  /* construct.py:287-288 */
  if (width > 1) {
    zeros[0] = hist[0];
  } else {
    int64_t nnz = 0;
    for (int64_t i = 0; i < n; ++i) nnz += sym_at(text, sb, i) != 0;
    zeros[0] = n - nnz;
  }
  free(hist);
  free(borders);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* ps: construct.build_by_prefix_sorting, construct.py:322-387, with p POSIX
 * threads and a barrier between phases (construct._run_phase, :229-235).     */

typedef struct {
  const void* text;
  int sb;
  int64_t n;
  int width;
  int kind;
  int p;
  int64_t* lo;      /* [p] slice starts (construct._aligned_slices, :199-211) */
  int64_t* hi;      /* [p] */
  int64_t* hists;   /* [p][2^w] */
  int64_t* cursors; /* [p][2^w] */
  void* scratch;    /* n symbols */
  uint64_t* words;
  int64_t nwords;
  int64_t* zeros;
  pthread_barrier_t bar;
} ps_shared;

typedef struct {
  ps_shared* sh;
  int c;
} ps_task;

static void* ps_worker(void* arg) {
  ps_task* t = (ps_task*)arg;
  ps_shared* S = t->sh;
  const int c = t->c, width = S->width;
  const int64_t nb = 1ll << width;
  int64_t* hist = S->hists + (int64_t)c * nb;
  int64_t* cur = S->cursors + (int64_t)c * nb;
  const int64_t lo = S->lo[c], hi = S->hi[c];
  /* phase: per-slice histogram + level-0 bits (construct.py:347-355) */
  if (hi > lo) hist_and_msb_bits(S->text, S->sb, lo, hi, hist, S->words + (lo >> 6), width);
  pthread_barrier_wait(&S->bar);
  for (int ell = width - 1; ell >= 1; --ell) {
    const int64_t m = 1ll << ell;
    if (c == 0 && S->kind == KIND_WM) {
      /* zeros[ell] = hists[:, 0:2m:2].sum(), construct.py:358-359 */
      int64_t ev = 0;
      for (int cc = 0; cc < S->p; ++cc)
        for (int64_t i = 0; i < 2 * m; i += 2) ev += S->hists[(int64_t)cc * nb + i];
      S->zeros[ell] = ev;
    }
    pthread_barrier_wait(&S->bar);
    fold_pairs(hist, m); /* construct.py:360-363 */
    pthread_barrier_wait(&S->bar);
    if (c == 0) {
      /* interleaved_starts_into, levelstats.py:97-137 (sequential form,
       * _kernels.py:75-100): (prefix in order, core) major scan */
      int64_t run = 0;
      for (int64_t r = 0; r < m; ++r) {
        const int64_t q = S->kind == KIND_WM ? (int64_t)rev_bits((uint64_t)r, ell) : r;
        for (int cc = 0; cc < S->p; ++cc) {
          S->cursors[(int64_t)cc * nb + q] = run;
          run += S->hists[(int64_t)cc * nb + q];
        }
      }
    }
    pthread_barrier_wait(&S->bar);
    /* scatter_by_prefix, _kernels.py:146-160 */
    const int shift = width - ell;
    for (int64_t i = lo; i < hi; ++i) {
      const uint64_t v = sym_at(S->text, S->sb, i);
      const uint64_t q = v >> shift;
      const int64_t pos = cur[q]++;
      sym_put(S->scratch, S->sb, pos, v);
    }
    pthread_barrier_wait(&S->bar);
    /* write_bits_from_symbols, _kernels.py:179-193 (slice starts word aligned) */
    uint64_t* lw = S->words + (int64_t)ell * S->nwords + (lo >> 6);
    const int bsh = width - 1 - ell;
    for (int64_t i = lo; i < hi; i += 64) {
      const int64_t end = (i + 64 < hi) ? i + 64 : hi;
      uint64_t acc = 0;
      for (int64_t j = i; j < end; ++j) acc |= ((sym_at(S->scratch, S->sb, j) >> bsh) & 1u) << (j - i);
      lw[(i - lo) >> 6] = acc;
    }
    pthread_barrier_wait(&S->bar);
  }
  return NULL;
}

int oracle_build_ps(const void* text, int sb, int64_t n, int64_t sigma, int kind, int threads, uint64_t* level_words,
                    int64_t* zeros) {
  const int width = oracle_code_width(sigma);
  const int64_t nwords = (n + 63) >> 6;
  if (width == 0) return 0;
  if (threads < 1) return -2;
  memset(level_words, 0, (size_t)width * nwords * 8);
  const int p = threads;
  const int64_t nb = 1ll << width;
  ps_shared S;
  memset(&S, 0, sizeof(S));
  S.text = text; S.sb = sb; S.n = n; S.width = width; S.kind = kind; S.p = p;
  S.lo = (int64_t*)malloc(sizeof(int64_t) * p);
  S.hi = (int64_t*)malloc(sizeof(int64_t) * p);
  S.hists = (int64_t*)calloc((size_t)p * nb, 8);
  S.cursors = (int64_t*)malloc((size_t)p * nb * 8);
  S.scratch = malloc((size_t)(n ? n : 1) * (size_t)sb);
  S.words = level_words;
  S.nwords = nwords;
  S.zeros = zeros;
  for (int l = 0; l < width; ++l) zeros[l] = 0;
  if (!S.lo || !S.hi || !S.hists || !S.cursors || !S.scratch) return -1;
  {
    /* construct._aligned_slices, construct.py:199-211 */
    const int64_t per = (n + p - 1) / p;
    const int64_t chunk = (per + SLICE_ALIGNMENT - 1) / SLICE_ALIGNMENT * SLICE_ALIGNMENT;
    for (int c = 0; c < p; ++c) {
      int64_t lo = c * chunk;
      if (lo > n) lo = n;
      int64_t hi = lo + chunk;
      if (hi > n) hi = n;
      if (c == p - 1) hi = n;
      S.lo[c] = lo;
      S.hi[c] = hi;
    }
  }
  pthread_barrier_init(&S.bar, NULL, (unsigned)p);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * p);
  ps_task* tasks = (ps_task*)malloc(sizeof(ps_task) * p);
  for (int c = 0; c < p; ++c) {
    tasks[c].sh = &S;
    tasks[c].c = c;
    pthread_create(&th[c], NULL, ps_worker, &tasks[c]);
  }
  for (int c = 0; c < p; ++c) pthread_join(th[c], NULL);
  pthread_barrier_destroy(&S.bar);
  /* construct.py:384-385 */
  if (kind == KIND_WM) {
    if (width > 1) {
      int64_t z0 = 0;
      for (int c = 0; c < p; ++c) z0 += S.hists[(int64_t)c * nb];
      zeros[0] = z0;
    } else {
      int64_t nnz = 0;
      for (int64_t i = 0; i < n; ++i) nnz += sym_at(text, sb, i) != 0;
      zeros[0] = n - nnz;
    }
  }
  free(th);
  free(tasks);
  free(S.lo);
  free(S.hi);
  free(S.hists);
  free(S.cursors);
  free(S.scratch);
  return 0;
}

/* Full histogram padded to 2^width: levelstats.symbol_histogram, levelstats.py:30-47 */
int oracle_histogram(const void* text, int sb, int64_t n, int64_t sigma, int64_t* hist) {
  const int width = oracle_code_width(sigma);
  memset(hist, 0, ((size_t)1 << width) * 8);
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t v = sym_at(text, sb, i);
    if (v >= (uint64_t)sigma) return -4;
    hist[v] += 1;
  }
  return 0;
}

/* Node borders for levels 1..width-1 at [2^l - 2, 2^(l+1) - 2): WT numeric
 * order (levelstats.interval_starts, levelstats.py:58-73), WM bit-reversed
 * order (wt2wm.interval_start_table, wt2wm.py:55-78). */
int oracle_borders(const int64_t* hist_in, int width, int kind, int64_t* out) {
  if (width < 2) return 0;
  const int64_t nb = 1ll << width;
  int64_t* h = (int64_t*)malloc((size_t)nb * 8);
  if (!h) return -1;
  memcpy(h, hist_in, (size_t)nb * 8);
  for (int ell = width - 1; ell >= 1; --ell) {
    const int64_t m = 1ll << ell;
    fold_pairs(h, m);
    starts(h, out + (m - 2), ell, kind == KIND_WM);
  }
  free(h);
  return 0;
}

/* _kernels.gather_bits, _kernels.py:196-232 */
void oracle_merge_bits(uint64_t* dst, int64_t word_lo, int64_t word_hi, int64_t n_bits, const int64_t* bounds,
                       const int64_t* src_starts, const uint64_t* src, int64_t t0) {
  int64_t t = t0;
  for (int64_t wd = word_lo; wd < word_hi; ++wd) {
    const int64_t base = wd << 6;
    int64_t nbits = n_bits - base;
    if (nbits > 64) nbits = 64;
    uint64_t acc = 0;
    int64_t filled = 0;
    while (filled < nbits) {
      const int64_t here = base + filled;
      while (bounds[t + 1] <= here) ++t;
      int64_t take = nbits - filled;
      const int64_t avail = bounds[t + 1] - here;
      if (avail < take) take = avail;
      const int64_t sp = src_starts[t] + (here - bounds[t]);
      const int64_t wi = sp >> 6;
      const int sh = (int)(sp & 63);
      uint64_t chunk = src[wi] >> sh;
      if (sh + take > 64) chunk |= src[wi + 1] << (64 - sh);
      if (take < 64) chunk &= (1ull << take) - 1ull;
      acc |= chunk << filled;
      filled += take;
    }
    dst[wd] = acc;
  }
}

/* ------------------------------------------------------------------------
 * construct.build_domain_decomposed (construct.py:437-513) with its
 * _merge_plan (construct.py:516-543): p aligned slices (construct.py:199-211)
 * each built independently by the inner algorithm (pc, or ps on one thread),
 * the partial levels concatenated at the slices' word offsets, then every
 * level merged by gather_bits over p destination word ranges
 * (construct.py:214-217), one thread each.  inner: 0 = pc, 1 = ps.
 * ------------------------------------------------------------------------ */
typedef struct {
  const void* text;
  int sb, kind, inner, width;
  int64_t sigma, lo, hi;
  uint64_t* partial; /* width rows of nwords */
  int64_t nwords;
  int64_t* hist;     /* 2^width */
  int rc;
} dd_slice;

static void* dd_slice_worker(void* arg) {
  dd_slice* t = (dd_slice*)arg;
  const int64_t m = t->hi - t->lo;
  const int64_t mw = (m + 63) >> 6;
  const void* piece = (const char*)t->text + (size_t)t->lo * t->sb;
  uint64_t* w = (uint64_t*)calloc((size_t)(t->width * mw) + 1, 8);
  int64_t* z = (int64_t*)calloc((size_t)t->width + 1, 8);
  if (!w || !z) { t->rc = -1; free(w); free(z); return NULL; }
  t->rc = t->inner == 0 ? oracle_build_pc(piece, t->sb, m, t->sigma, t->kind, w, z, t->hist)
                        : oracle_build_ps(piece, t->sb, m, t->sigma, t->kind, 1, w, z);
  if (!t->rc && t->inner != 0) t->rc = oracle_histogram(piece, t->sb, m, t->sigma, t->hist);
  for (int l = 0; l < t->width && !t->rc; ++l)
    memcpy(t->partial + (int64_t)l * t->nwords + (t->lo >> 6), w + (int64_t)l * mw, (size_t)mw * 8);
  free(w);
  free(z);
  return NULL;
}

typedef struct {
  uint64_t* dst;
  const uint64_t* src;
  const int64_t* bounds;
  const int64_t* src_starts;
  int64_t ntasks, w0, w1, n;
} dd_merge;

static void* dd_merge_worker(void* arg) {
  dd_merge* t = (dd_merge*)arg;
  if (t->w1 <= t->w0) return NULL;
  /* t0 = searchsorted(bounds, 64 w0, side="right") - 1 (construct.py:503) */
  int64_t lo = 0, hi = t->ntasks;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (t->bounds[mid] <= 64 * t->w0) lo = mid;
    else hi = mid;
  }
  oracle_merge_bits(t->dst, t->w0, t->w1, t->n, t->bounds, t->src_starts, t->src, lo);
  return NULL;
}

int oracle_build_dd(const void* text, int sb, int64_t n, int64_t sigma, int kind, int threads, int inner,
                    uint64_t* level_words, int64_t* zeros) {
  const int width = oracle_code_width(sigma);
  const int64_t nwords = (n + 63) >> 6;
  if (threads < 1) return -2;
  if (width == 0) return 0;
  memset(level_words, 0, (size_t)width * nwords * 8);
  for (int l = 0; l < width; ++l) zeros[l] = 0;
  if (n == 0) return 0; /* construct.py:457-458 */
  const int p = threads;
  const int64_t nb = 1ll << width;
  uint64_t* partial = (uint64_t*)calloc((size_t)width * nwords + 1, 8);
  int64_t* hists = (int64_t*)calloc((size_t)p * nb, 8);
  dd_slice* sl = (dd_slice*)calloc((size_t)p, sizeof(dd_slice));
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * p);
  if (!partial || !hists || !sl || !th) return -1;
  const int64_t per = (n + p - 1) / p;
  const int64_t chunk = (per + SLICE_ALIGNMENT - 1) / SLICE_ALIGNMENT * SLICE_ALIGNMENT;
  int nact = 0;
  for (int c = 0; c < p; ++c) {
    int64_t lo = c * chunk;
    if (lo > n) lo = n;
    int64_t hi = lo + chunk;
    if (hi > n || c == p - 1) hi = n;
    if (hi <= lo) continue;
    dd_slice* t = &sl[nact++];
    t->text = text; t->sb = sb; t->kind = kind; t->inner = inner; t->width = width; t->sigma = sigma;
    t->lo = lo; t->hi = hi; t->partial = partial; t->nwords = nwords; t->hist = hists + (int64_t)(nact - 1) * nb;
  }
  for (int c = 0; c < nact; ++c) pthread_create(&th[c], NULL, dd_slice_worker, &sl[c]);
  for (int c = 0; c < nact; ++c) pthread_join(th[c], NULL);
  int rc = 0;
  for (int c = 0; c < nact; ++c) rc = rc ? rc : sl[c].rc;
  /* per-slice count chains: level l counts at chain[c][l] (fold of the histogram) */
  int64_t* chain = (int64_t*)malloc((size_t)nact * (2 * nb) * 8); /* level l at offset 2^l - 1 */
  int64_t* lens = (int64_t*)malloc((size_t)nact * nb * 8 + 8);
  int64_t* src = (int64_t*)malloc((size_t)nact * nb * 8 + 8);
  int64_t* bounds = (int64_t*)malloc(((size_t)nact * nb + 1) * 8);
  dd_merge* mt = (dd_merge*)malloc(sizeof(dd_merge) * p);
  if (!chain || !lens || !src || !bounds || !mt) rc = -1;
  for (int c = 0; c < nact && !rc; ++c) {
    int64_t* ch = chain + (int64_t)c * 2 * nb;
    memcpy(ch + nb - 1, sl[c].hist, (size_t)nb * 8);
    for (int l = width - 1; l >= 0; --l)
      for (int64_t q = 0; q < (1ll << l); ++q)
        ch[(1ll << l) - 1 + q] = ch[(2ll << l) - 1 + 2 * q] + ch[(2ll << l) - 1 + 2 * q + 1];
  }
  /* WM zero counts: sum over slices of the even (l+1)-prefix counts (construct.py:486-488) */
  if (kind == KIND_WM && !rc)
    for (int l = 0; l < width; ++l)
      for (int c = 0; c < nact; ++c) {
        const int64_t* cl = chain + (int64_t)c * 2 * nb + (2ll << l) - 1;
        for (int64_t q = 0; q < (1ll << l); ++q) zeros[l] += cl[2 * q];
      }
  for (int l = width - 1; l >= 0 && !rc; --l) {
    /* _merge_plan: prefixes in interval order, slices in text order inside */
    int64_t k = 0;
    const int64_t m = 1ll << l;
    for (int64_t r = 0; r < m; ++r) {
      const int64_t q = (kind == KIND_WM && l >= 2) ? (int64_t)rev_bits((uint64_t)r, l) : r;
      for (int c = 0; c < nact; ++c) {
        const int64_t* cl = chain + (int64_t)c * 2 * nb + (1ll << l) - 1;
        const int64_t len = l == 0 ? sl[c].hi - sl[c].lo : cl[q];
        if (len > 0) { lens[k] = len; src[k] = c; bounds[k] = q; ++k; }
      }
    }
    /* local starts: per slice a running sum over the interval order */
    int64_t* run = (int64_t*)calloc((size_t)nact, 8);
    int64_t acc = 0;
    for (int64_t t = 0; t < k; ++t) {
      const int c = (int)src[t];
      const int64_t s0 = sl[c].lo + run[c];
      run[c] += lens[t];
      src[t] = s0;
      bounds[t] = acc;
      acc += lens[t];
    }
    bounds[k] = acc;
    free(run);
    const uint64_t* srcw = partial + (int64_t)l * nwords;
    uint64_t* dstw = level_words + (int64_t)l * nwords;
    for (int c = 0; c < p; ++c) {
      mt[c].dst = dstw; mt[c].src = srcw; mt[c].bounds = bounds; mt[c].src_starts = src; mt[c].ntasks = k;
      mt[c].w0 = nwords * c / p; mt[c].w1 = nwords * (c + 1) / p; mt[c].n = n;
      pthread_create(&th[c], NULL, dd_merge_worker, &mt[c]);
    }
    for (int c = 0; c < p; ++c) pthread_join(th[c], NULL);
  }
  free(chain); free(lens); free(src); free(bounds); free(mt); free(partial); free(hists); free(sl); free(th);
  return rc;
}
