// wvlt_b200.cu -- sm_100a wavelet tree / wavelet matrix construction.
//
// The reference builds every level with a counting-sort pass over the text
// (pkg/src/wvlt/construct.py:242-387, kernels in pkg/src/wvlt/_kernels.py).
// This file re-designs that hot path for B200:
//
//   K1  symbol histogram + range check, one read of the text
//       (replaces hist_and_msb_bits / full_histogram, _kernels.py:23-42)
//   K2  one small kernel deriving every table from that histogram: the fold
//       chain (fold_pairs, _kernels.py:45-49), per-level zero counts
//       (construct.py:238-239,273-288), node borders (starts_identity /
//       starts_ordered, _kernels.py:52-72) and the per-pass placement tables
//   K3  fused level pass: K levels per read of the current symbol order.  A
//       tile of the order is staged in shared memory, split stably by one bit
//       per level (the wavelet-matrix refinement, structures.py:176-182),
//       every level's bits are taken with __ballot_sync in the tile-local
//       order, tile offsets come from one single-pass decoupled look-back over
//       the 2^K digit counts, and the bits are emitted as aligned 64-bit words
//       (replaces sort_level_pass / scatter_by_prefix / write_bits_from_symbols,
//       _kernels.py:146-193).  The order after K levels is written back to HBM
//       narrowed to the bits still live.
//   K5  bit-interval shift-merge (replaces gather_bits, _kernels.py:196-232).
//
// Position algebra (derivation in DESIGN.md §3).  Let A_l be the level-l
// order, b_i(v) the i-th code bit of v (MSB first) and, for a pass starting at
// level l, d_j(v) = sum_{i<j} b_{l+i}(v) << i (an LSD digit).  Then
//   WM: A_{l+j} = stable sort of A_l by d_j, so
//       pos_{l+j}(x) = G_j[d] + C_j[d](x)
//   WT: A_{l+j} = stable sort of A_l by the (l+j)-bit prefix P, and
//       pos_{l+j}(x) = corr_j[P] + C_j[d](x)
// where C_j[d](x) counts symbols of A_l before x with digit d (tile look-back
// prefix + rank inside the tile), G_j is the exclusive scan of the global
// digit counts and corr_j[P] = wtstart_{l+j}[P] - sum_{q'<q} cnt_{l+j}[q'2^j+e]
// for P = q 2^j + e.  Both tables come from the histogram alone (K2).

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "wvlt_b200.h"

namespace {

constexpr int KMAX = 4;             // levels fused per pass
constexpr int NDIG = 1 << KMAX;     // digit bins per pass
constexpr int PASS_THREADS = 512;
constexpr int MAXP = 32;            // passes per build (width <= 24 => <= 6 at K = 4)
constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ unsigned rev_bits(unsigned d, int j) {  // j >= 1
  return __brev(d) >> (32 - j);
}

// look-back status word: [63:62] state (1 aggregate, 2 inclusive), [61:42] epoch, [41:0] value
constexpr uint64_t ST_VALUE_MASK = (1ull << 42) - 1;
__device__ __forceinline__ uint64_t pack_status(unsigned state, unsigned epoch, uint64_t v) {
  return ((uint64_t)state << 62) | ((uint64_t)(epoch & 0xFFFFFu) << 42) | (v & ST_VALUE_MASK);
}
__device__ __forceinline__ unsigned status_state(uint64_t s, unsigned epoch) {
  return (((s >> 42) & 0xFFFFFu) == (epoch & 0xFFFFFu)) ? (unsigned)(s >> 62) : 0u;
}

// ---------------------------------------------------------------------------
// K1: histogram.  Byte texts with width <= 8 use a bit-sliced counter: per
// 32-symbol warp chunk, one ballot per code bit, and lane b counts bins
// b + 32i as popc of the AND of the matching ballots (no shared-memory
// atomics, no contention on Zipf heavy hitters).
// ---------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(256) hist_u8_kernel(const uint8_t* __restrict__ text, int64_t n,
                                                      unsigned long long* __restrict__ hist,
                                                      int32_t* __restrict__ status) {
  constexpr int NB = 1 << W;
  constexpr int PER = (NB + 31) / 32;
  constexpr int LOWB = W < 5 ? W : 5;
  __shared__ unsigned s_hist[NB];
  for (int i = threadIdx.x; i < NB; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();

  const int lane = threadIdx.x & 31;
  unsigned sel[LOWB];
#pragma unroll
  for (int k = 0; k < LOWB; ++k) sel[k] = ((lane >> k) & 1) ? 0u : FULL;
  unsigned cnt[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) cnt[i] = 0;
  unsigned bad = 0;

  const int64_t nvec = (n + 15) >> 4;
  const bool aligned = (((uintptr_t)text) & 15) == 0;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t wv = gwarp * 32; wv < nvec; wv += nwarps * 32) {
    const int64_t vi = wv + lane;
    const int64_t first = vi * 16;
    uint32_t word[4] = {0, 0, 0, 0};
    int nvalid = 0;
    if (vi < nvec) {
      nvalid = (int)min((int64_t)16, n - first);
      if (aligned && nvalid == 16) {
        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(text) + vi);
        word[0] = q.x; word[1] = q.y; word[2] = q.z; word[3] = q.w;
      } else {
        for (int e = 0; e < nvalid; ++e) word[e >> 2] |= (uint32_t)text[first + e] << (8 * (e & 3));
      }
    }
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
      if (W < 8) bad |= word[wd] & (((0xFFu << W) & 0xFFu) * 0x01010101u);
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const unsigned byte = (word[e >> 2] >> (8 * (e & 3))) & 0xFFu;
      const unsigned V = __ballot_sync(FULL, e < nvalid);
      unsigned B[W];
#pragma unroll
      for (int k = 0; k < W; ++k) B[k] = __ballot_sync(FULL, (byte >> k) & 1u);
      unsigned low = V;
#pragma unroll
      for (int k = 0; k < LOWB; ++k) low &= B[k] ^ sel[k];
      if (W <= 5) {
        cnt[0] += __popc(low);
      } else {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          unsigned m = low;
#pragma unroll
          for (int k = 5; k < W; ++k) m &= ((i >> (k - 5)) & 1) ? B[k] : ~B[k];
          cnt[i] += __popc(m);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int bin = lane + 32 * i;
    if (bin < NB && cnt[i]) atomicAdd(&s_hist[bin], cnt[i]);
  }
  if (bad) atomicOr(status, WVLT_STATUS_RANGE);
  __syncthreads();
  for (int i = threadIdx.x; i < NB; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&hist[i], (unsigned long long)s_hist[i]);
}

// Generic histogram for wide symbols / wide alphabets: shared-memory bins when
// 2^w fits, else warp-aggregated global atomics (Zipf heavy hitters collapse
// to one atomic per warp via __match_any_sync).
template <typename TIn, bool SMEM>
__global__ void __launch_bounds__(256) hist_generic_kernel(const TIn* __restrict__ text, int64_t n, int w,
                                                           unsigned long long* __restrict__ hist,
                                                           int32_t* __restrict__ status) {
  extern __shared__ unsigned s_bins[];
  const int64_t nb = 1ll << w;
  if (SMEM) {
    for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) s_bins[i] = 0;
    __syncthreads();
  }
  unsigned bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t start = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nround = (n + stride - 1) / stride;
  for (int64_t r = 0; r < nround; ++r) {  // warp-uniform trip count for __match_any_sync
    const int64_t i = start + r * stride;
    const bool valid = i < n;
    uint32_t v = valid ? (uint32_t)__ldcs(text + i) : 0u;
    const bool ok = valid && (w >= 32 || (v >> w) == 0);
    if (valid && !ok) bad = 1;
    if (SMEM) {
      if (ok) atomicAdd(&s_bins[v], 1u);
    } else {
      const unsigned act = __ballot_sync(FULL, ok);
      if (ok) {
        const unsigned peers = __match_any_sync(act, v);
        if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1) && hist)
          atomicAdd(&hist[v], (unsigned long long)__popc(peers));
      }
    }
  }
  if (bad) atomicOr(status, WVLT_STATUS_RANGE);
  if (SMEM && hist) {
    __syncthreads();
    for (int64_t i = threadIdx.x; i < nb; i += blockDim.x)
      if (s_bins[i]) atomicAdd(&hist[i], (unsigned long long)s_bins[i]);
  }
}

__global__ void fill_i64_kernel(int64_t* p, int64_t v) { *p = v; }

// ---------------------------------------------------------------------------
// Build plan shared by host and the tables kernel
// ---------------------------------------------------------------------------
struct Plan {
  int width;
  int kind;
  int npass;
  int lvl[MAXP];        // first level of the pass
  int K[MAXP];          // levels in the pass
  int in_bytes[MAXP];   // element bytes of A_lvl
  int out_bytes[MAXP];  // element bytes of A_{lvl+K} (0 = no output)
  int tile[MAXP];       // symbols per tile
  int64_t ntiles[MAXP];
  int64_t corr_off[MAXP][KMAX + 1];  // WT placement tables (int64 offsets into corr)
  int64_t corr_total;
  // workspace carve (byte offsets)
  size_t off_chain, off_wtstart, off_wmbase, off_corr, off_counter, off_status, off_buf0, off_buf1;
  size_t status_bytes, buf_bytes, total;
};

__host__ __device__ inline int64_t chain_off(int k) { return (1ll << k) - 1; }  // level-k table in a 2^(w+1)-1 array

// ---------------------------------------------------------------------------
// K2: tables.  One CTA; everything here is O(2^width) and tiny next to the
// O(n width) passes.
// ---------------------------------------------------------------------------
constexpr int TAB_THREADS = 1024;
constexpr int TAB_ITEMS = 8;

struct TablesArgs {
  Plan plan;
  int64_t sigma;
  int64_t n;
  const unsigned long long* hist_in;  // == chain level w (int64 view)
  int64_t* chain;
  int64_t* wtstart;
  int64_t* wm_base;  // [MAXP][KMAX+1][NDIG]
  int64_t* corr;
  uint32_t* counters;
  int64_t* zeros_out;    // may be null
  int64_t* hist_out;     // may be null
  int64_t* borders_out;  // may be null
  int32_t* status;
};

__device__ int64_t block_sum_i64(int64_t v, int64_t* s_red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) s_red[wid] = v;
  __syncthreads();
  int64_t t = 0;
  if (wid == 0) {
    t = (lane < (int)(blockDim.x >> 5)) ? s_red[lane] : 0;
    t = warp_sum(t);
    if (lane == 0) s_red[32] = t;
  }
  __syncthreads();
  return s_red[32];
}

// Exclusive scan of get(i), i < count, written through put(i, value).
template <typename Get, typename Put>
__device__ void block_scan_excl(int64_t count, Get get, Put put, int64_t* s_red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t carry = 0;
  const int64_t per_iter = (int64_t)blockDim.x * TAB_ITEMS;
  for (int64_t base = 0; base < count; base += per_iter) {
    const int64_t i0 = base + (int64_t)threadIdx.x * TAB_ITEMS;
    int64_t loc[TAB_ITEMS];
    int64_t tsum = 0;
#pragma unroll
    for (int k = 0; k < TAB_ITEMS; ++k) {
      loc[k] = (i0 + k < count) ? get(i0 + k) : 0;
      tsum += loc[k];
    }
    int64_t incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    __syncthreads();
    if (lane == 31) s_red[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const int64_t v = lane < nw ? s_red[lane] : 0;
      int64_t s = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(FULL, s, o);
        if (lane >= o) s += t;
      }
      s_red[lane] = s - v;
      if (lane == 31) s_red[32] = s;
    }
    __syncthreads();
    int64_t run = carry + s_red[wid] + incl - tsum;
#pragma unroll
    for (int k = 0; k < TAB_ITEMS; ++k) {
      if (i0 + k < count) put(i0 + k, run);
      run += loc[k];
    }
    carry += s_red[32];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(TAB_THREADS) tables_kernel(const TablesArgs a) {
  __shared__ int64_t s_red[33];
  __shared__ unsigned long long s_dig[NDIG];
  const Plan& P = a.plan;
  const int w = P.width;
  const int tid = threadIdx.x;
  const int64_t nb = 1ll << w;

  // counters for the passes' dynamic tile ids
  if (tid < MAXP) a.counters[tid] = 0;

  // 1. chain level w = histogram; range check of bins at or above sigma
  int64_t* cw = a.chain + chain_off(w);
  for (int64_t v = tid; v < nb; v += blockDim.x) {
    const int64_t h = (int64_t)a.hist_in[v];
    if (v >= a.sigma && h) atomicOr(a.status, WVLT_STATUS_RANGE);
    if (a.hist_out) a.hist_out[v] = h;
  }
  __syncthreads();
  // 2. fold chain (fold_pairs, _kernels.py:45-49)
  for (int k = w - 1; k >= 0; --k) {
    const int64_t* up = a.chain + chain_off(k + 1);
    int64_t* dn = a.chain + chain_off(k);
    for (int64_t q = tid; q < (1ll << k); q += blockDim.x) dn[q] = up[2 * q] + up[2 * q + 1];
    __syncthreads();
  }
  // 3. zero counts Z[l] = sum of even (l+1)-prefix counts (construct.py:238-239)
  for (int l = 0; l < w; ++l) {
    const int64_t* c = a.chain + chain_off(l + 1);
    int64_t s = 0;
    for (int64_t q = tid; q < (1ll << l); q += blockDim.x) s += c[2 * q];
    s = block_sum_i64(s, s_red);
    if (tid == 0 && a.zeros_out) a.zeros_out[l] = s;
  }
  // 4. node borders: WT in numeric prefix order, WM in bit-reversed order
  for (int k = 0; k <= w; ++k) {
    const int64_t* c = a.chain + chain_off(k);
    int64_t* ws = a.wtstart + chain_off(k);
    block_scan_excl(
        1ll << k, [&](int64_t i) { return c[i]; }, [&](int64_t i, int64_t v) { ws[i] = v; }, s_red);
    if (a.borders_out && k >= 1 && k < w) {
      int64_t* out = a.borders_out + ((1ll << k) - 2);
      if (P.kind == WVLT_KIND_WT) {
        for (int64_t i = tid; i < (1ll << k); i += blockDim.x) out[i] = ws[i];
        __syncthreads();
      } else {
        block_scan_excl(
            1ll << k, [&](int64_t r) { return c[rev_bits((unsigned)r, k)]; },
            [&](int64_t r, int64_t v) { out[rev_bits((unsigned)r, k)] = v; }, s_red);
      }
    }
  }
  // 5. per-pass placement tables
  for (int p = 0; p < P.npass; ++p) {
    const int l = P.lvl[p], K = P.K[p];
    if (P.kind == WVLT_KIND_WM) {
      // global counts of the K-bit LSD digit of bits l..l+K-1
      if (tid < NDIG) s_dig[tid] = 0;
      __syncthreads();
      const int64_t* c = a.chain + chain_off(l + K);
      const int64_t tot = 1ll << (l + K);
      const int nd = 1 << K;
      int64_t acc[NDIG];
#pragma unroll
      for (int d = 0; d < NDIG; ++d) acc[d] = 0;
      for (int64_t i = tid; i < tot; i += blockDim.x) {
        const unsigned e = (unsigned)(i & (nd - 1));  // numeric digit (MSB first)
        const unsigned d = rev_bits(e, K);
#pragma unroll
        for (int dd = 0; dd < NDIG; ++dd)
          if (dd == (int)d) acc[dd] += c[i];
      }
#pragma unroll
      for (int d = 0; d < NDIG; ++d) {
        const int64_t s = warp_sum(acc[d]);
        if ((tid & 31) == 0 && s) atomicAdd(&s_dig[d], (unsigned long long)s);
      }
      __syncthreads();
      if (tid == 0) {
        int64_t* g = a.wm_base + (int64_t)p * (KMAX + 1) * NDIG;
        for (int j = 1; j <= K; ++j) {
          const int mj = 1 << j;
          int64_t run = 0;
          for (int d = 0; d < mj; ++d) {
            int64_t cj = 0;
            for (int e = d; e < nd; e += mj) cj += (int64_t)s_dig[e];
            g[j * NDIG + d] = run;
            run += cj;
          }
        }
      }
      __syncthreads();
    } else {
      for (int j = 1; j <= K; ++j) {
        if (j == K && P.out_bytes[p] == 0) break;
        const int64_t* c = a.chain + chain_off(l + j);
        const int64_t* ws = a.wtstart + chain_off(l + j);
        int64_t* corr = a.corr + P.corr_off[p][j];
        const int mj = 1 << j;
        const int64_t rows = 1ll << l;
        // column-wise exclusive scans over the node index q
        for (int e = 0; e < mj; ++e) {
          block_scan_excl(
              rows, [&](int64_t q) { return c[q * mj + e]; },
              [&](int64_t q, int64_t v) { corr[q * mj + e] = ws[q * mj + e] - v; }, s_red);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K3: fused level pass
// ---------------------------------------------------------------------------
struct PassArgs {
  const void* src;
  void* dst;
  uint64_t* words;  // level words base (level L at words + L * nwords)
  int64_t nwords;
  int64_t n;
  int level, width, kind, has_out;
  uint64_t* status;
  uint32_t* counter;
  unsigned epoch;
  const int64_t* wm_base;  // this pass: [KMAX+1][NDIG]
  const int64_t* corr;     // WT tables of this pass: table j at corr + corr_off[j]
  int64_t corr_off[KMAX + 1];
};

template <typename TIn, int K, int E>
struct PassSmem {
  static constexpr int T = PASS_THREADS * E;
  static constexpr int NC = T / 32;
  static constexpr size_t buf_bytes = (size_t)(K + 1) * T * sizeof(TIn);
  static constexpr size_t bits_bytes = (size_t)K * (NC + 2) * 4;
  static constexpr size_t scan_bytes = (size_t)(NC + 1) * 4;
  static constexpr size_t total = buf_bytes + bits_bytes + scan_bytes;
};

__device__ __forceinline__ uint64_t extract_bits(const uint32_t* L, int off, int cnt) {
  const int i = off >> 5, s = off & 31;
  uint64_t v = ((uint64_t)L[i] | ((uint64_t)L[i + 1] << 32)) >> s;
  if (s) v |= (uint64_t)L[i + 2] << (64 - s);
  return cnt >= 64 ? v : (v & ((1ull << cnt) - 1));
}

// Copy runs of the tile-local bit string L to the level's global words:
// run r = local bits [ls[r], ls[r]+len[r]) -> global bits [gs[r], gs[r]+len[r]).
// Whole destination words are stored, words shared with another run are OR-ed
// into the pre-zeroed level (the "owner writes whole words" rule of
// gather_bits, _kernels.py:197-205, relaxed to atomics at run edges).
__device__ void emit_runs(const uint32_t* L, int R, const int* ls, const int* len, const int64_t* gs,
                          uint64_t* gw, int* s_wpre) {
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int r = 0; r < R; ++r) {
      s_wpre[r] = acc;
      if (len[r]) acc += (int)(((gs[r] + len[r] - 1) >> 6) - (gs[r] >> 6) + 1);
    }
    s_wpre[R] = acc;
  }
  __syncthreads();
  const int total = s_wpre[R];
  for (int f = threadIdx.x; f < total; f += blockDim.x) {
    int r = 0;
    while (s_wpre[r + 1] <= f) ++r;
    const int64_t g = gs[r];
    const int64_t W = (g >> 6) + (f - s_wpre[r]);
    const int64_t wb = W << 6;
    const int64_t a0 = g > wb ? g : wb;
    const int64_t e = g + len[r];
    const int64_t b0 = e < wb + 64 ? e : wb + 64;
    const int c = (int)(b0 - a0);
    const int lo = (int)(a0 - wb);
    const uint64_t v = extract_bits(L, ls[r] + (int)(a0 - g), c) << lo;
    if (c == 64)
      gw[W] = v;
    else
      atomicOr(reinterpret_cast<unsigned long long*>(gw + W), (unsigned long long)v);
  }
  __syncthreads();
}

template <typename TIn>
__device__ __forceinline__ unsigned digit_of(TIn x, int top_shift, int j) {
  // d_j = sum_{i<j} bit(top_shift - i) << i
  unsigned d = 0;
  for (int i = 0; i < j; ++i) d |= (((uint32_t)x >> (top_shift - i)) & 1u) << i;
  return d;
}

template <typename TIn, typename TOut, int K, int E>
__global__ void __launch_bounds__(PASS_THREADS) level_pass_kernel(const PassArgs a) {
  using S = PassSmem<TIn, K, E>;
  constexpr int T = S::T;
  constexpr int NC = S::NC;
  constexpr int NW = PASS_THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  TIn* buf = reinterpret_cast<TIn*>(smem);
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + S::buf_bytes);
  uint32_t* scan = reinterpret_cast<uint32_t*>(smem + S::buf_bytes + S::bits_bytes);

  __shared__ int s_cnt[K + 1][NDIG];
  __shared__ int s_ls[K + 1][NDIG];
  __shared__ int64_t s_lb[K + 1][NDIG];
  __shared__ int64_t s_gs[NDIG];
  __shared__ int s_wpre[NDIG + 1];
  __shared__ uint32_t s_wtot[NW + 1];
  __shared__ int s_tile;
  __shared__ int s_q1;
  __shared__ int64_t s_q;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int w = a.width, l0 = a.level;

  if (tid == 0) s_tile = (int)atomicAdd(a.counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * T;
  const int cnt = (int)min((int64_t)T, a.n - base);
  const TIn* src = reinterpret_cast<const TIn*>(a.src) + base;

  // ---- stage the tile (invalid tail slots = all ones so they sort last) ----
  if (cnt == T && ((((uintptr_t)src) & 15) == 0)) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(buf);
    for (int i = tid; i < (int)(T * sizeof(TIn) / 16); i += PASS_THREADS) d4[i] = __ldcs(s4 + i);
  } else {
    for (int p = tid; p < T; p += PASS_THREADS) buf[p] = p < cnt ? src[p] : (TIn)~(TIn)0;
  }
  if (tid == 0) {
    s_cnt[0][0] = cnt;
    s_ls[0][0] = 0;
  }
  __syncthreads();

  // WT: does the tile lie inside one level-l0 node?
  if (a.kind == WVLT_KIND_WT && tid == 0) {
    const int sh = w - l0;
    const uint64_t qf = sh >= 32 ? 0 : ((uint64_t)(uint32_t)buf[0] >> sh);
    const uint64_t ql = sh >= 32 ? 0 : ((uint64_t)(uint32_t)buf[cnt - 1] >> sh);
    s_q1 = qf == ql;
    s_q = (int64_t)qf;
  }

  // ---- K stable one-bit splits in shared memory ----
  TIn x[E];
  uint32_t m[E];
#pragma unroll 1
  for (int j = 0; j < K; ++j) {
    const TIn* cur = buf + (size_t)j * T;
    uint32_t* bj = bits + j * (NC + 2);
    const int sh = w - 1 - l0 - j;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int p = e * PASS_THREADS + tid;
      x[e] = cur[p];
      m[e] = __ballot_sync(FULL, ((uint32_t)x[e] >> sh) & 1u);
      if (lane == 0) {
        bj[p >> 5] = m[e];
        scan[p >> 5] = __popc(m[e]);
      }
    }
    if (tid < 2) bj[NC + tid] = 0;
    __syncthreads();
    // exclusive scan of the chunk popcounts (NC <= PASS_THREADS)
    {
      const uint32_t v = tid < NC ? scan[tid] : 0u;
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) s_wtot[wid] = incl;
      __syncthreads();
      if (wid == 0) {
        const uint32_t t = lane < NW ? s_wtot[lane] : 0u;
        uint32_t s = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t u = __shfl_up_sync(FULL, s, o);
          if (lane >= o) s += u;
        }
        if (lane < NW) s_wtot[lane] = s - t;
        if (lane == NW - 1) s_wtot[NW] = s;
      }
      __syncthreads();
      if (tid < NC) scan[tid] = incl - v + s_wtot[wid];
      if (tid == 0) scan[NC] = s_wtot[NW];
      __syncthreads();
    }
    // group sizes of the next digit: split each d_j group by this bit
    if (tid < (1 << j)) {
      const int d = tid;
      const int gs0 = s_ls[j][d], c0 = s_cnt[j][d];
      auto rank1 = [&](int p) -> int {
        const int c = p >> 5, r = p & 31;
        return (int)scan[c] + (r ? __popc(bj[c] & ((1u << r) - 1u)) : 0);
      };
      const int ones = rank1(gs0 + c0) - rank1(gs0);
      s_cnt[j + 1][d] = c0 - ones;
      s_cnt[j + 1][d + (1 << j)] = ones;
    }
    // scatter into the next order
    if (j + 1 < K || a.has_out) {
      const int Z = T - (int)scan[NC];
      TIn* nxt = buf + (size_t)(j + 1) * T;
      const unsigned lt = lanemask_lt();
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int p = e * PASS_THREADS + tid;
        const int r1 = (int)scan[p >> 5] + __popc(m[e] & lt);
        const int dst = ((m[e] >> lane) & 1u) ? Z + r1 : p - r1;
        nxt[dst] = x[e];
      }
    }
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int d = 0; d < (2 << j); ++d) {
        s_ls[j + 1][d] = run;
        run += s_cnt[j + 1][d];
      }
    }
    // level l0 bits are already in global order: aligned word stores
    if (j == 0) {
      uint32_t* g32 = reinterpret_cast<uint32_t*>(a.words + (int64_t)l0 * a.nwords);
      const int64_t lim = 2 * a.nwords;
      for (int c = tid; c < NC; c += PASS_THREADS) {
        const int64_t gi = (base >> 5) + c;
        if (gi < lim) {
          const int first = c * 32;
          uint32_t v = bj[c];
          if (first + 32 > cnt) v = first >= cnt ? 0u : (v & ((1u << (cnt - first)) - 1u));
          g32[gi] = v;
        }
      }
    }
    __syncthreads();
  }

  // ---- decoupled look-back over the 2^K digit counts ----
  const int nd = 1 << K;
  if (wid == 0) {
    uint64_t* st = a.status + tile * NDIG;
    if (lane < nd) st_relaxed_u64(st + lane, pack_status(tile == 0 ? 2u : 1u, a.epoch, (uint64_t)s_cnt[K][lane]));
    int64_t acc = 0;
    if (tile > 0) {
      unsigned pending = (1u << nd) - 1u;
      int64_t wb = tile - 1;
      while (pending) {
        const int64_t tt = wb - lane;
#pragma unroll 1
        for (int d = 0; d < nd; ++d) {
          if (!((pending >> d) & 1u)) continue;
          uint64_t s;
          unsigned state;
          if (tt < 0) {
            s = 0;
            state = 2;
          } else {
            s = ld_relaxed_u64(a.status + tt * NDIG + d);
            state = status_state(s, a.epoch);
            while (state == 0) {
              __nanosleep(64);
              s = ld_relaxed_u64(a.status + tt * NDIG + d);
              state = status_state(s, a.epoch);
            }
          }
          const unsigned im = __ballot_sync(FULL, state == 2u);
          const int k = im ? __ffs(im) - 1 : 31;
          uint64_t v = (lane <= k) ? (s & ST_VALUE_MASK) : 0ull;
          v = warp_sum(v);
          if (lane == d) acc += (int64_t)v;
          if (im) pending &= ~(1u << d);
        }
        wb -= 32;
      }
      if (lane < nd) st_relaxed_u64(st + lane, pack_status(2u, a.epoch, (uint64_t)(acc + s_cnt[K][lane])));
    }
    if (lane < nd) s_lb[K][lane] = acc;
  }
  __syncthreads();
  // fold the digit prefixes to every shorter digit
  if (tid < NDIG) {
    for (int j = 1; j < K; ++j) {
      if (tid < (1 << j)) {
        int64_t s = 0;
        for (int e = tid; e < nd; e += (1 << j)) s += s_lb[K][e];
        s_lb[j][tid] = s;
      }
    }
  }
  __syncthreads();

  const bool wm = a.kind == WVLT_KIND_WM;
  const bool uniform = wm || s_q1;  // placement is a per-digit constant in this tile

  // ---- emit levels l0+1 .. l0+K-1 ----
#pragma unroll 1
  for (int j = 1; j < K; ++j) {
    const int mj = 1 << j;
    uint64_t* gw = a.words + (int64_t)(l0 + j) * a.nwords;
    const uint32_t* L = bits + j * (NC + 2);
    if (uniform) {
      if (tid < mj) {
        const int d = tid;
        const int64_t tb =
            wm ? a.wm_base[j * NDIG + d]
               : a.corr[a.corr_off[j] + (s_q << j) + (int64_t)rev_bits((unsigned)d, j)];
        s_gs[d] = tb + s_lb[j][d];
      }
      __syncthreads();
      emit_runs(L, mj, s_ls[j], s_cnt[j], s_gs, gw, s_wpre);
    } else {
      // WT tile spanning several nodes: per-symbol placement, runs found by
      // contiguity of the global position inside each warp chunk
      const TIn* cur = buf + (size_t)j * T;
      const int tshift = w - 1 - l0;
      const int pshift = w - l0 - j;
      const int64_t* ctab = a.corr + a.corr_off[j];
#pragma unroll 1
      for (int e = 0; e < E; ++e) {
        const int p = e * PASS_THREADS + tid;
        const bool valid = p < cnt;
        const TIn xv = cur[p];
        int64_t gpos = 0;
        unsigned bit = 0;
        if (valid) {
          const unsigned d = digit_of(xv, tshift, j);
          const uint64_t P = pshift >= 32 ? 0 : ((uint64_t)(uint32_t)xv >> pshift);
          gpos = ctab[P] + s_lb[j][d] + p - s_ls[j][d];
          bit = ((uint32_t)xv >> (tshift - j)) & 1u;
        }
        const int64_t key = gpos - p;
        const int64_t pkey = __shfl_up_sync(FULL, key, 1);
        const bool leader = valid && (lane == 0 || pkey != key);
        const unsigned Lm = __ballot_sync(FULL, leader);
        const unsigned Bm = __ballot_sync(FULL, bit);
        const unsigned Vm = __ballot_sync(FULL, valid);
        if (leader) {
          const unsigned rest = Lm & ~((2u << lane) - 1u);
          const int next = rest ? __ffs(rest) - 1 : __popc(Vm);
          const int len = next - lane;
          uint64_t seg = (uint64_t)(Bm >> lane);
          if (len < 32) seg &= (1ull << len) - 1ull;
          const int64_t W = gpos >> 6;
          const int o = (int)(gpos & 63);
          if (seg) {
            atomicOr(reinterpret_cast<unsigned long long*>(gw + W), (unsigned long long)(seg << o));
            if (o + len > 64)
              atomicOr(reinterpret_cast<unsigned long long*>(gw + W + 1), (unsigned long long)(seg >> (64 - o)));
          }
        }
      }
      __syncthreads();
    }
  }

  // ---- write A_{l0+K}, narrowed to the bits still needed ----
  if (a.has_out) {
    const TIn* fin = buf + (size_t)K * T;
    TOut* dst = reinterpret_cast<TOut*>(a.dst);
    const uint32_t keep = wm ? ((w - l0 - K) >= 32 ? FULL : ((1u << (w - l0 - K)) - 1u)) : FULL;
    if (uniform) {
      if (tid < nd) {
        const int d = tid;
        const int64_t tb = wm ? a.wm_base[K * NDIG + d]
                              : a.corr[a.corr_off[K] + (s_q << K) + (int64_t)rev_bits((unsigned)d, K)];
        s_gs[d] = tb + s_lb[K][d] - s_ls[K][d];
      }
      __syncthreads();
      // group d occupies [ls_K[d], ls_K[d+1]) of the final order; find it by a
      // short search (<= 16 groups), then one coalesced store per symbol
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int p = e * PASS_THREADS + tid;
        if (p < cnt) {
          int d = 0;
          while (d + 1 < nd && s_ls[K][d + 1] <= p) ++d;
          dst[s_gs[d] + p] = (TOut)((uint32_t)fin[p] & keep);
        }
      }
    } else {
      const int tshift = w - 1 - l0;
      const int pshift = w - l0 - K;
      const int64_t* ctab = a.corr + a.corr_off[K];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int p = e * PASS_THREADS + tid;
        if (p < cnt) {
          const TIn xv = fin[p];
          const unsigned d = digit_of(xv, tshift, K);
          const uint64_t P = pshift >= 32 ? 0 : ((uint64_t)(uint32_t)xv >> pshift);
          dst[ctab[P] + s_lb[K][d] + p - s_ls[K][d]] = (TOut)((uint32_t)xv & keep);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K5: merge (gather_bits)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) merge_bits_kernel(uint64_t* __restrict__ dst, int64_t wlo, int64_t whi,
                                                         int64_t nbits, const int64_t* __restrict__ bounds,
                                                         const int64_t* __restrict__ src_starts, int64_t ntasks,
                                                         const uint64_t* __restrict__ src) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t wd = wlo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; wd < whi; wd += stride) {
    const int64_t wb = wd << 6;
    int64_t nb = nbits - wb;
    if (nb > 64) nb = 64;
    uint64_t acc = 0;
    if (nb > 0) {
      // task containing bit wb: last t with bounds[t] <= wb
      int64_t lo = 0, hi = ntasks;  // answer in [0, ntasks)
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (bounds[mid] <= wb) lo = mid; else hi = mid;
      }
      int64_t t = lo;
      int filled = 0;
      while (filled < nb) {
        const int64_t here = wb + filled;
        while (bounds[t + 1] <= here) ++t;
        int64_t take = nb - filled;
        const int64_t avail = bounds[t + 1] - here;
        if (avail < take) take = avail;
        const int64_t sp = src_starts[t] + (here - bounds[t]);
        const int64_t wi = sp >> 6;
        const int sh = (int)(sp & 63);
        uint64_t chunk = src[wi] >> sh;
        if (sh + take > 64) chunk |= src[wi + 1] << (64 - sh);
        if (take < 64) chunk &= (1ull << take) - 1ull;
        acc |= chunk << filled;
        filled += (int)take;
      }
    }
    dst[wd] = acc;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int code_width_host(int64_t sigma) {
  if (sigma <= 1) return 0;
  uint64_t v = (uint64_t)(sigma - 1);
  int w = 0;
  while (v) {
    ++w;
    v >>= 1;
  }
  return w;
}

int bytes_for_bits(int bits) { return bits <= 8 ? 1 : (bits <= 16 ? 2 : 4); }

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int tile_for(int in_bytes) { return in_bytes == 4 ? PASS_THREADS * 8 : PASS_THREADS * 16; }

bool make_plan(int64_t n, int sym_bytes, int64_t sigma, int kind, Plan* P) {
  memset(P, 0, sizeof(*P));
  const int w = code_width_host(sigma);
  P->width = w;
  P->kind = kind;
  if (w > WVLT_MAX_WIDTH) return false;
  const int vbits = sym_bytes * 8;  // symbols never need more bits than their storage
  int l = 0, p = 0;
  int64_t corr = 0;
  int64_t max_tiles = 0;
  size_t max_buf = 0;
  while (l < w) {
    const int K = (w - l) < KMAX ? (w - l) : KMAX;
    P->lvl[p] = l;
    P->K[p] = K;
    const int live_in = kind == WVLT_KIND_WM ? (w - l) : w;
    const int live_out = kind == WVLT_KIND_WM ? (w - l - K) : w;
    P->in_bytes[p] = p == 0 ? sym_bytes : bytes_for_bits(live_in < vbits ? live_in : vbits);
    P->out_bytes[p] = (l + K < w) ? bytes_for_bits(live_out < vbits ? live_out : vbits) : 0;
    if (P->out_bytes[p] > P->in_bytes[p]) P->out_bytes[p] = P->in_bytes[p];
    P->tile[p] = tile_for(P->in_bytes[p]);
    P->ntiles[p] = (n + P->tile[p] - 1) / P->tile[p];
    if (P->ntiles[p] > max_tiles) max_tiles = P->ntiles[p];
    if ((size_t)P->out_bytes[p] * (size_t)n > max_buf) max_buf = (size_t)P->out_bytes[p] * (size_t)n;
    if (kind == WVLT_KIND_WT) {
      for (int j = 1; j <= K; ++j) {
        P->corr_off[p][j] = corr;
        corr += 1ll << (l + j);
      }
    }
    l += K;
    ++p;
  }
  P->npass = p;
  P->corr_total = corr;
  size_t off = 0;
  const size_t chain_bytes = ((size_t)2 << w) * 8;
  P->off_chain = off;
  off = align_up(off + chain_bytes, 256);
  P->off_wtstart = off;
  off = align_up(off + chain_bytes, 256);
  P->off_wmbase = off;
  off = align_up(off + (size_t)MAXP * (KMAX + 1) * NDIG * 8, 256);
  P->off_corr = off;
  off = align_up(off + (size_t)(corr ? corr : 1) * 8, 256);
  P->off_counter = off;  // MAXP pass counters + one scratch status word
  off = align_up(off + (MAXP + 1) * 4, 256);
  P->off_status = off;
  P->status_bytes = (size_t)(max_tiles ? max_tiles : 1) * NDIG * 8;
  off = align_up(off + P->status_bytes, 256);
  P->buf_bytes = align_up(max_buf ? max_buf : 16, 256);
  P->off_buf0 = off;
  off += P->buf_bytes;
  P->off_buf1 = off;
  off += P->buf_bytes;
  P->total = off;
  return true;
}

template <typename TIn, typename TOut, int K>
cudaError_t launch_pass_t(const PassArgs& a, int64_t ntiles, cudaStream_t s) {
  constexpr int E = sizeof(TIn) == 4 ? 8 : 16;
  using S = PassSmem<TIn, K, E>;
  auto kern = level_pass_kernel<TIn, TOut, K, E>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::total);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<(unsigned)ntiles, PASS_THREADS, S::total, s>>>(a);
  return cudaGetLastError();
}

template <typename TIn, typename TOut>
cudaError_t launch_pass_k(int K, const PassArgs& a, int64_t ntiles, cudaStream_t s) {
  switch (K) {
    case 1: return launch_pass_t<TIn, TOut, 1>(a, ntiles, s);
    case 2: return launch_pass_t<TIn, TOut, 2>(a, ntiles, s);
    case 3: return launch_pass_t<TIn, TOut, 3>(a, ntiles, s);
    default: return launch_pass_t<TIn, TOut, 4>(a, ntiles, s);
  }
}

cudaError_t launch_pass(int in_bytes, int out_bytes, int K, const PassArgs& a, int64_t ntiles, cudaStream_t s) {
  const int ob = out_bytes ? out_bytes : in_bytes;
  if (in_bytes == 1) return launch_pass_k<uint8_t, uint8_t>(K, a, ntiles, s);
  if (in_bytes == 2) {
    if (ob == 1) return launch_pass_k<uint16_t, uint8_t>(K, a, ntiles, s);
    return launch_pass_k<uint16_t, uint16_t>(K, a, ntiles, s);
  }
  if (ob == 1) return launch_pass_k<uint32_t, uint8_t>(K, a, ntiles, s);
  if (ob == 2) return launch_pass_k<uint32_t, uint16_t>(K, a, ntiles, s);
  return launch_pass_k<uint32_t, uint32_t>(K, a, ntiles, s);
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

cudaError_t launch_hist(const void* text, int sym_bytes, int64_t n, int w, unsigned long long* hist,
                        int32_t* status, cudaStream_t s) {
  const int blocks = sm_count() * 4;
  if (sym_bytes == 1 && w <= 8 && w >= 1) {
    const uint8_t* t = (const uint8_t*)text;
    switch (w) {
      case 1: hist_u8_kernel<1><<<blocks, 256, 0, s>>>(t, n, hist, status); break;
      case 2: hist_u8_kernel<2><<<blocks, 256, 0, s>>>(t, n, hist, status); break;
      case 3: hist_u8_kernel<3><<<blocks, 256, 0, s>>>(t, n, hist, status); break;
      case 4: hist_u8_kernel<4><<<blocks, 256, 0, s>>>(t, n, hist, status); break;
      case 5: hist_u8_kernel<5><<<blocks, 256, 0, s>>>(t, n, hist, status); break;
      case 6: hist_u8_kernel<6><<<blocks, 256, 0, s>>>(t, n, hist, status); break;
      case 7: hist_u8_kernel<7><<<blocks, 256, 0, s>>>(t, n, hist, status); break;
      default: hist_u8_kernel<8><<<blocks, 256, 0, s>>>(t, n, hist, status); break;
    }
    return cudaGetLastError();
  }
  const bool smem = w <= 14;
  const size_t sb = smem ? ((size_t)4 << w) : 0;
  if (smem && sb > 48 * 1024) {
    cudaError_t e;
    if (sym_bytes == 1) e = cudaFuncSetAttribute(hist_generic_kernel<uint8_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    else if (sym_bytes == 2) e = cudaFuncSetAttribute(hist_generic_kernel<uint16_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    else e = cudaFuncSetAttribute(hist_generic_kernel<uint32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    if (e != cudaSuccess) return e;
  }
#define WVLT_HG(T)                                                                                   \
  (smem ? (hist_generic_kernel<T, true><<<blocks, 256, sb, s>>>((const T*)text, n, w, hist, status)) \
        : (hist_generic_kernel<T, false><<<blocks, 256, 0, s>>>((const T*)text, n, w, hist, status)))
  if (sym_bytes == 1) WVLT_HG(uint8_t);
  else if (sym_bytes == 2) WVLT_HG(uint16_t);
  else WVLT_HG(uint32_t);
#undef WVLT_HG
  return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

int wvlt_abi_version(void) { return WVLT_ABI_VERSION; }

const char* wvlt_error_string(int code) {
  switch (code) {
    case 0: return "ok";
    case WVLT_E_ARG: return "wvlt: bad argument";
    case WVLT_E_WIDTH: return "wvlt: code width above WVLT_MAX_WIDTH";
    case WVLT_E_WORKSPACE: return "wvlt: workspace too small";
    case WVLT_E_RANGE: return "wvlt: symbol outside [0, sigma)";
    default: return code > 0 ? cudaGetErrorString((cudaError_t)code) : "wvlt: unknown error";
  }
}

int wvlt_code_width(int64_t sigma) { return code_width_host(sigma); }

size_t wvlt_workspace_bytes(int64_t n, int sym_bytes, int64_t sigma, int kind) {
  Plan P;
  if (n < 0 || !(sym_bytes == 1 || sym_bytes == 2 || sym_bytes == 4)) return 0;
  if (!make_plan(n, sym_bytes, sigma, kind, &P)) return 0;
  return P.total;
}

int wvlt_histogram(const void* text, int sym_bytes, int64_t n, int64_t sigma, int64_t* hist, int32_t* status,
                   void* stream) {
  if (!(sym_bytes == 1 || sym_bytes == 2 || sym_bytes == 4) || n < 0 || sigma < 1 || !hist) return WVLT_E_ARG;
  if (n > 0 && !text) return WVLT_E_ARG;
  const int w = code_width_host(sigma);
  if (w > WVLT_MAX_WIDTH) return WVLT_E_WIDTH;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(hist, 0, ((size_t)1 << w) * 8, s);
  if (e != cudaSuccess) return (int)e;
  if (n == 0) return 0;
  if (w == 0) {  // a single bin holding every symbol; range = all zero
    int32_t* st = status;
    e = launch_hist(text, sym_bytes, n, 0, (unsigned long long*)hist, st, s);
    return (int)e;
  }
  e = launch_hist(text, sym_bytes, n, w, (unsigned long long*)hist, status, s);
  return (int)e;
}

int wvlt_build_device(const void* text, int sym_bytes, int64_t n, int64_t sigma, int kind, uint64_t* level_words,
                      int64_t* zeros, int64_t* hist, int64_t* borders, void* workspace, size_t workspace_bytes,
                      int32_t* status, void* stream) {
  if (!(sym_bytes == 1 || sym_bytes == 2 || sym_bytes == 4) || n < 0 || sigma < 1) return WVLT_E_ARG;
  if (kind != WVLT_KIND_WT && kind != WVLT_KIND_WM) return WVLT_E_ARG;
  Plan P;
  if (!make_plan(n, sym_bytes, sigma, kind, &P)) return WVLT_E_WIDTH;
  const int w = P.width;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (status) {
    e = cudaMemsetAsync(status, 0, 4, s);
    if (e != cudaSuccess) return (int)e;
  }
  const int64_t nwords = (n + 63) >> 6;
  if (n == 0 || w == 0) {
    // degenerate: no level bits to build (construct.py:457-458, bitperm.code_width)
    if (w == 0 && hist) {
      fill_i64_kernel<<<1, 1, 0, s>>>(hist, n);
      e = cudaGetLastError();
      if (e != cudaSuccess) return (int)e;
    } else if (hist) {
      e = cudaMemsetAsync(hist, 0, ((size_t)1 << w) * 8, s);
      if (e != cudaSuccess) return (int)e;
    }
    if (w > 0 && zeros) {
      e = cudaMemsetAsync(zeros, 0, (size_t)w * 8, s);
      if (e != cudaSuccess) return (int)e;
    }
    if (w > 0 && borders && w >= 2) {
      e = cudaMemsetAsync(borders, 0, (((size_t)1 << w) - 2) * 8, s);
      if (e != cudaSuccess) return (int)e;
    }
    if (w == 0 && n > 0 && status) {  // range check still applies: every symbol must be 0
      e = launch_hist(text, sym_bytes, n, 0, nullptr, status, s);
      if (e != cudaSuccess) return (int)e;
    }
    return 0;
  }
  if (!text || !level_words || !workspace) return WVLT_E_ARG;
  if (workspace_bytes < P.total) return WVLT_E_WORKSPACE;
  unsigned char* ws = (unsigned char*)workspace;
  int64_t* chain = (int64_t*)(ws + P.off_chain);
  int64_t* wtstart = (int64_t*)(ws + P.off_wtstart);
  int64_t* wm_base = (int64_t*)(ws + P.off_wmbase);
  int64_t* corr = (int64_t*)(ws + P.off_corr);
  uint32_t* counters = (uint32_t*)(ws + P.off_counter);
  uint64_t* stat = (uint64_t*)(ws + P.off_status);
  void* bufs[2] = {ws + P.off_buf0, ws + P.off_buf1};
  int32_t* st_flag = status;
  if (!st_flag) st_flag = (int32_t*)(counters + MAXP);  // scratch status word

  e = cudaMemsetAsync(level_words, 0, (size_t)w * nwords * 8, s);
  if (e != cudaSuccess) return (int)e;
  e = cudaMemsetAsync(stat, 0, P.status_bytes, s);
  if (e != cudaSuccess) return (int)e;
  unsigned long long* hw = (unsigned long long*)(chain + chain_off(w));
  e = cudaMemsetAsync(hw, 0, ((size_t)1 << w) * 8, s);
  if (e != cudaSuccess) return (int)e;
  e = launch_hist(text, sym_bytes, n, w, hw, st_flag, s);
  if (e != cudaSuccess) return (int)e;

  TablesArgs ta;
  memset(&ta, 0, sizeof(ta));
  ta.plan = P;
  ta.sigma = sigma;
  ta.n = n;
  ta.hist_in = hw;
  ta.chain = chain;
  ta.wtstart = wtstart;
  ta.wm_base = wm_base;
  ta.corr = corr;
  ta.counters = counters;
  ta.zeros_out = zeros;
  ta.hist_out = hist;
  ta.borders_out = (w >= 2) ? borders : nullptr;
  ta.status = st_flag;
  tables_kernel<<<1, TAB_THREADS, 0, s>>>(ta);
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;

  const void* cur = text;
  for (int p = 0; p < P.npass; ++p) {
    PassArgs pa;
    memset(&pa, 0, sizeof(pa));
    pa.src = cur;
    pa.dst = P.out_bytes[p] ? bufs[p & 1] : nullptr;
    pa.words = level_words;
    pa.nwords = nwords;
    pa.n = n;
    pa.level = P.lvl[p];
    pa.width = w;
    pa.kind = kind;
    pa.has_out = P.out_bytes[p] ? 1 : 0;
    pa.status = stat;
    pa.counter = counters + p;
    pa.epoch = (unsigned)(p + 1);
    pa.wm_base = wm_base + (int64_t)p * (KMAX + 1) * NDIG;
    pa.corr = corr;
    for (int j = 0; j <= KMAX; ++j) pa.corr_off[j] = P.corr_off[p][j];
    e = launch_pass(P.in_bytes[p], P.out_bytes[p], P.K[p], pa, P.ntiles[p], s);
    if (e != cudaSuccess) return (int)e;
    cur = pa.dst;
  }
  return 0;
}

int wvlt_build_host(const void* host_text, int sym_bytes, int64_t n, int64_t sigma, int kind,
                    uint64_t* host_level_words, int64_t* host_zeros, int64_t* host_hist, void* dev_text,
                    uint64_t* dev_level_words, void* dev_small, void* workspace, size_t workspace_bytes,
                    void* stream) {
  if (!(sym_bytes == 1 || sym_bytes == 2 || sym_bytes == 4) || n < 0 || sigma < 1) return WVLT_E_ARG;
  const int w = code_width_host(sigma);
  if (w > WVLT_MAX_WIDTH) return WVLT_E_WIDTH;
  if (!dev_small) return WVLT_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  int64_t* small = (int64_t*)dev_small;
  int32_t* dstatus = (int32_t*)small;
  int64_t* dzeros = small + 1;
  int64_t* dhist = small + 1 + w;
  if (n > 0) {
    if (!host_text || !dev_text) return WVLT_E_ARG;
    e = cudaMemcpyAsync(dev_text, host_text, (size_t)n * sym_bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return (int)e;
  }
  int rc = wvlt_build_device(dev_text, sym_bytes, n, sigma, kind, dev_level_words, dzeros, dhist, nullptr, workspace,
                             workspace_bytes, dstatus, s);
  if (rc) return rc;
  const int64_t nwords = (n + 63) >> 6;
  if (w > 0 && nwords > 0) {
    if (!host_level_words) return WVLT_E_ARG;
    e = cudaMemcpyAsync(host_level_words, dev_level_words, (size_t)w * nwords * 8, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return (int)e;
  }
  int32_t hstatus = 0;
  e = cudaMemcpyAsync(&hstatus, dstatus, 4, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return (int)e;
  if (host_zeros && w > 0) {
    e = cudaMemcpyAsync(host_zeros, dzeros, (size_t)w * 8, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return (int)e;
  }
  if (host_hist) {
    e = cudaMemcpyAsync(host_hist, dhist, ((size_t)1 << w) * 8, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return (int)e;
  }
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return (int)e;
  return (hstatus & WVLT_STATUS_RANGE) ? WVLT_E_RANGE : 0;
}

int wvlt_merge_bits(uint64_t* dst_words, int64_t word_lo, int64_t word_hi, int64_t n_bits, const int64_t* bounds,
                    const int64_t* src_starts, int64_t ntasks, const uint64_t* src_words, void* stream) {
  if (word_hi < word_lo || word_lo < 0 || n_bits < 0 || ntasks < 0) return WVLT_E_ARG;
  if (word_hi == word_lo) return 0;
  if (!dst_words || (n_bits > 0 && (!bounds || !src_starts || !src_words || ntasks < 1))) return WVLT_E_ARG;
  const int64_t nw = word_hi - word_lo;
  int64_t blocks = (nw + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  merge_bits_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dst_words, word_lo, word_hi, n_bits, bounds,
                                                                         src_starts, ntasks, src_words);
  return (int)cudaGetLastError();
}

}  // extern "C"
