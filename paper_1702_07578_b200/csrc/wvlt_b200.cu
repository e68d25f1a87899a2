// wvlt_b200.cu -- sm_100a wavelet tree / wavelet matrix construction.
//
// The reference builds every level with a counting-sort pass over the text
// (pkg/src/wvlt/construct.py:242-387, kernels in pkg/src/wvlt/_kernels.py).
// This file re-designs that hot path for B200:
//
//   K1  symbol histogram + range check, one read of the text; it also counts,
//       per tile of the first level pass, the digits that pass splits on
//       (replaces hist_and_msb_bits / full_histogram, _kernels.py:23-42)
//   K2  one small kernel deriving every table from that histogram: the fold
//       chain (fold_pairs, _kernels.py:45-49), per-level zero counts
//       (construct.py:238-239,273-288), node borders (starts_identity /
//       starts_ordered, _kernels.py:52-72) and the per-pass placement tables
//   S   per pass, an exclusive scan of the per-tile digit counts over tiles
//       (the interleaved (prefix, core) scan of levelstats.py:76-137 with
//       cores -> tiles)
//   K3  fused level pass: K levels per read of the current symbol order.  A
//       tile is staged in shared memory and split stably by one bit per level
//       (the wavelet-matrix refinement, structures.py:176-182); every level's
//       bits are taken with __ballot_sync in the tile-local order and emitted
//       as aligned 64-bit words at their global place; the order after K
//       levels is scattered to HBM narrowed to the bits still live, counting
//       the next pass's digits on the way (replaces sort_level_pass /
//       scatter_by_prefix / write_bits_from_symbols, _kernels.py:146-193).
//       Tiles never wait on each other: their digit prefixes are known at start.
//   K5  bit-interval shift-merge (replaces gather_bits, _kernels.py:196-232).
//
// Position algebra.  Let A_l be the level-l order,
// b_i(v) the i-th code bit of v (MSB first) and, for a pass starting at level
// l, d_j(v) = sum_{i<j} b_{l+i}(v) << i (an LSD digit).  Then
//   WM: A_{l+j} = stable sort of A_l by d_j, so
//       pos_{l+j}(x) = G_j[d] + C_j[d](x)
//   WT: A_{l+j} = stable sort of A_l by the (l+j)-bit prefix P, and
//       pos_{l+j}(x) = corr_j[P] + C_j[d](x)
// where C_j[d](x) counts symbols of A_l before x with digit d (tile prefix +
// rank inside the tile), G_j is the exclusive scan of the global digit counts
// and corr_j[P] = wtstart_{l+j}[P] - sum_{q'<q} cnt_{l+j}[q'2^j+e] for
// P = q 2^j + e.  Both tables come from the histogram alone (K2).

#include <cuda_runtime.h>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include <algorithm>
#include <stdint.h>
#include <string.h>

#include "wvlt_b200.h"

namespace {

constexpr int KMAX = 4;             // levels fused per pass
constexpr int NDIG = 1 << KMAX;     // digit bins per pass
constexpr int PASS_THREADS = 512;
#ifndef U8_CTAS_PER_SM
#define U8_CTAS_PER_SM 3
#endif
#ifndef U8_THREADS
#define U8_THREADS 512  // compute threads of the byte pass kernel (tile = 16 per thread)
#endif
#ifndef U8_FINAL_BUF
// 1: the last split goes to its own buffer (required with persistent CTAs: stage
// buffers then only ever receive bulk copies); 0: back into the stage buffer
#define U8_FINAL_BUF 1
#endif
#ifndef U8_TABLE_WARP
#define U8_TABLE_WARP 1  // 1: a 17th warp builds the tile tables concurrently; 0: the last compute warp does
#endif
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

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__host__ __device__ __forceinline__ unsigned rev_bits(unsigned d, int j) {  // j >= 1
#ifdef __CUDA_ARCH__
  return __brev(d) >> (32 - j);
#else
  unsigned r = 0;
  for (int i = 0; i < j; ++i) r |= ((d >> i) & 1u) << (j - 1 - i);
  return r;
#endif
}

// Keep a value opaque to the optimizer (so `x & mask` stays one LOP3 with a
// predicate output instead of being rewritten into shift/and/compare).
__device__ __forceinline__ uint32_t opaque(uint32_t v) {
  asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}

// Two-stream split store: `one ? smem[a1] = v : smem[a0] = v` as two predicated
// st.shared, so the zeros and the ones stream (each contiguous) are separate
// conflict-free wavefronts instead of one store with a selected address.
__device__ __forceinline__ void st_split_u8(uint32_t a1, uint32_t a0, uint32_t one, uint32_t v) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u8 [%0], %3;\n\t@!p st.shared.u8 [%1], %3;\n\t}"
      ::"r"(a1), "r"(a0), "r"(one), "r"(v) : "memory");
}
__device__ __forceinline__ void st_split_u16(uint32_t a1, uint32_t a0, uint32_t one, uint32_t v) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u16 [%0], %3;\n\t@!p st.shared.u16 [%1], %3;\n\t}"
      ::"r"(a1), "r"(a0), "r"(one), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void st_split_u32(uint32_t a1, uint32_t a0, uint32_t one, uint32_t v) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u32 [%0], %3;\n\t@!p st.shared.u32 [%1], %3;\n\t}"
      ::"r"(a1), "r"(a0), "r"(one), "r"(v) : "memory");
}
template <typename T>
__device__ __forceinline__ void st_split(uint32_t a1, uint32_t a0, uint32_t one, uint32_t v) {
  if (sizeof(T) == 1) st_split_u8(a1, a0, one, v);
  else if (sizeof(T) == 2) st_split_u16(a1, a0, one, v);
  else st_split_u32(a1, a0, one, v);
}

// PRMT selectors that stably sort 8 bytes by an 8-bit mask (zeros first, then
// ones), two nibble selectors per byte pair packed 8 x 4 bits; built at compile
// time and copied into shared memory by each byte pass CTA.
struct SortLut {
  uint32_t sel[256];
  constexpr SortLut() : sel() {
    for (int m = 0; m < 256; ++m) {
      uint32_t v = 0;
      int o = 0;
      for (int bit = 0; bit < 2; ++bit)
        for (int i = 0; i < 8; ++i)
          if (((m >> i) & 1) == bit) v |= (uint32_t)i << (4 * o++);
      sel[m] = v;
    }
  }
};
__device__ constexpr SortLut g_sort_lut{};

// Byte permute with the selector used as is (nibbles <= 7, so no masking).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// v >> (32 - k) through the multiplier (keeps the shift off the integer ALU pipe)
template <int SH>
__device__ __forceinline__ uint32_t shr_mul(uint32_t v) {
  if (SH == 0) return v;
#ifndef U8_SHR_MUL
  return v >> SH;
#endif
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(v), "n"(1u << (32 - SH)));
  return d;
}

// Inclusive warp scan (sum): shfl.up's in-range predicate guards the add, two
// instructions per step.
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  asm("{\n\t.reg .u32 t;\n\t.reg .pred p;\n\t"
      "shfl.sync.up.b32 t|p, %0, 1, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
      "shfl.sync.up.b32 t|p, %0, 2, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
      "shfl.sync.up.b32 t|p, %0, 4, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
      "shfl.sync.up.b32 t|p, %0, 8, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
      "shfl.sync.up.b32 t|p, %0, 16, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t}"
      : "+r"(v));
  return v;
}

// mbarrier + bulk async copy (global -> shared), completion by transaction bytes
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT;\n\t}" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// K1: histogram + first-pass tile digit counts.  Byte texts with width <= 8:
// one warp per tile; every lane owns a private column of 16-bit counters in
// shared memory (two bins per 32-bit word at (v >> 1) * 32 + lane, so a
// warp's 32 increments always hit 32 distinct banks): no atomics, no
// contention on Zipf heavy hitters.  After each tile the warp sums the columns
// (mod 2^16, as differences to the previous sums, so counters may wrap) to get
// the tile's bin counts, folds them to the pass-0 digit counts and keeps
// running totals in registers for the global histogram.
// ---------------------------------------------------------------------------
constexpr int HIST_WARPS = 4;

#ifndef WVLT_E_SMALL
#define WVLT_E_SMALL 16
#endif
constexpr int E_SMALL = WVLT_E_SMALL;  // symbols per thread per split for 1-2 byte symbols
constexpr int TILE_U8 = U8_THREADS * 16;  // tile of every pass that reads byte symbols

template <int W>
__global__ void __launch_bounds__(HIST_WARPS * 32) hist_u8_kernel(const uint8_t* __restrict__ text, int64_t n,
                                                                 int dshift_unused, int nd0,
                                                                 unsigned long long* __restrict__ hist,
                                                                 uint32_t* __restrict__ tcnt0, int64_t ntiles,
                                                                 int32_t* __restrict__ status) {
  constexpr int NB = 1 << W;
  constexpr int HALF = NB / 2;        // counter word p holds bins p (low 16 bits) and p + HALF (high)
  constexpr int WORDS = HALF * 32;    // per warp
  constexpr int K0 = W < KMAX ? W : KMAX;
  constexpr int DSH = W - K0;         // pass-0 digit = bin >> DSH; word p: digits p >> DSH, + ND / 2
  constexpr int ND = 1 << K0;
  constexpr int FLUSH_TILES = 128;    // a lane adds 256 per tile: < 2^16 between flushes, so
                                      // low-half sums never carry into the high half
  extern __shared__ __align__(16) uint32_t s_cols[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* c32 = s_cols + (size_t)wid * WORDS;
  for (int i = lane; i < WORDS; i += 32) c32[i] = 0;
  __syncwarp();
  uint32_t* c32w = c32 + lane;        // counter word p of this lane: c32w[32 p]
  uint32_t prev[ND];  // this lane's column sums per digit at the previous tile
#pragma unroll
  for (int d = 0; d < ND; ++d) prev[d] = 0;
  uint32_t bad = 0;
  const uint32_t badmask = ((0xFFu << W) & 0xFFu) * 0x01010101u;
  const bool aligned = (((uintptr_t)text) & 15) == 0;
  const int64_t gw = (int64_t)blockIdx.x * HIST_WARPS + wid;
  const int64_t nwarps = (int64_t)gridDim.x * HIST_WARPS;
  int since = 0;
  auto flush = [&]() {
    // exact bin totals since the last flush: column sums per word
    for (int p = 0; p < HALF; ++p) {
      const uint32_t wv = c32[p * 32 + lane];
      const uint32_t lo = __reduce_add_sync(FULL, wv & 0xFFFFu);
      const uint32_t hi = __reduce_add_sync(FULL, wv >> 16);
      if (lane == 0) {
        if (lo) atomicAdd(&hist[p], (unsigned long long)lo);
        if (hi) atomicAdd(&hist[p + HALF], (unsigned long long)hi);
      }
    }
    __syncwarp();
    for (int i = lane; i < WORDS; i += 32) c32[i] = 0;
#pragma unroll
    for (int d = 0; d < ND; ++d) prev[d] = 0;
    __syncwarp();
  };
  for (int64_t t = gw; t < ntiles; t += nwarps) {
    const int64_t first = t * TILE_U8;
    const int cnt = (int)min((int64_t)TILE_U8, n - first);
    if (cnt == TILE_U8 && aligned) {
      const uint4* v4 = reinterpret_cast<const uint4*>(text + first);
#ifndef HIST_BATCH
#define HIST_BATCH 8
#endif
#pragma unroll 1
      for (int k0 = 0; k0 < TILE_U8 / 16 / 32; k0 += HIST_BATCH) {
        uint4 q[HIST_BATCH];
#pragma unroll
        for (int k = 0; k < HIST_BATCH; ++k) q[k] = __ldcs(v4 + (k0 + k) * 32 + lane);
#pragma unroll
        for (int k = 0; k < HIST_BATCH; ++k) {
          const uint32_t wd[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (W < 8) bad |= wd[u] & badmask;
            // per byte: counter word from the low W-1 bits, increment 1 or
            // 1 << 16 from bit W-1 (two PRMT, one LEA, one IMAD)
            const uint32_t lo = wd[u] & ((uint32_t)(HALF - 1) * 0x01010101u);
            const uint32_t hb = (wd[u] >> (W - 1)) & 0x01010101u;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              // fire-and-forget shared atomic on the packed counter word: no
              // load->store dependency chain between consecutive symbols
              atomicAdd(c32w + prmt(lo, 0, 0x4440 + b) * 32, prmt(hb, 0, 0x4440 + b) * 0xFFFFu + 1u);
            }
          }
        }
      }
    } else {
      for (int i = lane; i < cnt; i += 32) {
        const uint32_t v = text[first + i];
        if (v >> W)
          bad = 1;
        else
          c32w[(v & (HALF - 1)) * 32] += (v >> (W - 1)) ? 0x10000u : 1u;
      }
    }
    __syncwarp();
    // the tile's pass-0 digit counts: each lane sums its own column (packed:
    // digit q low, digit q + ND/2 high; conflict-free), differences to the
    // previous tile, one reduction per digit
    uint32_t acc[ND / 2];
#pragma unroll
    for (int q = 0; q < ND / 2; ++q) acc[q] = 0;
#pragma unroll
    for (int p = 0; p < HALF; ++p) acc[p >> DSH] += c32[p * 32 + lane];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const uint32_t cur = d < ND / 2 ? (acc[d] & 0xFFFFu) : (acc[d - ND / 2] >> 16);
      const uint32_t delta = cur - prev[d];
      prev[d] = cur;
      const uint32_t c = __reduce_add_sync(FULL, delta);
      if (lane == d) tcnt0[(int64_t)d * ntiles + t] = c;
    }
    if (++since == FLUSH_TILES) {
      flush();
      since = 0;
    }
  }
  flush();
  (void)nd0;
  if (bad) atomicOr(status, WVLT_STATUS_RANGE);
}

// Generic histogram for wide symbols / wide alphabets.  Bins [0, 2^min(w,16))
// live in shared memory as 16-bit counters packed two per word (128 KB at
// most); an increment that wraps a counter is detected from the atomic's
// returned old value and carried into the global histogram exactly.  All the
// accounting comes from that single atomic's old value (no second shared
// atomic, so no interleaving can observe a half-corrected word): a low-half
// wrap leaks its carry into the high half, which then over-reports the high
// bin by one — the global high bin is debited 1 — and if that leaked carry in
// turn wrapped the high half (old high == 0xFFFF), it is credited 65536, the
// same as a high increment that wraps.  Bins at or above 2^16 (code widths
// 17..24) go to global atomics.
constexpr int HISTG_THREADS = 1024;
template <typename TIn>
__global__ void __launch_bounds__(HISTG_THREADS) hist_generic_kernel(const TIn* __restrict__ text, int64_t n, int w,
                                                                    unsigned long long* __restrict__ hist,
                                                                    int32_t* __restrict__ status) {
  extern __shared__ uint32_t s_pairs[];
  const int sw = w < 16 ? w : 16;          // shared-memory window: bins [0, 2^sw)
  const int npairs = ((1 << sw) + 1) >> 1;
  for (int i = threadIdx.x; i < npairs; i += blockDim.x) s_pairs[i] = 0;
  __syncthreads();
  unsigned bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t v = (uint32_t)__ldcs(text + i);
    if (w < 32 && (v >> w)) {
      bad = 1;
      continue;
    }
    if ((v >> sw) == 0) {
      const uint32_t hi = v & 1u;
      const uint32_t old = atomicAdd(&s_pairs[v >> 1], hi ? 0x10000u : 1u);
      if (hist) {
        if (hi) {
          if ((old >> 16) == 0xFFFFu) atomicAdd(&hist[v], 65536ull);  // high half wrapped out of the word
        } else if ((old & 0xFFFFu) == 0xFFFFu) {                     // low half wrapped
          atomicAdd(&hist[v], 65536ull);
          if (v + 1 < (1u << sw)) {
            // The carry landed in the high half: debit it, and credit the
            // high half's own wrap if the carry caused one.
            const unsigned long long adj = (old >> 16) == 0xFFFFu ? 65535ull : ~0ull;
            atomicAdd(&hist[v + 1], adj);
          }
        }
      }
    } else if (hist) {
      atomicAdd(&hist[v], 1ull);
    }
  }
  if (bad) atomicOr(status, WVLT_STATUS_RANGE);
  __syncthreads();
  if (hist) {
    for (int i = threadIdx.x; i < npairs; i += blockDim.x) {
      const uint32_t c = s_pairs[i];
      if (c & 0xFFFFu) atomicAdd(&hist[2 * i], (unsigned long long)(c & 0xFFFFu));
      if ((c >> 16) && 2 * i + 1 < (1 << sw)) atomicAdd(&hist[2 * i + 1], (unsigned long long)(c >> 16));
    }
  }
}

__global__ void fill_i64_kernel(int64_t* p, int64_t v) { *p = v; }

// Pass-0 tile digit counts for the generic path (wide symbols or alphabets):
// one warp per tile, lane-private 32-bit counters (bank = lane).
__global__ void __launch_bounds__(256) digits_kernel(const void* __restrict__ text, int sym_bytes, int64_t n, int tile,
                                                     int dshift, int nd0, int64_t ntiles,
                                                     uint32_t* __restrict__ tcnt0) {
  __shared__ uint32_t s_c[8][NDIG * 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* c = s_c[wid];
  const int64_t gw = (int64_t)blockIdx.x * 8 + wid;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t t = gw; t < ntiles; t += nwarps) {
    for (int i = lane; i < NDIG * 32; i += 32) c[i] = 0;
    __syncwarp();
    const int64_t first = t * tile;
    const int cnt = (int)min((int64_t)tile, n - first);
    for (int i = lane; i < cnt; i += 32) {
      uint32_t v;
      if (sym_bytes == 1) v = ((const uint8_t*)text)[first + i];
      else if (sym_bytes == 2) v = ((const uint16_t*)text)[first + i];
      else v = ((const uint32_t*)text)[first + i];
      const uint32_t e = (dshift >= 32 ? 0u : (v >> dshift)) & (uint32_t)(nd0 - 1);
      c[e * 32 + lane] += 1;
    }
    __syncwarp();
    if (lane < nd0) {
      uint32_t s = 0;
      for (int l = 0; l < 32; ++l) s += c[lane * 32 + l];
      tcnt0[(int64_t)lane * ntiles + t] = s;
    }
    __syncwarp();
  }
}

// K1 of a lean WM build (no histogram requested): pass-0 tile digit counts and
// the range check only -- the WM placement tables need nothing finer than each
// pass's digit totals, which the tile scans provide.  One warp per tile,
// lane-private 32-bit counter columns (fire-and-forget atomics, no overflow).
template <typename TIn, bool CHECK>
__global__ void __launch_bounds__(256) digits_fast_kernel(const TIn* __restrict__ text, int64_t n, int tile, int dshift,
                                                          int nd0, int64_t ntiles, uint32_t vmax_ok,
                                                          uint32_t* __restrict__ tcnt0, int32_t* __restrict__ status) {
  constexpr int PER = 16 / sizeof(TIn);  // symbols per 16-byte load
  __shared__ uint32_t s_c[8][NDIG * 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* c = s_c[wid];
  for (int i = lane; i < NDIG * 32; i += 32) c[i] = 0;
  __syncwarp();
  uint32_t* cl = c + lane;
  const uint32_t dmask = (uint32_t)nd0 - 1u;
  uint32_t prev[NDIG];
#pragma unroll
  for (int d = 0; d < NDIG; ++d) prev[d] = 0;
  uint32_t vmax = 0;
  const bool aligned = (((uintptr_t)text) & 15) == 0;
  const int64_t gw = (int64_t)blockIdx.x * 8 + wid;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t t = gw; t < ntiles; t += nwarps) {
    const int64_t first = t * tile;
    const int cnt = (int)min((int64_t)tile, n - first);
    if (cnt == tile && aligned) {
      const uint4* v4 = reinterpret_cast<const uint4*>(text + first);
      const int nq = tile / PER;
#pragma unroll 4
      for (int k = lane; k < nq; k += 32) {
        const uint4 q = __ldcs(v4 + k);
        const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (sizeof(TIn) == 1) {
            if (CHECK) vmax = __vmaxu4(vmax, wd[u]);
            const uint32_t dg = (wd[u] >> dshift) & (dmask * 0x01010101u);
#pragma unroll
            for (int b = 0; b < 4; ++b) atomicAdd(cl + prmt(dg, 0, 0x4440 + b) * 32, 1u);
          } else if (sizeof(TIn) == 2) {
            if (CHECK) vmax = __vmaxu2(vmax, wd[u]);
            atomicAdd(cl + (((wd[u] & 0xFFFFu) >> dshift) & dmask) * 32, 1u);
            atomicAdd(cl + ((wd[u] >> (16 + dshift)) & dmask) * 32, 1u);
          } else {
            if (CHECK) vmax = max(vmax, wd[u]);
            atomicAdd(cl + ((dshift >= 32 ? 0u : (wd[u] >> dshift)) & dmask) * 32, 1u);
          }
        }
      }
    } else {
      for (int i = lane; i < cnt; i += 32) {
        const uint32_t v = (uint32_t)text[first + i];
        vmax = max(vmax, v);
        atomicAdd(cl + ((dshift >= 32 ? 0u : (v >> dshift)) & dmask) * 32, 1u);
      }
    }
    __syncwarp();
#pragma unroll
    for (int d = 0; d < NDIG; ++d) {
      if (d < nd0) {
        const uint32_t cur = cl[d * 32];
        const uint32_t tot = __reduce_add_sync(FULL, cur - prev[d]);
        prev[d] = cur;
        if (lane == d) tcnt0[(int64_t)d * ntiles + t] = tot;
      }
    }
  }
  // SIMD maxima hold per-lane maxima of byte / halfword lanes: fold them
  if (sizeof(TIn) == 1) vmax = max(max(vmax & 0xFFu, (vmax >> 8) & 0xFFu), max((vmax >> 16) & 0xFFu, vmax >> 24));
  if (sizeof(TIn) == 2) vmax = max(vmax & 0xFFFFu, vmax >> 16);
  if (CHECK && vmax > vmax_ok) atomicOr(status, WVLT_STATUS_RANGE);
}

// Per-pass WM tables from the pass's digit totals (lean builds): the G table
// of every level of the pass (as tables_kernel step 5) and its zero counts.
__global__ void wm_pass_tables_kernel(const uint32_t* __restrict__ tcnt, const int64_t* __restrict__ tpre,
                                      int64_t ntiles, int K, int l0, int64_t* __restrict__ wm_base,
                                      int64_t* __restrict__ zeros) {
  __shared__ int64_t s_tot[NDIG];  // by LSD digit d = rev(numeric e)
  const int lane = threadIdx.x;
  const int nd = 1 << K;
  if (lane < nd) {
    const int64_t i = (int64_t)lane * ntiles + ntiles - 1;
    s_tot[rev_bits((unsigned)lane, K)] = tpre[i] + (int64_t)tcnt[i];
  }
  __syncwarp();
  if (lane == 0) {
    for (int j = 1; j <= K; ++j) {
      const int mj = 1 << j;
      int64_t run = 0;
      for (int d = 0; d < mj; ++d) {
        int64_t cj = 0;
        for (int e = d; e < nd; e += mj) cj += s_tot[e];
        wm_base[j * NDIG + d] = run;
        run += cj;
      }
    }
    if (zeros) {
      // level l0 + j: symbols whose (j+1)-th digit bit from the top is 0, i.e.
      // LSD digit d with bit j clear
      for (int j = 0; j < K; ++j) {
        int64_t z = 0;
        for (int d = 0; d < nd; ++d)
          if (!((d >> j) & 1)) z += s_tot[d];
        zeros[l0 + j] = z;
      }
    }
  }
}

// Widen symbols stored narrower than the code width (e.g. uint8 storage with
// sigma > 256) so the all-ones tail sentinel of the pass kernel covers every
// code bit.
template <typename TI, typename TO>
__global__ void widen_kernel(const TI* __restrict__ in, TO* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (TO)in[i];
}



// ---------------------------------------------------------------------------
// Build plan shared by host and kernels
// ---------------------------------------------------------------------------
struct Plan {
  int width;
  int kind;
  int npass;
  int widen_bytes;      // > 0: text is widened to this many bytes before pass 0
  int lvl[MAXP];        // first level of the pass
  int K[MAXP];          // levels in the pass
  int in_bytes[MAXP];   // element bytes of A_lvl
  int out_bytes[MAXP];  // element bytes of A_{lvl+K} (0 = no output)
  int tile[MAXP];       // symbols per tile
  int tshift[MAXP];     // log2(tile)
  int64_t ntiles[MAXP];
  int64_t corr_off[MAXP][KMAX + 1];  // WT placement tables (int64 offsets into corr)
  int64_t corr_total;
  // workspace carve (byte offsets)
  size_t off_chain, off_wtstart, off_wmbase, off_corr, off_scratch, off_tcnt[MAXP], off_tpre[MAXP], off_bsum,
      off_buf0, off_buf1, off_wide;
  size_t tcnt_bytes, buf_bytes, total;
  // WM with w > 8: the last tail_w <= 8 levels (from tail_lvl) are one fused
  // byte pass (k8.cuh) over the u8 output of the stage before; its workspace
  // is the other ping-pong buffer
  int tail_w, tail_lvl;
  // WM, 2-byte input with 10..16 live bits (lean builds): the k16_w = live - 8
  // levels from k16_lvl are one fused 2-byte pass (k16.cuh) whose byte output
  // feeds the tail; output + its tables in the other ping-pong buffer
  int k16_w, k16_lvl;
  // WM, 4-byte input with 18..24 live bits (lean builds): the k32_w = live - 16
  // levels from k32_lvl are one fused 4-byte pass (k32.cuh) whose 2-byte
  // output feeds the fused 2-byte pass
  int k32_w, k32_lvl;
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
  // 4. node borders: WT in numeric prefix order (also the WT placement tables'
  // input), WM in bit-reversed order (only when requested)
  for (int k = 0; k <= w; ++k) {
    if (P.kind == WVLT_KIND_WM && !a.borders_out) break;
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
      // blockDim.x is a multiple of nd: thread tid only ever sees numeric digit tid % nd
      int64_t acc = 0;
      for (int64_t i = tid; i < tot; i += blockDim.x) acc += c[i];
      if (acc) atomicAdd(&s_dig[rev_bits((unsigned)(tid & (nd - 1)), K)], (unsigned long long)acc);
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
// S: exclusive scan of the per-tile digit counts over tiles, digit-major
// layout cnt[e][tile] -> pre[e][tile].  Two launches: block totals, then each
// block adds the totals of the blocks before it and scans its own range.
// ---------------------------------------------------------------------------
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__global__ void __launch_bounds__(SCAN_THREADS) scan_reduce_kernel(const uint32_t* __restrict__ cnt, int64_t ntiles,
                                                                   int64_t nblk, int64_t* __restrict__ bsum) {
  __shared__ int64_t s_red[32];
  const int e = blockIdx.y;
  const int64_t b = blockIdx.x;
  const uint32_t* row = cnt + (int64_t)e * ntiles;
  int64_t s = 0;
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    const int64_t i = b * SCAN_TILE + (int64_t)k * SCAN_THREADS + threadIdx.x;
    if (i < ntiles) s += row[i];
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    int64_t v = threadIdx.x < SCAN_THREADS / 32 ? s_red[threadIdx.x] : 0;
    v = warp_sum(v);
    if (threadIdx.x == 0) bsum[(int64_t)e * nblk + b] = v;
  }
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_apply_kernel(const uint32_t* __restrict__ cnt, int64_t ntiles,
                                                                  int64_t nblk, const int64_t* __restrict__ bsum,
                                                                  int64_t* __restrict__ pre) {
  __shared__ int64_t s_red[33];
  const int e = blockIdx.y;
  const int64_t b = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // offset = totals of the blocks before b
  int64_t off = 0;
  for (int64_t i = threadIdx.x; i < b; i += SCAN_THREADS) off += bsum[(int64_t)e * nblk + i];
  off = warp_sum(off);
  if (lane == 0) s_red[wid] = off;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < SCAN_THREADS / 32; ++w) t += s_red[w];
    s_red[32] = t;
  }
  __syncthreads();
  const int64_t boff = s_red[32];
  __syncthreads();
  // block scan, SCAN_ITEMS consecutive tiles per thread
  const uint32_t* row = cnt + (int64_t)e * ntiles;
  int64_t* out = pre + (int64_t)e * ntiles;
  const int64_t i0 = b * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  uint32_t v[SCAN_ITEMS];
  int64_t ts = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = (i0 + k < ntiles) ? row[i0 + k] : 0u;
    ts += v[k];
  }
  int64_t incl = ts;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_red[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int64_t x = lane < SCAN_THREADS / 32 ? s_red[lane] : 0;
    int64_t sc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(FULL, sc, o);
      if (lane >= o) sc += t;
    }
    if (lane < SCAN_THREADS / 32) s_red[lane] = sc - x;
  }
  __syncthreads();
  int64_t run = boff + s_red[wid] + incl - ts;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (i0 + k < ntiles) out[i0 + k] = run;
    run += v[k];
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
  int64_t ntiles;
  int level, width, kind, has_out;
  const uint32_t* tcnt;  // this pass: [2^K][ntiles] digit counts (numeric digit)
  const int64_t* tpre;   // this pass: [2^K][ntiles] exclusive prefixes over tiles
  uint32_t* ncnt;        // next pass: [2^K'][ntiles'] digit counts (accumulated here), or null
  int64_t nntiles;
  int ntshift;           // log2(next tile)
  int nK;                // next pass K
  const int64_t* wm_base;  // this pass: [KMAX+1][NDIG]
  const int64_t* corr;     // WT tables of this pass: table j at corr + corr_off[j]
  int64_t corr_off[KMAX + 1];
};

template <typename TIn, int K, int E, int NT = PASS_THREADS>
struct PassSmem {
  static constexpr int T = NT * E;
  static constexpr int NC = T / 32;
  // order buffers A_l .. A_{l+K-1} in the tile-local digit orders d_0 .. d_{K-1}
  static constexpr size_t buf_bytes = (size_t)K * T * sizeof(TIn);
  // ballot words of every level in its local order (+pad words for extract_bits)
  static constexpr size_t bits_bytes = (size_t)K * (NC + 4) * 4;
  static constexpr size_t total = buf_bytes + bits_bytes;
};

__device__ __forceinline__ uint64_t extract_bits(const uint32_t* L, int off, int cnt) {
  const int i = off >> 5, s = off & 31;
  uint64_t v = ((uint64_t)L[i] | ((uint64_t)L[i + 1] << 32)) >> s;
  if (s) v |= (uint64_t)L[i + 2] << (64 - s);
  return cnt >= 64 ? v : (v & ((1ull << cnt) - 1));
}

template <typename TIn>
__device__ __forceinline__ unsigned digit_of(TIn x, int top_shift, int j) {
  // LSD digit d_j = sum_{i<j} bit(top_shift - i) << i
  unsigned d = 0;
  for (int i = 0; i < j; ++i) d |= (((uint32_t)x >> (top_shift - i)) & 1u) << i;
  return d;
}

// Per-tile placement tables, built by the table warp while the compute warps
// run the splits.
template <typename TOut, int K>
struct TileTables {
  int cnt[K + 1][NDIG];     // group sizes per digit length j (LSD digit)
  int ls[K + 1][NDIG];      // group starts in the tile-local order of length j
  int64_t lb[K + 1][NDIG];  // symbols of earlier tiles with the same digit
  int64_t gs[K + 1][NDIG];  // uniform tiles: global start of each group's run
  TOut* row[NDIG];          // uniform tiles: output row of each numeric digit (dst + offset)
  int thr[NDIG];            // local position where that run crosses into the next pass's next tile
  int64_t ft[NDIG];         // first next-pass tile of each run
  int ipre[NDIG + 1];       // byte copy-out: 16-byte destination chunks before each group (tile order)
  int q1;                   // tile lies inside one level-l node (always for WM)
};

template <typename TIn, typename TOut, int K>
__device__ __forceinline__ void table_warp(const PassArgs& a, TileTables<TOut, K>& tt, const TIn* buf0, int64_t tile,
                                           int cnt, int lane, int allt) {
  constexpr int nd = 1 << K;
  const int w = a.width, l0 = a.level;
  const bool wm = a.kind == WVLT_KIND_WM;
  if (lane < nd) {
    const int d = (int)rev_bits((unsigned)lane, K);  // lane = numeric digit
    tt.cnt[K][d] = (int)__ldg(a.tcnt + (int64_t)lane * a.ntiles + tile);
    tt.lb[K][d] = __ldg(a.tpre + (int64_t)lane * a.ntiles + tile);
  }
  __syncwarp();
  // every shorter digit: sums over the digits sharing the low j bits
  for (int j = 0; j < K; ++j) {
    if (lane < (1 << j)) {
      int c = 0;
      int64_t lb = 0;
      for (int e = lane; e < nd; e += (1 << j)) {
        c += tt.cnt[K][e];
        lb += tt.lb[K][e];
      }
      tt.cnt[j][lane] = c;
      tt.lb[j][lane] = lb;
    }
  }
  __syncwarp();
  // group starts in the tile-local orders (groups by increasing LSD digit)
  for (int j = 0; j <= K; ++j) {
    const int mj = 1 << j;
    const int c = lane < mj ? tt.cnt[j][lane] : 0;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane < mj) tt.ls[j][lane] = incl - c;
  }
  bool q1 = true;
  int64_t q = 0;
  if (!wm) {
    if (allt > 0) bar_sync(3, allt);  // tile staged (inline callers have staged it)
    const int sh = w - l0;
    const uint64_t qf = sh >= 32 ? 0 : ((uint64_t)(uint32_t)buf0[0] >> sh);
    const uint64_t ql = sh >= 32 ? 0 : ((uint64_t)(uint32_t)buf0[cnt - 1] >> sh);
    q1 = qf == ql;
    q = (int64_t)qf;
  }
  if (lane == 0) tt.q1 = q1;
  __syncwarp();
  if (q1) {  // placement is a per-digit constant in this tile
    for (int j = 1; j <= K; ++j) {
      if (lane < (1 << j)) {
        const int d = lane;
        const int64_t tb = wm ? __ldg(a.wm_base + j * NDIG + d)
                              : __ldg(a.corr + a.corr_off[j] + (q << j) + (int64_t)rev_bits((unsigned)d, j));
        tt.gs[j][d] = tb + tt.lb[j][d];
      }
    }
    __syncwarp();
    if (lane < nd && a.has_out) {
      const int d = (int)rev_bits((unsigned)lane, K);  // lane = numeric digit
      const int64_t g = tt.gs[K][d];
      tt.row[lane] = reinterpret_cast<TOut*>(a.dst) + (g - tt.ls[K][d]);
      const int64_t ntile = (int64_t)1 << a.ntshift;
      tt.thr[lane] = tt.ls[K][d] + (int)(ntile - (g & (ntile - 1)));
      tt.ft[lane] = g >> a.ntshift;
    }
    if (sizeof(TOut) == 1 && a.has_out) {
      // whole 16-byte-aligned destination chunks inside each group's run,
      // prefix in tile order (the partial edge chunks are handled separately)
      __syncwarp();
      int c = 0;
      if (lane < nd) {
        const int n = tt.cnt[K][lane];
        const uintptr_t lo = (uintptr_t)(tt.row[rev_bits((unsigned)lane, K)] + tt.ls[K][lane]);
        const intptr_t f = (intptr_t)((lo + n) >> 4) - (intptr_t)((lo + 15) >> 4);
        c = f > 0 ? (int)f : 0;
      }
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane < nd) tt.ipre[lane] = incl - c;
      if (lane == nd - 1) tt.ipre[nd] = incl;
    }
  }
  if (allt > 0) {
    __threadfence_block();
    bar_arrive(2, allt);
  }
}

// Levels l0+1 .. l0+K-1 of a uniform tile: one warp per (level j, run r),
// task t = 2^j - 2 + r; whole words stored, run-edge words OR-ed into the
// pre-zeroed level (gather_bits' owner rule, _kernels.py:197-205, relaxed to
// atomics at run edges).
template <typename TOut, int K, int NC>
__device__ __forceinline__ void emit_uniform(const PassArgs& a, const TileTables<TOut, K>& tt, const uint32_t* bits,
                                             int wid, int lane, int nwarps) {
  constexpr int nd = 1 << K;
  for (int t = wid; t < nd - 2; t += nwarps) {
    const int j = 31 - __clz(t + 2);
    const int r = t + 2 - (1 << j);
    const int len = tt.cnt[j][r];
    if (!len) continue;
    const int64_t g = tt.gs[j][r];
    const int ls = tt.ls[j][r];
    const uint32_t* L = bits + j * (NC + 4);
    uint64_t* gw = a.words + (int64_t)(a.level + j) * a.nwords;
    const int64_t W0 = g >> 6, W1 = (g + len - 1) >> 6;
    for (int64_t W = W0 + lane; W <= W1; W += 32) {
      const int64_t wb = W << 6;
      const int64_t a0 = g > wb ? g : wb;
      const int64_t e0 = g + len;
      const int64_t b0 = e0 < wb + 64 ? e0 : wb + 64;
      const int c = (int)(b0 - a0);
      const uint64_t v = extract_bits(L, ls + (int)(a0 - g), c) << (int)(a0 - wb);
      if (c == 64)
        gw[W] = v;
      else
        atomicOr(reinterpret_cast<unsigned long long*>(gw + W), (unsigned long long)v);
    }
  }
}

// Levels l0+1 .. l0+K-1 of a WT tile spanning several nodes: per-symbol
// placement (elements of order j are buf + j*T, linear layout), runs found by
// contiguity of the global position inside each warp chunk.
template <typename TIn, typename TOut, int K>
__device__ __forceinline__ void emit_multinode(const PassArgs& a, const TileTables<TOut, K>& tt, const TIn* buf,
                                               int T, int cnt, int tid, int lane, int nthreads) {
  const int w = a.width, l0 = a.level;
#pragma unroll 1
  for (int j = 1; j < K; ++j) {
    uint64_t* gw = a.words + (int64_t)(l0 + j) * a.nwords;
    const TIn* cur = buf + (size_t)j * T;
    const int tshift = w - 1 - l0;
    const int pshift = w - l0 - j;
    const int64_t* ctab = a.corr + a.corr_off[j];
#pragma unroll 1
    for (int p0 = (tid >> 5) * 32; p0 < T; p0 += nthreads) {
      const int p = p0 + lane;
      const bool valid = p < cnt;
      const TIn xv = cur[p];
      int64_t gpos = 0;
      unsigned bit = 0;
      if (valid) {
        const unsigned d = digit_of(xv, tshift, j);
        const uint64_t P = pshift >= 32 ? 0 : ((uint64_t)(uint32_t)xv >> pshift);
        gpos = ctab[P] + tt.lb[j][d] + p - tt.ls[j][d];
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
  }
}

// One CTA = one tile of T = 512 * E symbols of A_l; CTAs are independent.
// Generic (striped) variant for 2- and 4-byte symbols: symbol p of the
// tile-local order lives in lane p % 32 of warp p / (32 E) (warp-contiguous
// 32-symbol chunks), so a ballot gives 32 consecutive bits.  Warps 0..15 stage
// the tile and run the splits; warp 16 builds the placement tables
// concurrently (named barriers 1: compute warps, 2: tables ready, 3: staged).
constexpr int TAB_WARP_THREADS = 32;
template <typename TIn, typename TOut, int K, int E>
__global__ void __launch_bounds__(PASS_THREADS + TAB_WARP_THREADS, 2) level_pass_kernel(const PassArgs a) {
  using S = PassSmem<TIn, K, E>;
  constexpr int T = S::T;
  constexpr int NC = S::NC;
  constexpr int NW = PASS_THREADS / 32;
  constexpr int ALLT = PASS_THREADS + TAB_WARP_THREADS;
  constexpr int nd = 1 << K;
  extern __shared__ __align__(16) unsigned char smem[];
  TIn* buf = reinterpret_cast<TIn*>(smem);
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + S::buf_bytes);

  __shared__ TileTables<TOut, K> tt;
  __shared__ __align__(16) uint32_t s_wtot[2][NW];
  __shared__ uint32_t s_ncnt[2 * NDIG * NDIG];  // next-pass digit counts per (run, next tile)

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int w = a.width, l0 = a.level;
  const bool wm = a.kind == WVLT_KIND_WM;
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * T;
  const int cnt = (int)min((int64_t)T, a.n - base);

  if (wid == NW) {
    table_warp<TIn, TOut, K>(a, tt, buf, tile, cnt, lane, ALLT);
    return;
  }

  // ---- stage the tile (invalid tail slots = all ones so they sort last) ----
  const TIn* src = reinterpret_cast<const TIn*>(a.src) + base;
  if (cnt == T && ((((uintptr_t)src) & 15) == 0)) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(buf);
#pragma unroll
    for (int i = tid; i < (int)(T * sizeof(TIn) / 16); i += PASS_THREADS) d4[i] = __ldcs(s4 + i);
  } else {
    for (int p = tid; p < T; p += PASS_THREADS) buf[p] = p < cnt ? src[p] : (TIn)~(TIn)0;
  }
  if (tid < 2 * NDIG * NDIG) s_ncnt[tid] = 0;
  bar_sync(1, PASS_THREADS);
  if (!wm) bar_arrive(3, ALLT);

  const unsigned lt = lanemask_lt();
  const int pbase = wid * E * 32;  // this warp's first symbol (warp-contiguous chunks)
  uint32_t m[E];

#pragma unroll 1
  for (int j = 0; j < K; ++j) {
    const uint32_t bmask = opaque(1u << (w - 1 - l0 - j));
    const TIn* cur = buf + (size_t)j * T;
#pragma unroll
    for (int e = 0; e < E; ++e) m[e] = __ballot_sync(FULL, (uint32_t)cur[pbase + e * 32 + lane] & bmask);
    if (j == 0) {
      // level l0 is in global order already: aligned word stores
      uint32_t* g32 = reinterpret_cast<uint32_t*>(a.words + (int64_t)l0 * a.nwords) + (base >> 5) + wid * E;
      if (cnt == T) {
        if (lane == 0) {
#pragma unroll
          for (int q4 = 0; q4 < E / 4; ++q4)
            reinterpret_cast<uint4*>(g32)[q4] = make_uint4(m[4 * q4], m[4 * q4 + 1], m[4 * q4 + 2], m[4 * q4 + 3]);
        }
      } else {
        uint32_t mine = 0;
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (lane == e) mine = m[e];
        const int64_t lim = 2 * a.nwords - ((base >> 5) + wid * E);
        if (lane < E && lane < lim) {
          const int first = (wid * E + lane) * 32;
          uint32_t v = mine;
          if (first + 32 > cnt) v = first >= cnt ? 0u : (v & ((1u << (cnt - first)) - 1u));
          g32[lane] = v;
        }
      }
    } else if (lane == 0) {
      uint4* b4 = reinterpret_cast<uint4*>(bits + j * (NC + 4) + wid * E);
#pragma unroll
      for (int q4 = 0; q4 < E / 4; ++q4) b4[q4] = make_uint4(m[4 * q4], m[4 * q4 + 1], m[4 * q4 + 2], m[4 * q4 + 3]);
    }
    if (j + 1 == K && !a.has_out) break;
    uint32_t run = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) run += __popc(m[e]);
    if (lane == 0) s_wtot[j & 1][wid] = run;
    bar_sync(1, PASS_THREADS);
    const uint32_t wv = lane < NW ? s_wtot[j & 1][lane] : 0u;
    const uint32_t wpre = __reduce_add_sync(FULL, lane < wid ? wv : 0u);
    const uint32_t tot = __reduce_add_sync(FULL, wv);
    // ones of chunk e go to U1 + ce + rank, zeros to U0 + 32 e - ce - rank
    const int U1 = T - (int)tot + (int)wpre;
    const int U0 = pbase + lane - (int)wpre;
    int ce = 0;  // ones in this warp's earlier chunks
    if (j + 1 < K) {
      const uint32_t nxt = (uint32_t)__cvta_generic_to_shared(buf + (size_t)(j + 1) * T);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t xv = (uint32_t)cur[pbase + e * 32 + lane];
        const int r = __popc(m[e] & lt);
        st_split<TIn>(nxt + (uint32_t)(U1 + ce + r) * (uint32_t)sizeof(TIn),
                      nxt + (uint32_t)(U0 + 32 * e - ce - r) * (uint32_t)sizeof(TIn), xv & bmask, xv);
        ce += __popc(m[e]);
      }
      bar_sync(1, PASS_THREADS);
    } else {
      // last split: straight to HBM, counting the next pass's digits per (run, next tile)
      bar_sync(2, ALLT);  // placement tables
      const uint32_t keep = wm ? ((w - l0 - K) >= 32 ? FULL : ((1u << (w - l0 - K)) - 1u)) : FULL;
      const int eshift = w - l0 - K;
      const int nshift = w - l0 - K - a.nK;  // next pass digit = bits l0+K .. l0+K+nK-1
      const unsigned nmask = (1u << a.nK) - 1u;
      const bool q1 = tt.q1;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int r = __popc(m[e] & lt);
        const uint32_t xv = (uint32_t)cur[pbase + e * 32 + lane];
        const int pos = (xv & bmask) ? U1 + ce + r : U0 + 32 * e - ce - r;
        ce += __popc(m[e]);
        if (pos < cnt) {
          if (q1) {
            const unsigned dig = (xv >> eshift) & (nd - 1);
            tt.row[dig][pos] = (TOut)(xv & keep);
            const unsigned h = pos >= tt.thr[dig] ? 1u : 0u;
            if (a.ncnt) atomicAdd(&s_ncnt[(((dig << 1) | h) << a.nK) | ((xv >> nshift) & nmask)], 1u);
          } else {
            const unsigned d = rev_bits((xv >> eshift) & (nd - 1), K);
            const uint64_t P = eshift >= 32 ? 0 : ((uint64_t)xv >> eshift);
            const int64_t gpos = a.corr[a.corr_off[K] + P] + tt.lb[K][d] + pos - tt.ls[K][d];
            reinterpret_cast<TOut*>(a.dst)[gpos] = (TOut)(xv & keep);
            if (a.ncnt) atomicAdd(&a.ncnt[(int64_t)((xv >> nshift) & nmask) * a.nntiles + (gpos >> a.ntshift)], 1u);
          }
        }
      }
      bar_sync(1, PASS_THREADS);
      if (q1 && a.ncnt) {
        const int ncount = 2 * nd << a.nK;
        for (int i = tid; i < ncount; i += PASS_THREADS) {
          const uint32_t v = s_ncnt[i];
          if (v) {
            const int slot = i >> a.nK, ne = i & (int)nmask;
            atomicAdd(&a.ncnt[(int64_t)ne * a.nntiles + tt.ft[slot >> 1] + (slot & 1)], v);
          }
        }
      }
    }
  }
  if (!a.has_out) {
    bar_sync(1, PASS_THREADS);  // every warp's ballot words are stored
    bar_sync(2, ALLT);          // placement tables
  }
  if (tt.q1)
    emit_uniform<TOut, K, NC>(a, tt, bits, wid, lane, NW);
  else
    emit_multinode<TIn, TOut, K>(a, tt, buf, T, cnt, tid, lane, PASS_THREADS);
}

// Copy-out of a uniform byte tile sorted into `fin` (groups in tile order).
// Work items are the whole 16-byte-aligned destination chunks inside every
// group's run (TileTables::ipre): a chunk is read from shared memory at any
// byte offset (five words, four PRMT) and written with one 16-byte store.  The
// partial chunks at both ends of a run (< 16 bytes each) go byte by byte, one
// warp per group.  Every symbol also counts its next-pass digit per (run, next
// tile) in s_ncnt.
template <int K>
__device__ __forceinline__ void copy_out_u8(const PassArgs& a, const TileTables<uint8_t, K>& tt, const uint8_t* fin,
                                            uint32_t* s_ncnt, int tid) {
  constexpr int nd = 1 << K;
  static_assert(nd <= U8_THREADS / 32, "one warp per group for the run edges");
  const int nK = a.nK;
  const int nshift = a.width - a.level - K - nK;
  const uint32_t nmask = (1u << nK) - 1u;
  const uint32_t nrep = nmask * 0x01010101u;
  const uint32_t keep = a.kind == WVLT_KIND_WM ? ((1u << (a.width - a.level - K)) - 1u) : 0xFFu;
  const uint32_t krep = keep * 0x01010101u;
  const int nitems = tt.ipre[nd];
  const uint32_t* fw = reinterpret_cast<const uint32_t*>(fin);
  for (int it = tid; it < nitems; it += U8_THREADS) {
    int d = 0;
#pragma unroll
    for (int s = nd / 2; s >= 1; s >>= 1)
      if (tt.ipre[d + s] <= it) d += s;
    const int num = (int)rev_bits((unsigned)d, K);
    uint8_t* row = tt.row[num];
    const uintptr_t D = ((((uintptr_t)(row + tt.ls[K][d]) + 15) >> 4) + (uintptr_t)(it - tt.ipre[d])) << 4;
    const int p = (int)(D - (uintptr_t)row);  // tile-local position of the chunk's first byte
    const int thr = tt.thr[num];
    const uint32_t cb = (uint32_t)(num << 1) << nK;
    const uint32_t* q = fw + (p >> 2);
    const uint32_t sel = 0x3210u + 0x1111u * (uint32_t)(p & 3);
    const uint32_t w0 = q[0], w1 = q[1], w2 = q[2], w3 = q[3], w4 = q[4];
    uint32_t v[4] = {prmt(w0, w1, sel), prmt(w1, w2, sel), prmt(w2, w3, sel), prmt(w3, w4, sel)};
    if (p >= thr || p + 16 <= thr) {
      uint32_t* cnt = s_ncnt + (cb | (p >= thr ? (1u << nK) : 0u));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t m = (v[k] >> nshift) & nrep;
#pragma unroll
        for (int i = 0; i < 4; ++i) atomicAdd(cnt + __byte_perm(m, 0, 0x4440 + i), 1u);
      }
    } else {  // the chunk where the run crosses into the next pass's next tile
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t m = (v[k] >> nshift) & nrep;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          atomicAdd(s_ncnt + (cb | (p + 4 * k + i >= thr ? (1u << nK) : 0u) | __byte_perm(m, 0, 0x4440 + i)), 1u);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] &= krep;
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(D), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
                 : "memory");
  }
  // run edges: warp d, lanes 0-15 the head bytes, lanes 16-31 the tail bytes
  const int wid = tid >> 5, lane = tid & 31;
  if (wid < nd) {
    const int d = wid;
    const int n = tt.cnt[K][d];
    const int num = (int)rev_bits((unsigned)d, K);
    uint8_t* row = tt.row[num];
    const int s0 = tt.ls[K][d], e0 = s0 + n;
    const uintptr_t lo = (uintptr_t)(row + s0), hi = lo + n;
    const uintptr_t hend = ((lo + 15) & ~(uintptr_t)15) < hi ? ((lo + 15) & ~(uintptr_t)15) : hi;
    const uintptr_t tbeg = (hi & ~(uintptr_t)15) > hend ? (hi & ~(uintptr_t)15) : hend;
    const int hlen = (int)(hend - lo), tlen = (int)(hi - tbeg);
    const int pos = lane < 16 ? s0 + lane : (int)(tbeg - (uintptr_t)row) + (lane - 16);
    if ((lane < 16 && lane < hlen) || (lane >= 16 && lane - 16 < tlen)) {
      const uint32_t x = fin[pos];
      row[pos] = (uint8_t)(x & keep);
      const uint32_t cb = (uint32_t)(num << 1) << nK;
      atomicAdd(s_ncnt + (cb | (pos >= tt.thr[num] ? (1u << nK) : 0u) | ((x >> nshift) & nmask)), 1u);
    }
    (void)e0;
  }
}

// Byte variant (all passes of byte alphabets): SIMD within a register.  Thread
// t owns the two 8-symbol halves [8t, 8t+8) and [T/2 + 8t, T/2 + 8t + 8) of
// the tile-local order (two 64-bit shared loads).  A split sorts each half in
// registers by the split bit with two byte permutes (PRMT selectors from a
// 256-entry shared table indexed by the half's 8-bit mask), so the half's
// zeros and ones become two contiguous byte runs; the CTA prefix of both
// halves comes from one packed warp-shuffle scan, and byte k of a sorted half
// is stored once, to the zeros run when k < (number of zeros), else to the
// ones run -- no per-symbol rank extraction.  The last split of a pass with
// output scatters symbol by symbol to HBM.
template <int K>
struct U8Smem {
  static constexpr int T = U8_THREADS * 16;
  // two staging buffers (tile i in stage i % 2, the next tile prefetched into
  // the other) + the orders of levels l+1 .. l+K-1
  // + one buffer for the last split (so stage buffers only ever receive bulk copies)
  static constexpr size_t buf_bytes = (size_t)(K + 1 + U8_FINAL_BUF) * T;
  static constexpr size_t bits_bytes = PassSmem<uint8_t, K, 16, U8_THREADS>::bits_bytes;
  static constexpr size_t total = buf_bytes + bits_bytes;
};

constexpr int U8_TABW = U8_TABLE_WARP ? TAB_WARP_THREADS : 0;

template <int K>
__global__ void __launch_bounds__(U8_THREADS + U8_TABW, U8_CTAS_PER_SM) level_pass_u8_kernel(const PassArgs a) {
  using S = U8Smem<K>;
  constexpr int T = S::T;
  constexpr int H = T / 2;
  constexpr int NC = T / 32;
  constexpr int NW = U8_THREADS / 32;
  constexpr int ALLT = U8_THREADS + U8_TABW;
  constexpr int nd = 1 << K;
  constexpr uint32_t B1 = 0x01010101u;
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + S::buf_bytes);

  __shared__ TileTables<uint8_t, K> tt;
  __shared__ __align__(16) uint32_t s_wtot[2][NW];
  __shared__ uint32_t s_ncnt[2 * NDIG * NDIG];
  __shared__ uint32_t s_lut[256];  // PRMT selectors: zeros of the 8-bit mask first, then ones
  __shared__ __align__(8) uint64_t s_mbar[2];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int w = a.width, l0 = a.level;
  const bool wm = a.kind == WVLT_KIND_WM;
  const int64_t G = gridDim.x;
  const uint8_t* text = reinterpret_cast<const uint8_t*>(a.src);
  const bool bulk_ok = (((uintptr_t)text) & 15) == 0;  // full tiles are then 16-byte aligned

  if (U8_TABLE_WARP && wid == NW) {  // table warp: one tile after the other, in step with the compute warps
    int i = 0;
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += G, ++i) {
      if (i) bar_sync(4, ALLT);  // previous tile's tables consumed
      const int cnt = (int)min((int64_t)T, a.n - tile * T);
      table_warp<uint8_t, uint8_t, K>(a, tt, smem + (i & 1) * T, tile, cnt, lane, ALLT);
    }
    return;
  }

  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t mbar0 = (uint32_t)__cvta_generic_to_shared(&s_mbar[0]);
  uint8_t* bits8 = reinterpret_cast<uint8_t*>(bits);
  for (int i = tid; i < 2 * NDIG * NDIG; i += U8_THREADS) s_ncnt[i] = 0;
  for (int i = tid; i < 256; i += U8_THREADS) s_lut[i] = g_sort_lut.sel[i];
  if (tid == 0) {
    mbar_init(mbar0, 1);
    mbar_init(mbar0 + 8, 1);
    fence_mbar_init();
    if (bulk_ok && (int64_t)blockIdx.x * T + T <= a.n)
      bulk_load(sbase, text + (int64_t)blockIdx.x * T, T, mbar0);
  }
  bar_sync(1, U8_THREADS);

  int i = 0;
#pragma unroll 1
  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += G, ++i) {
    const int st = i & 1;
    const int64_t base = tile * T;
    const int cnt = (int)min((int64_t)T, a.n - base);
    uint8_t* stage = smem + st * T;
    // prefetch the next tile into the other stage buffer (its previous tile is done)
    if (tid == 0 && bulk_ok && tile + G < a.ntiles && (tile + G) * T + T <= a.n)
      bulk_load(sbase + (st ^ 1) * T, text + (tile + G) * T, T, mbar0 + 8 * (st ^ 1));
    // ---- this tile (invalid tail slots = all ones so they sort last) ----
    if (bulk_ok && cnt == T) {
      mbar_wait(mbar0 + 8 * st, (uint32_t)(i >> 1) & 1u);
    } else {
      for (int p = tid; p < T; p += U8_THREADS) stage[p] = p < cnt ? text[base + p] : (uint8_t)0xFF;
      bar_sync(1, U8_THREADS);
    }
    if (U8_TABLE_WARP) {
      if (!wm) bar_arrive(3, ALLT);
    } else if (wid == NW - 1) {
      // tables by the last compute warp (visible to all after the next CTA barrier)
      table_warp<uint8_t, uint8_t, K>(a, tt, stage, tile, cnt, lane, 0);
    }

#pragma unroll  // constant j: buffer and scan addresses fold (32 registers at 3 CTAs/SM)
    for (int j = 0; j < K; ++j) {
      const int sh = w - 1 - l0 - j;
      const uint8_t* cur = j ? smem + (size_t)(j + 1) * T : stage;
      const uint2 q0 = reinterpret_cast<const uint2*>(cur)[tid];
      const uint2 q1 = reinterpret_cast<const uint2*>(cur + H)[tid];
      const uint32_t x[4] = {q0.x, q0.y, q1.x, q1.y};
      uint32_t b[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) b[k] = (x[k] >> sh) & B1;
      // this thread's level bits: byte t (first half) and byte T/16 + t (second half)
      // one multiply gathers a half's 8 flags (bits at 8i and 8i + 4 -> 24 + i, 28 + i)
      const uint32_t m0 = ((b[1] * 16u + b[0]) * 0x01020408u) >> 24;
      const uint32_t m1 = ((b[3] * 16u + b[2]) * 0x01020408u) >> 24;
      const uint32_t ones0 = __popc(m0), ones1 = __popc(m1);
      if (j == 0) {
        // level l0 is in global order already: byte stores (32 lanes = 32 consecutive bytes)
        uint8_t* g8 = reinterpret_cast<uint8_t*>(a.words + (int64_t)l0 * a.nwords) + (base >> 3);
        const int64_t lim = 8 * a.nwords - (base >> 3);
        const int f0 = 8 * tid, f1 = H + 8 * tid;
        if (tid < lim) g8[tid] = (uint8_t)(f0 + 8 <= cnt ? m0 : (f0 >= cnt ? 0u : (m0 & ((1u << (cnt - f0)) - 1u))));
        if (H / 8 + tid < lim)
          g8[H / 8 + tid] = (uint8_t)(f1 + 8 <= cnt ? m1 : (f1 >= cnt ? 0u : (m1 & ((1u << (cnt - f1)) - 1u))));
      } else {
        bits8[j * 4 * (NC + 4) + tid] = (uint8_t)m0;
        bits8[j * 4 * (NC + 4) + H / 8 + tid] = (uint8_t)m1;
      }
      if (j + 1 == K && !a.has_out) break;
      // CTA-wide exclusive scans of both halves' ones counts (packed 16|16)
      const uint32_t pk = ones0 | (ones1 << 16);
      const uint32_t incl = warp_incl_scan(pk);
      if (lane == 31) s_wtot[j & 1][wid] = incl;
      bar_sync(1, U8_THREADS);
      const uint32_t wv = lane < NW ? s_wtot[j & 1][lane] : 0u;
      const uint32_t wpre = __reduce_add_sync(FULL, lane < wid ? wv : 0u);
      const uint32_t tot = __reduce_add_sync(FULL, wv);
      const uint32_t ex = wpre + incl - pk;
      const int tot0 = (int)(tot & 0xFFFFu), tot1 = (int)(tot >> 16);
      const int Z = T - tot0 - tot1;
      const int opre0 = (int)(ex & 0xFFFFu);
      const int opre1 = tot0 + (int)(ex >> 16);
      // ones: OBh + (inclusive rank); zeros: ZBh + symbol index - (inclusive ones)
      const int OB[2] = {Z + opre0 - 1, Z + opre1 - 1};
      const int ZB[2] = {8 * tid - opre0, H + 8 * tid - opre1};
      const bool last = j + 1 == K;
      bool in_smem = !last;
      if (last) {
        if (U8_TABLE_WARP) bar_sync(2, ALLT);  // placement tables
        in_smem = tt.q1;
      }
      if (in_smem) {
        // the last split of a uniform tile goes to buffer K + 1 and is copied
        // out run by run
        const uint32_t nxt = sbase + (uint32_t)(last && !U8_FINAL_BUF ? st : j + 2) * T;
        // each half sorted in registers (zeros first): byte k goes to the zeros
        // run (k < nz) or to the ones run, one store per symbol
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t sel = s_lut[hh ? m1 : m0];  // prmt reads selector bits 0-15
          const uint32_t sv[2] = {prmt(x[2 * hh], x[2 * hh + 1], sel), prmt(x[2 * hh], x[2 * hh + 1], sel >> 16)};
          const int nz = 8 - (int)(hh ? ones1 : ones0);
          const uint32_t za = opaque(nxt + (uint32_t)ZB[hh]);
          const uint32_t oa = opaque(nxt + (uint32_t)(OB[hh] + 1 - nz));
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t v = sv[kk >> 2];
            const uint32_t vb = (kk & 3) == 0 ? v : (kk & 3) == 1 ? shr_mul<8>(v) : (kk & 3) == 2 ? shr_mul<16>(v) : shr_mul<24>(v);
            // (measured: predicated dual stores and a flag-table IMAD address are
            // both slower than this compare + select)
            const uint32_t addr = (kk < nz ? za : oa) + kk;
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(vb) : "memory");
          }
        }
        bar_sync(1, U8_THREADS);
        if (last) {
          copy_out_u8<K>(a, tt, U8_FINAL_BUF ? smem + (size_t)(K + 1) * T : stage, s_ncnt, tid);
          bar_sync(1, U8_THREADS);
          const int ncount = 2 * nd << a.nK;
          const unsigned nmask = (1u << a.nK) - 1u;
          for (int q = tid; q < ncount; q += U8_THREADS) {
            const uint32_t v = s_ncnt[q];
            if (v) {
              s_ncnt[q] = 0;
              const int slot = q >> a.nK, ne = q & (int)nmask;
              atomicAdd(&a.ncnt[(int64_t)ne * a.nntiles + tt.ft[slot >> 1] + (slot & 1)], v);
            }
          }
        }
      } else {
        // last split of a tile spanning several nodes (WT): symbol by symbol to HBM
        const uint32_t keep = wm ? ((w - l0 - K) >= 32 ? FULL : ((1u << (w - l0 - K)) - 1u)) : FULL;
        const int eshift = w - l0 - K;
        const int nshift = w - l0 - K - a.nK;
        const unsigned nmask = (1u << a.nK) - 1u;
        uint32_t p[4];  // inclusive ones count through each byte, per half
        p[0] = b[0] * B1;
        p[1] = (b[1] + (p[0] >> 24)) * B1;
        p[2] = b[2] * B1;
        p[3] = (b[3] + (p[2] >> 24)) * B1;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = (int)__byte_perm(p[k], 0, 0x4440 + e);
            const uint32_t xv = __byte_perm(x[k], 0, 0x4440 + e);
            const int pos = (b[k] & (0xFFu << (8 * e))) ? OB[k >> 1] + r : ZB[k >> 1] + 4 * (k & 1) + e - r;
            if (pos < cnt) {
              const unsigned d = rev_bits((xv >> eshift) & (nd - 1), K);
              const uint64_t P = (uint64_t)xv >> eshift;
              const int64_t gpos = a.corr[a.corr_off[K] + P] + tt.lb[K][d] + pos - tt.ls[K][d];
              reinterpret_cast<uint8_t*>(a.dst)[gpos] = (uint8_t)(xv & keep);
              atomicAdd(&a.ncnt[(int64_t)((xv >> nshift) & nmask) * a.nntiles + (gpos >> a.ntshift)], 1u);
            }
          }
        }
        bar_sync(1, U8_THREADS);
      }
    }
    if (!a.has_out) {
      bar_sync(1, U8_THREADS);
      if (U8_TABLE_WARP) bar_sync(2, ALLT);
    }
    if (tt.q1)
      emit_uniform<uint8_t, K, NC>(a, tt, bits, wid, lane, NW);
    else
      emit_multinode<uint8_t, uint8_t, K>(a, tt, smem + T, T, cnt, tid, lane, U8_THREADS);
    // stage buffers are only read here (no generic writes except for the
    // final partial tile, after which no bulk copy targets them)
    bar_sync(1, U8_THREADS);
    if (U8_TABLE_WARP && tile + G < a.ntiles) bar_arrive(4, ALLT);
  }
}

// ---------------------------------------------------------------------------
// K5: merge (gather_bits)
// ---------------------------------------------------------------------------
// The task holding bit `here`, forward from task t whose end bounds[t + 1] <= here.
// Pieces are usually longer than a word and a lane's next word is a few pieces on:
// a linear walk.  `sparse` plans (many more pieces than destination words: the 2^l
// groups of a wide alphabet over a few thousand words, nearly all empty) first look
// 64 pieces ahead and binary-search from there.  bounds[ntasks] > here.
__device__ __forceinline__ int64_t advance_task(const int64_t* __restrict__ bounds, int64_t t, int64_t ntasks,
                                                int64_t here, bool sparse, int64_t* end = nullptr) {
  if (sparse) {
    const int64_t far = min(t + 64, ntasks);
    if (__ldg(bounds + far) <= here) {
      int64_t lo = far, hi = ntasks;  // bounds[lo] <= here < bounds[hi]
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(bounds + mid) <= here) lo = mid;
        else hi = mid;
      }
      if (end) *end = __ldg(bounds + lo + 1);
      return lo;
    }
  }
  int64_t b1;
  do b1 = __ldg(bounds + (++t) + 1);
  while (b1 <= here);
  if (end) *end = b1;
  return t;
}

// many more pieces than destination words: long stretches of empty pieces
__device__ __forceinline__ bool merge_sparse(int64_t ntasks, int64_t nwords) { return ntasks > 8 * nwords; }

// destination word wd of a gather_bits plan, walking forward from task t
__device__ __forceinline__ uint64_t merge_word(int64_t wd, int64_t nbits, const int64_t* __restrict__ bounds,
                                               const int64_t* __restrict__ src_starts,
                                               const uint64_t* __restrict__ src, int64_t t, int64_t ntasks, bool sparse) {
  const int64_t wb = wd << 6;
  int64_t nb = nbits - wb;
  if (nb > 64) nb = 64;
  uint64_t acc = 0;
  int filled = 0;
  while (filled < nb) {
    const int64_t here = wb + filled;
    if (__ldg(bounds + t + 1) <= here) t = advance_task(bounds, t, ntasks, here, sparse);
    int64_t take = nb - filled;
    const int64_t avail = __ldg(bounds + t + 1) - here;
    if (avail < take) take = avail;
    const int64_t sp = __ldg(src_starts + t) + (here - __ldg(bounds + t));
    const int64_t wi = sp >> 6;
    const int sh = (int)(sp & 63);
    uint64_t chunk = __ldcs(reinterpret_cast<const unsigned long long*>(src) + wi) >> sh;
    if (sh + take > 64) chunk |= __ldcs(reinterpret_cast<const unsigned long long*>(src) + wi + 1) << (64 - sh);
    if (take < 64) chunk &= (1ull << take) - 1ull;
    acc |= chunk << filled;
    filled += (int)take;
  }
  return acc;
}

#ifndef MERGE_WPL
#define MERGE_WPL 8  // measured: 8 < 4 ms (more source loads in flight)
#endif
constexpr int MERGE_WORDS_PER_LANE = MERGE_WPL;

// destination words [wlo, whi) of one gather_bits plan; warp `gw` of `nwarps`
// PEER: task t's source is rank ranks[t]'s level (srcs[ranks[t]]) instead of `src`
// (merge_word_peer is defined below)
__device__ __forceinline__ uint64_t merge_word_peer(int64_t wd, int64_t nbits, const int64_t* __restrict__ bounds,
                                                    const int64_t* __restrict__ starts,
                                                    const int32_t* __restrict__ ranks,
                                                    const uint64_t* const* __restrict__ srcs, int64_t t,
                                                    int64_t ntasks, bool sparse);
template <bool PEER, bool SPARSE>
__device__ __forceinline__ void merge_range(uint64_t* __restrict__ dst, int64_t wlo, int64_t whi, int64_t nbits,
                                            const int64_t* __restrict__ bounds,
                                            const int64_t* __restrict__ src_starts, int64_t ntasks,
                                            const uint64_t* __restrict__ src, const int32_t* __restrict__ ranks,
                                            const uint64_t* const* __restrict__ srcs, int64_t gw, int64_t nwarps) {
  // a warp owns 32 * MERGE_WORDS_PER_LANE consecutive destination words
  // (coalesced stores; within a task coalesced source loads); lane 0
  // binary-searches the task of the warp's first bit, every lane walks forward
  constexpr int CH = 32 * MERGE_WORDS_PER_LANE;
  const int lane = threadIdx.x & 31;
  constexpr bool sparse = SPARSE;  // (see advance_task; chosen per launch by merge_sparse)
  for (int64_t w0 = wlo + gw * CH; w0 < whi; w0 += nwarps * CH) {
    int64_t t0 = 0;
    if (lane == 0 && (w0 << 6) < nbits) {
      int64_t lo = 0, hi = ntasks;  // last t with bounds[t] <= bit
      const int64_t bit = w0 << 6;
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(bounds + mid) <= bit) lo = mid;
        else hi = mid;
      }
      t0 = lo;
    }
    t0 = __shfl_sync(FULL, t0, 0);
    uint64_t v[MERGE_WORDS_PER_LANE];
    // the task of every word's first bit first, then all source loads at once
    // (independent, in flight together), then the words that straddle a task
    // boundary on the slow path.  The current task's bounds, source start and
    // source level stay in registers: a lane's words are 2048 bits apart and
    // mostly fall into the same piece, so the small plan arrays are read only
    // when the task changes (no dependent lookups in front of the source loads).
    const unsigned long long* pw[MERGE_WORDS_PER_LANE];  // first source word of a one-piece destination word
    int shnb[MERGE_WORDS_PER_LANE];                      // its shift | (bits << 8); -1 - (t - t0): slow path from task t
    int64_t t = t0;
    int64_t b0 = 0, b1 = 0, st = 0;
    const unsigned long long* sbase = reinterpret_cast<const unsigned long long*>(src);
    bool have = false;
#pragma unroll
    for (int k = 0; k < MERGE_WORDS_PER_LANE; ++k) {
      const int64_t wd = w0 + 32 * k + lane;
      const int64_t here = wd << 6;
      pw[k] = nullptr;
      shnb[k] = 0;
      if (wd < whi && here < nbits) {
        if (!have || b1 <= here) {
          if (!have) b1 = __ldg(bounds + t + 1);
          if (b1 <= here) {
            t = advance_task(bounds, t, ntasks, here, sparse, &b1);
          }
          b0 = __ldg(bounds + t);
          st = __ldg(src_starts + t);
          if (PEER) sbase = reinterpret_cast<const unsigned long long*>(srcs[__ldg(ranks + t)]);
          have = true;
        }
        const int64_t nb = min((int64_t)64, nbits - here);
        if (b1 >= here + nb) {
          const int64_t pos = st + (here - b0);
          pw[k] = sbase + (pos >> 6);
          shnb[k] = (int)(pos & 63) | ((int)nb << 8);
        } else {
          shnb[k] = -1 - (int)(t - t0);
        }
      }
    }
    uint64_t lo[MERGE_WORDS_PER_LANE], hi[MERGE_WORDS_PER_LANE];
#pragma unroll
    for (int k = 0; k < MERGE_WORDS_PER_LANE; ++k) {
      lo[k] = hi[k] = 0;
      if (pw[k]) {
        // the next source word only when the bits run into it (never past the source's end);
        // peer memory: plain loads (written by another device before the collective)
        lo[k] = PEER ? pw[k][0] : __ldg(pw[k]);
        if ((shnb[k] & 63) + (shnb[k] >> 8) > 64) hi[k] = PEER ? pw[k][1] : __ldg(pw[k] + 1);
      }
    }
#pragma unroll
    for (int k = 0; k < MERGE_WORDS_PER_LANE; ++k) {
      const int64_t wd = w0 + 32 * k + lane;
      if (pw[k]) {
        const int sh = shnb[k] & 63, nbk = shnb[k] >> 8;
        uint64_t x = sh ? ((lo[k] >> sh) | (hi[k] << (64 - sh))) : lo[k];
        if (nbk < 64) x &= (1ull << nbk) - 1ull;
        v[k] = x;
      } else if (shnb[k] < 0) {
        const int64_t tk = t0 + (int64_t)(-1 - shnb[k]);
        v[k] = PEER ? merge_word_peer(wd, nbits, bounds, src_starts, ranks, srcs, tk, ntasks, sparse)
                    : merge_word(wd, nbits, bounds, src_starts, src, tk, ntasks, sparse);
      } else {
        v[k] = 0ull;
      }
    }
#pragma unroll
    for (int k = 0; k < MERGE_WORDS_PER_LANE; ++k) {
      const int64_t wd = w0 + 32 * k + lane;
      if (wd < whi) __stcs(reinterpret_cast<unsigned long long*>(dst) + wd, v[k]);
    }
  }
}

__global__ void __launch_bounds__(256) merge_bits_kernel(uint64_t* __restrict__ dst, int64_t wlo, int64_t whi,
                                                         int64_t nbits, const int64_t* __restrict__ bounds,
                                                         const int64_t* __restrict__ src_starts, int64_t ntasks,
                                                         const uint64_t* __restrict__ src) {
  const int64_t gw = (((int64_t)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5);
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (merge_sparse(ntasks, whi - wlo))
    merge_range<false, true>(dst, wlo, whi, nbits, bounds, src_starts, ntasks, src, nullptr, nullptr, gw, nwarps);
  else
    merge_range<false, false>(dst, wlo, whi, nbits, bounds, src_starts, ntasks, src, nullptr, nullptr, gw, nwarps);
}

// Multi-GPU merge over peer memory: every level's owned destination words are
// assembled straight from the source ranks' local levels (P2P / symmetric-memory
// pointers over NVLink), so the exchange and the shift-merge are one kernel.
// Task t of level l: destination bits [bounds[t], bounds[t+1]) come from rank
// ranks[t]'s local level l starting at bit starts[t].
__device__ __forceinline__ uint64_t merge_word_peer(int64_t wd, int64_t nbits, const int64_t* __restrict__ bounds,
                                                    const int64_t* __restrict__ starts,
                                                    const int32_t* __restrict__ ranks,
                                                    const uint64_t* const* __restrict__ srcs, int64_t t,
                                                    int64_t ntasks, bool sparse) {
  const int64_t wb = wd << 6;
  int64_t nb = nbits - wb;
  if (nb > 64) nb = 64;
  uint64_t acc = 0;
  int filled = 0;
  while (filled < nb) {
    const int64_t here = wb + filled;
    if (__ldg(bounds + t + 1) <= here) t = advance_task(bounds, t, ntasks, here, sparse);
    int64_t take = nb - filled;
    const int64_t avail = __ldg(bounds + t + 1) - here;
    if (avail < take) take = avail;
    const int64_t sp = __ldg(starts + t) + (here - __ldg(bounds + t));
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(srcs[__ldg(ranks + t)]);
    const int64_t wi = sp >> 6;
    const int sh = (int)(sp & 63);
    uint64_t chunk = src[wi] >> sh;
    if (sh + take > 64) chunk |= src[wi + 1] << (64 - sh);
    if (take < 64) chunk &= (1ull << take) - 1ull;
    acc |= chunk << filled;
    filled += (int)take;
  }
  return acc;
}

__global__ void __launch_bounds__(256) merge_peer_kernel(uint64_t* __restrict__ dst, int64_t dst_row, int64_t wlo,
                                                         int64_t whi, int64_t nbits,
                                                         const int64_t* __restrict__ bounds_all,
                                                         const int64_t* __restrict__ bounds_off,
                                                         const int64_t* __restrict__ starts_all,
                                                         const int32_t* __restrict__ ranks_all,
                                                         const int64_t* __restrict__ task_off,
                                                         const uint64_t* const* __restrict__ level_src, int nranks) {
  const int l = blockIdx.y;
  const int64_t t_lo = task_off[l], ntasks = task_off[l + 1] - t_lo;
  if (ntasks <= 0) return;
  // the same word loop as the one-source merge: every word's task first, then
  // all of a lane's source loads in flight together (peer reads over NVLink
  // have a few microseconds of latency), words that straddle pieces last
  const int64_t gw = (((int64_t)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5);
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t* drow = dst + (int64_t)l * dst_row - wlo;
  if (merge_sparse(ntasks, whi - wlo))
    merge_range<true, true>(drow, wlo, whi, nbits, bounds_all + bounds_off[l], starts_all + t_lo, ntasks, nullptr,
                            ranks_all + t_lo, level_src + (int64_t)l * nranks, gw, nwarps);
  else
    merge_range<true, false>(drow, wlo, whi, nbits, bounds_all + bounds_off[l], starts_all + t_lo, ntasks, nullptr,
                             ranks_all + t_lo, level_src + (int64_t)l * nranks, gw, nwarps);
}

// Merge plan of the sharded build on the device (construct._merge_plan,
// construct.py:516-543, for every level at once): level l's pieces are the
// (group q in interval order, rank r) pairs, group-major -- R 2^l tasks, empty
// ones kept (the merge kernels skip them).  Everything is elementwise given
// every rank's node borders B_r (its local group starts, indexed by prefix):
// a piece's source start is B_r(P), its length B_r(P') - B_r(P) (P' the next
// group in interval order; the rank's symbol count after the last), and its
// destination start sum_r' B_r'(P) + the lengths of the lower ranks' pieces of
// the group.  Level 0 is one group.  One thread per (level, group).
__global__ void peer_plan_kernel(const int64_t* __restrict__ rows, int64_t row_stride, int64_t borders_col,
                                 const int64_t* __restrict__ local_ns, int R, int w, int kind,
                                 int64_t* __restrict__ bounds, int64_t* __restrict__ starts,
                                 int32_t* __restrict__ ranks, int64_t* __restrict__ bounds_off,
                                 int64_t* __restrict__ task_off) {
  const int64_t items = (1ll << w) - 1;  // sum over levels of 2^l
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gtid <= w) {  // closed-form offsets: level l has R 2^l tasks and R 2^l + 1 bounds
    task_off[gtid] = (int64_t)R * ((1ll << gtid) - 1);
    if (gtid < w) bounds_off[gtid] = (int64_t)R * ((1ll << gtid) - 1) + gtid;
  }
  for (int64_t i = gtid; i < items; i += (int64_t)gridDim.x * blockDim.x) {
    const int l = 63 - __clzll(i + 1);
    const int64_t q = i + 1 - (1ll << l);
    const int64_t ng = 1ll << l;
    const bool last = q + 1 == ng;
    const bool rev = kind == WVLT_KIND_WM && l >= 2;
    const int64_t P = rev ? (int64_t)rev_bits((unsigned)q, l) : q;
    const int64_t Pn = last ? 0 : (rev ? (int64_t)rev_bits((unsigned)(q + 1), l) : q + 1);
    int64_t g = 0;
    for (int r = 0; r < R; ++r) g += l ? rows[r * row_stride + borders_col + (1ll << l) - 2 + P] : 0;
    int64_t* bl = bounds + (int64_t)R * ((1ll << l) - 1) + l;
    int64_t* sl = starts + (int64_t)R * ((1ll << l) - 1);
    int32_t* rl = ranks + (int64_t)R * ((1ll << l) - 1);
    int64_t run = g;
    for (int r = 0; r < R; ++r) {
      const int64_t* br = rows + r * row_stride + borders_col + (1ll << l) - 2;
      const int64_t st = l ? br[P] : 0;
      const int64_t en = (l && !last) ? br[Pn] : local_ns[r];
      bl[q * R + r] = run;
      sl[q * R + r] = st;
      rl[q * R + r] = r;
      run += en - st;
    }
    if (last) bl[(int64_t)R * ng] = run;  // = n
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

int tile_for(int in_bytes) { return in_bytes == 4 ? PASS_THREADS * 8 : (in_bytes == 1 ? TILE_U8 : PASS_THREADS * E_SMALL); }
int log2i(int v) {
  int r = 0;
  while ((1 << r) < v) ++r;
  return r;
}

size_t k8_workspace_total(int64_t n, int w);   // k8.cuh
size_t k16_workspace_total(int64_t n, int w);  // k16.cuh
size_t k32_workspace_total(int64_t n, int w);  // k32.cuh

// lean: a WM build without histogram / borders (the fused 2-byte pass needs it)
bool make_plan(int64_t n, int sym_bytes, int64_t sigma, int kind, Plan* P, bool lean = true) {
  memset(P, 0, sizeof(*P));
  const int w = code_width_host(sigma);
  P->width = w;
  P->kind = kind;
  if (w > WVLT_MAX_WIDTH) return false;
  // symbols stored narrower than the code width are widened first (the tail
  // sentinel of the pass kernel must set every code bit)
  int sb = sym_bytes;
  if (8 * sym_bytes < w) {
    P->widen_bytes = bytes_for_bits(w);
    sb = P->widen_bytes;
  }
  int l = 0, p = 0;
  int64_t corr = 0;
  size_t max_buf = 0;
  const bool tail = kind == WVLT_KIND_WM && w > 8 && n > 0 && n < (1ll << 32) - 64;
  const bool k16 = tail && lean;
  int cur_bytes = sb;  // element bytes of the next stage's input
  while (l < w && !(tail && w - l <= 8)) {
    if (k16 && !P->k32_w && w - l <= 24 && w - l >= 18 && cur_bytes == 4) {
      P->k32_w = w - l - 16;
      P->k32_lvl = l;
      l += P->k32_w;
      cur_bytes = 2;
      continue;
    }
    if (k16 && w - l <= 16 && w - l >= 10 && cur_bytes == 2) {
      P->k16_w = w - l - 8;
      P->k16_lvl = l;
      l += P->k16_w;
      break;
    }
    if (P->k32_w) break;  // (not reached: the 4-byte pass leaves exactly 16 live bits)
    const int K = (w - l) < KMAX ? (w - l) : KMAX;
    P->lvl[p] = l;
    P->K[p] = K;
    const int live_in = kind == WVLT_KIND_WM ? (w - l) : w;
    const int live_out = kind == WVLT_KIND_WM ? (w - l - K) : w;
    P->in_bytes[p] = p == 0 ? sb : bytes_for_bits(live_in);
    P->out_bytes[p] = (l + K < w) ? bytes_for_bits(live_out) : 0;
    if (P->out_bytes[p] > P->in_bytes[p]) P->out_bytes[p] = P->in_bytes[p];
    P->tile[p] = tile_for(P->in_bytes[p]);
    P->tshift[p] = log2i(P->tile[p]);
    P->ntiles[p] = (n + P->tile[p] - 1) / P->tile[p];
    if ((size_t)P->out_bytes[p] * (size_t)n > max_buf) max_buf = (size_t)P->out_bytes[p] * (size_t)n;
    if (kind == WVLT_KIND_WT) {
      for (int j = 1; j <= K; ++j) {
        P->corr_off[p][j] = corr;
        corr += 1ll << (l + j);
      }
    }
    cur_bytes = P->out_bytes[p];
    l += K;
    ++p;
  }
  P->npass = p;
  P->corr_total = corr;
  if (tail) {
    P->tail_w = w - l;
    P->tail_lvl = l;
  }
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
  P->off_scratch = off;  // scratch status word
  off = align_up(off + 64, 256);
  const size_t tcnt_start = off;
  int64_t max_nblk = 1;
  for (int q = 0; q < P->npass; ++q) {
    P->off_tcnt[q] = off;
    off = align_up(off + (size_t)(1 << P->K[q]) * P->ntiles[q] * 4, 256);
    const int64_t nblk = (P->ntiles[q] + SCAN_TILE - 1) / SCAN_TILE;
    if (nblk > max_nblk) max_nblk = nblk;
  }
  P->tcnt_bytes = off - tcnt_start;
  for (int q = 0; q < P->npass; ++q) {
    P->off_tpre[q] = off;
    off = align_up(off + (size_t)(1 << P->K[q]) * P->ntiles[q] * 8, 256);
  }
  P->off_bsum = off;
  off = align_up(off + (size_t)NDIG * max_nblk * 8, 256);
  if (tail) max_buf = std::max(max_buf, k8_workspace_total(n, P->tail_w));
  if (P->k16_w) max_buf = std::max(max_buf, align_up((size_t)n, 256) + k16_workspace_total(n, P->k16_w));
  if (P->k32_w) max_buf = std::max(max_buf, align_up((size_t)n * 2, 256) + k32_workspace_total(n, P->k32_w));
  P->buf_bytes = align_up(max_buf ? max_buf : 16, 256);
  P->off_buf0 = off;
  off += P->buf_bytes;
  P->off_buf1 = off;
  off += P->buf_bytes;
  P->off_wide = off;
  if (P->widen_bytes) off += align_up((size_t)n * P->widen_bytes, 256);
  P->total = off;
  return true;
}

int sm_count();

// Once per (kernel, device): the dynamic shared-memory limit above 48 KB (and
// optionally the max-shared carveout).  Function attributes are per device, so
// a process driving several GPUs sets them on each.
cudaError_t ensure_smem_attr(const void* fn, int bytes, bool carveout = false) {
  static std::mutex mu;
  static std::unordered_map<const void*, uint64_t> done;  // device bitmask per kernel
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  uint64_t& mask = done[fn];
  if ((mask >> (dev & 63)) & 1) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  if (carveout) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
  }
  mask |= 1ull << (dev & 63);
  return cudaSuccess;
}

template <typename TIn, typename TOut, int K>
cudaError_t launch_pass_t(const PassArgs& a, int64_t ntiles, cudaStream_t s) {
  constexpr int E = sizeof(TIn) == 4 ? 8 : E_SMALL;
  using S = PassSmem<TIn, K, E>;
  auto kern = level_pass_kernel<TIn, TOut, K, E>;
  cudaError_t e = ensure_smem_attr((const void*)kern, (int)S::total);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)ntiles, PASS_THREADS + TAB_WARP_THREADS, S::total, s>>>(a);
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

int sm_count();

template <int K>
cudaError_t launch_pass_u8(const PassArgs& a, int64_t ntiles, cudaStream_t s) {
  using S = U8Smem<K>;
  auto kern = level_pass_u8_kernel<K>;
  cudaError_t e = ensure_smem_attr((const void*)kern, (int)S::total, true);
  if (e != cudaSuccess) return e;
  // persistent CTAs: U8_CTAS_PER_SM per SM, tiles strided by the grid
#ifndef U8_GRID_PER_SM
#define U8_GRID_PER_SM 0  // 0: one CTA per tile (measured faster than persistent CTAs)
#endif
  const int64_t grid = U8_GRID_PER_SM ? std::min<int64_t>(ntiles, (int64_t)sm_count() * U8_GRID_PER_SM) : ntiles;
  kern<<<(unsigned)grid, U8_THREADS + U8_TABW, S::total, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pass(int in_bytes, int out_bytes, int K, const PassArgs& a, int64_t ntiles, cudaStream_t s) {
  const int ob = out_bytes ? out_bytes : in_bytes;
  if (in_bytes == 1) {
    switch (K) {
      case 1: return launch_pass_u8<1>(a, ntiles, s);
      case 2: return launch_pass_u8<2>(a, ntiles, s);
      case 3: return launch_pass_u8<3>(a, ntiles, s);
      default: return launch_pass_u8<4>(a, ntiles, s);
    }
  }
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

// Generic full histogram (wide symbols / alphabets) or the range check alone (hist == null).
cudaError_t launch_hist_generic(const void* text, int sym_bytes, int64_t n, int w, unsigned long long* hist,
                                int32_t* status, cudaStream_t s) {
  const int sw = w < 16 ? w : 16;
  const size_t sb = (size_t)((((1 << sw) + 1) >> 1)) * 4;
  const int per_sm = sb > 100 * 1024 ? 1 : 2;
  const int blocks = sm_count() * per_sm;
#define WVLT_HG(T)                                                                                          \
  do {                                                                                                      \
    ensure_smem_attr((const void*)hist_generic_kernel<T>, 128 * 1024);                                      \
    hist_generic_kernel<T><<<blocks, HISTG_THREADS, sb, s>>>((const T*)text, n, w, hist, status);          \
  } while (0)
  if (sym_bytes == 1) WVLT_HG(uint8_t);
  else if (sym_bytes == 2) WVLT_HG(uint16_t);
  else WVLT_HG(uint32_t);
#undef WVLT_HG
  return cudaGetLastError();
}

// K1 for a build: histogram of the text plus pass-0 tile digit counts.
cudaError_t launch_hist_build(const void* text, int sym_bytes, int64_t n, int w, int K0, int tile0, int64_t ntiles0,
                              unsigned long long* hist, uint32_t* tcnt0, int32_t* status, cudaStream_t s) {
  const bool fast = sym_bytes == 1 && w >= 1 && w <= 8 && tile0 == TILE_U8 && (((uintptr_t)text) & 15) == 0;
  if (fast) {
    const uint8_t* t = (const uint8_t*)text;
    const size_t sb = (size_t)HIST_WARPS * ((size_t)1 << (w - 1)) * 32 * 4;
    const int hb = sm_count() * (int)std::min<size_t>(8, (size_t)(220 * 1024) / (sb + 1024));
    const int dshift = w - K0;
    const int nd0 = 1 << K0;
#define WVLT_H8(WW)                                                                                         \
  do {                                                                                                      \
    ensure_smem_attr((const void*)hist_u8_kernel<WW>, (int)sb);                                             \
    hist_u8_kernel<WW><<<hb, HIST_WARPS * 32, sb, s>>>(t, n, dshift, nd0, hist, tcnt0, ntiles0, status);    \
  } while (0)
    switch (w) {
      case 1: WVLT_H8(1); break;
      case 2: WVLT_H8(2); break;
      case 3: WVLT_H8(3); break;
      case 4: WVLT_H8(4); break;
      case 5: WVLT_H8(5); break;
      case 6: WVLT_H8(6); break;
      case 7: WVLT_H8(7); break;
      default: WVLT_H8(8); break;
    }
#undef WVLT_H8
    return cudaGetLastError();
  }
  cudaError_t e = launch_hist_generic(text, sym_bytes, n, w, hist, status, s);
  if (e != cudaSuccess) return e;
  const int blocks = sm_count() * 8;
  digits_kernel<<<blocks, 256, 0, s>>>(text, sym_bytes, n, tile0, w - K0, 1 << K0, ntiles0, tcnt0);
  return cudaGetLastError();
}

// K1 of a lean WM build: pass-0 tile digit counts + range check.
cudaError_t launch_digits_fast(const void* text, int sym_bytes, int64_t n, int w, int64_t sigma, int K0, int tile0,
                               int64_t ntiles0, uint32_t* tcnt0, int32_t* status, cudaStream_t s) {
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((ntiles0 + 7) / 8, (int64_t)sm_count() * 8));
  const uint32_t vmax_ok = (uint32_t)std::min<int64_t>(sigma - 1, 0xFFFFFFFFll);
  const int dshift = w - K0;
  // every stored value is in range when sigma covers the whole storage type
  const bool check = sym_bytes == 4 ? vmax_ok < 0xFFFFFFFFu : vmax_ok < (1u << (8 * sym_bytes)) - 1u;
#define WVLT_DG(T)                                                                                           \
  do {                                                                                                       \
    if (check)                                                                                               \
      digits_fast_kernel<T, true><<<blocks, 256, 0, s>>>((const T*)text, n, tile0, dshift, 1 << K0, ntiles0, \
                                                         vmax_ok, tcnt0, status);                            \
    else                                                                                                     \
      digits_fast_kernel<T, false><<<blocks, 256, 0, s>>>((const T*)text, n, tile0, dshift, 1 << K0,         \
                                                          ntiles0, vmax_ok, tcnt0, status);                  \
  } while (0)
  if (sym_bytes == 1) WVLT_DG(uint8_t);
  else if (sym_bytes == 2) WVLT_DG(uint16_t);
  else WVLT_DG(uint32_t);
#undef WVLT_DG
  return cudaGetLastError();
}

cudaError_t launch_scan(const uint32_t* cnt, int K, int64_t ntiles, int64_t* bsum, int64_t* pre, cudaStream_t s) {
  const int64_t nblk = (ntiles + SCAN_TILE - 1) / SCAN_TILE;
  dim3 g((unsigned)nblk, 1u << K);
  scan_reduce_kernel<<<g, SCAN_THREADS, 0, s>>>(cnt, ntiles, nblk, bsum);
  scan_apply_kernel<<<g, SCAN_THREADS, 0, s>>>(cnt, ntiles, nblk, bsum, pre);
  return cudaGetLastError();
}

// kernels launched by the calling thread's last build (bench evidence)
thread_local int g_launches = 0;

// optional per-stage CUDA-event timing of wvlt_build_device (bench / profiling)
constexpr int PROF_MAX = 3 + 2 * MAXP + 1;
struct Prof {
  bool on = false;
  int n = 0;
  int ids[PROF_MAX];
  cudaEvent_t ev[PROF_MAX + 1];
  bool created = false;
};
thread_local Prof g_prof;

void prof_mark(cudaStream_t s, int stage_id) {
  Prof& P = g_prof;
  if (!P.on || P.n > PROF_MAX) return;
  if (!P.created) {
    for (int i = 0; i <= PROF_MAX; ++i) cudaEventCreate(&P.ev[i]);
    P.created = true;
  }
  if (stage_id >= 0 && P.n > 0) P.ids[P.n - 1] = stage_id;
  cudaEventRecord(P.ev[P.n], s);
  ++P.n;
}

}  // namespace

#include "k8.cuh"
#include "k16.cuh"
#include "k32.cuh"

namespace {
int build_device_impl(const void* text, int sym_bytes, int64_t n, int64_t sigma, int kind, uint64_t* level_words,
                      int64_t* zeros, int64_t* hist, int64_t* borders, void* workspace, size_t workspace_bytes,
                      int32_t* status, void* stream, void (*pass_done)(void*, int, int), void* ctx);
}
// ---------------------------------------------------------------------------
// WT of an alphabet wider than a byte: the WM levels (fused passes) reordered
// into tree order.  Both hold level l's bits grouped by l-bit prefix, the WM
// in bit-reversed prefix order, the WT in numeric order (structures.py:43-58,
// 176-182; the same fact wt2wm.py:205-227 uses the other way round), so every
// level is one gather_bits plan whose tasks are the prefix groups: destination
// bounds = WT interval starts, sources = WM group starts -- both from the
// histogram's fold chain.
// ---------------------------------------------------------------------------
namespace {

// Group sizes of the matrix levels from the matrix itself (the recurrence of
// recover_histogram, wt2wm.py:137-156, on the WM layout): the group of prefix
// P at level l starts at s and holds c symbols; its zero child 2P starts at
// rank0_l(s) in level l+1 and its one child 2P+1 at Z_l + s - rank0_l(s), with
// sizes rank0_l(s + c) - rank0_l(s) and the rest.  One rank query per group
// and level replaces the 2^w-bin histogram of the text.
// Rank directory: per level, per 512-bit block the ones before it inside its
// chunk of RK_CHUNK blocks (u32), and per chunk the ones before it (i64).
constexpr int RK_THREADS = 256;
constexpr int RK_PER = 4;  // blocks per thread
constexpr int RK_CHUNK = RK_THREADS * RK_PER;

__global__ void __launch_bounds__(RK_THREADS) rank_blocks_kernel(const uint64_t* __restrict__ words, int64_t nwords,
                                                                int64_t nblk, int64_t nchunk,
                                                                uint32_t* __restrict__ blk_pre,
                                                                int64_t* __restrict__ chunk_pre) {
  __shared__ uint32_t s_w[RK_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int level = blockIdx.y;
  const uint64_t* L = words + (int64_t)level * nwords;
  uint32_t* bp = blk_pre + (int64_t)level * nblk;
  uint32_t carry = 0;
#pragma unroll 1
  for (int i = 0; i < RK_PER; ++i) {
    // block b = chunk * RK_CHUNK + i * RK_THREADS + thread: a warp reads 2 KB contiguous
    const int64_t b = (int64_t)blockIdx.x * RK_CHUNK + i * RK_THREADS + threadIdx.x;
    uint32_t c = 0;
    if (b < nblk) {
      const int64_t w0 = b * 8;
      if (w0 + 8 <= nwords && !(reinterpret_cast<uintptr_t>(L + w0) & 15)) {
        const ulonglong2* q = reinterpret_cast<const ulonglong2*>(L + w0);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const ulonglong2 v = __ldcs(q + k);
          c += __popcll(v.x) + __popcll(v.y);
        }
      } else {
        for (int64_t wd = w0; wd < min(w0 + 8, nwords); ++wd) c += __popcll(L[wd]);
      }
    }
    const uint32_t incl = warp_incl_scan(c);
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < RK_THREADS / 32; ++k) {
      const uint32_t t = s_w[k];
      wpre += k < wid ? t : 0u;
      tot += t;
    }
    if (b < nblk) bp[b] = carry + wpre + incl - c;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) chunk_pre[(int64_t)level * nchunk + blockIdx.x] = carry;
}

// per level (one CTA each): exclusive scan of the chunk totals in place
__global__ void __launch_bounds__(TAB_THREADS) rank_chunks_kernel(int64_t* __restrict__ chunk_pre, int64_t nchunk) {
  __shared__ int64_t s_red[33];
  int64_t* c = chunk_pre + (int64_t)blockIdx.x * nchunk;
  block_scan_excl(
      nchunk, [&](int64_t i) { return c[i]; }, [&](int64_t i, int64_t v) { c[i] = v; }, s_red);
}

struct RankDir {
  const uint64_t* words;
  int64_t nwords, nblk, nchunk, n;
  const uint32_t* blk_pre;
  const int64_t* chunk_pre;
};

// ones of level l before position p (0 <= p <= n)
__device__ __forceinline__ int64_t level_rank1(const RankDir& d, int l, int64_t p, int64_t ones_total) {
  if (p >= d.n) return ones_total;
  const int64_t b = p >> 9;
  const uint64_t* L = d.words + (int64_t)l * d.nwords;
  int64_t r = d.chunk_pre[(int64_t)l * d.nchunk + b / RK_CHUNK] + d.blk_pre[(int64_t)l * d.nblk + b];
  const int64_t wp = p >> 6;
  for (int64_t wd = b * 8; wd < wp; ++wd) r += __popcll(L[wd]);
  if (p & 63) r += __popcll(L[wp] & ((1ull << (p & 63)) - 1ull));
  return r;
}

// level l -> level l + 1 of the count chain (numeric prefix order), of the WM
// group starts (indexed by numeric prefix) and of the WT interval starts
// (wt_bounds level k at chain_off(k) + k, 2^k starts + the end n as sentinel):
// the tree's interval of 2P starts where P's does, 2P+1 after 2P's symbols.
__global__ void wm_groups_kernel(const RankDir d, int l, const int64_t* __restrict__ zeros, int64_t* __restrict__ chain,
                                 int64_t* __restrict__ wmst, int64_t* __restrict__ wt_bounds) {
  const int64_t ng = 1ll << l;
  const int64_t z = zeros[l], ones = d.n - z;
  int64_t* wt1 = wt_bounds + chain_off(l + 1) + (l + 1);
  for (int64_t P = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; P < ng; P += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = l ? wmst[chain_off(l) + P] : 0;
    const int64_t c = l ? chain[chain_off(l) + P] : d.n;
    const int64_t wt = l ? wt_bounds[chain_off(l) + l + P] : 0;
    const int64_t rs = s - level_rank1(d, l, s, ones);
    const int64_t re = (s + c) - level_rank1(d, l, s + c, ones);
    chain[chain_off(l + 1) + 2 * P] = re - rs;
    chain[chain_off(l + 1) + 2 * P + 1] = c - (re - rs);
    wmst[chain_off(l + 1) + 2 * P] = rs;
    wmst[chain_off(l + 1) + 2 * P + 1] = z + s - rs;
    wt1[2 * P] = wt;
    wt1[2 * P + 1] = wt + (re - rs);
    if (P == 0) wt1[2 * ng] = d.n;
  }
}

struct WtViaWm {
  size_t off_temp, off_zeros, off_chain, off_bounds, off_wm, off_ws, total;
  size_t off_blk, off_chunk;  // rank directory (inside the matrix build's workspace, free by then)
  int64_t nblk, nchunk;
};

// kind WT: the matrix goes to a temporary and is reordered into the tree;
// kind WM (histogram / borders requested): the matrix is the output itself.
inline bool wt_via_wm_layout(int64_t n, int sym_bytes, int64_t sigma, int kind, WtViaWm* L) {
  Plan P;
  if (!make_plan(n, sym_bytes, sigma, WVLT_KIND_WM, &P, true) || !P.tail_w) return false;
  const int w = P.width;
  const int64_t nwords = (n + 63) >> 6;
  size_t off = 0;
  L->off_temp = off;
  if (kind == WVLT_KIND_WT) off = align_up(off + (size_t)w * nwords * 8, 256);
  L->off_zeros = off;
  off = align_up(off + (size_t)w * 8, 256);
  L->off_chain = off;
  off = align_up(off + ((size_t)2 << w) * 8, 256);
  L->off_bounds = off;
  off = align_up(off + (((size_t)2 << w) + w) * 8, 256);
  L->off_wm = off;
  off = align_up(off + ((size_t)2 << w) * 8, 256);
  L->off_ws = off;
  L->nblk = (nwords + 7) / 8;
  L->nchunk = (L->nblk + RK_CHUNK - 1) / RK_CHUNK;
  L->off_blk = off;
  size_t r = align_up(off + (size_t)w * L->nblk * 4, 256);
  L->off_chunk = r;
  r = align_up(r + (size_t)w * L->nchunk * 8, 256);
  L->total = std::max(off + P.total, r);
  return true;
}

// node borders of levels 1..w-1 (layout of wvlt_build_device) from the group
// recurrence's tables: WT interval starts (bounds, level k at chain_off(k) + k)
// or WM group starts (wmst, level k at chain_off(k)), both indexed by prefix
__global__ void borders_copy_kernel(const int64_t* __restrict__ src, int w, int wt, int64_t* __restrict__ out) {
  const int64_t total = (1ll << w) - 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = 63 - __clzll(i + 2);
    const int64_t P = i + 2 - (1ll << k);
    out[i] = src[chain_off(k) + (wt ? k : 0) + P];
  }
}

// Wide alphabets (w > 8) through the fused matrix build: kind WT reorders the
// matrix into the tree; both kinds take the histogram and the node borders
// from the group recurrence over the matrix levels (no pass over the text).
int build_wt_via_wm(int kind, const void* text, int sym_bytes, int64_t n, int64_t sigma, uint64_t* level_words,
                    int64_t* zeros, int64_t* hist, int64_t* borders, unsigned char* ws, const WtViaWm& L,
                    int32_t* status, cudaStream_t s, void (*pass_done)(void*, int, int), void* ctx) {
  const int w = code_width_host(sigma);
  const int64_t nwords = (n + 63) >> 6;
  const bool wt = kind == WVLT_KIND_WT;
  uint64_t* temp = wt ? (uint64_t*)(ws + L.off_temp) : level_words;
  int64_t* chain = (int64_t*)(ws + L.off_chain);
  int64_t* bounds = (int64_t*)(ws + L.off_bounds);
  int64_t* wmst = (int64_t*)(ws + L.off_wm);
  // the matrix (its kernels check the symbol range; a level's zero count is the
  // same in both layouts)
  int rc = build_device_impl(text, sym_bytes, n, sigma, WVLT_KIND_WM, temp, zeros ? zeros : (int64_t*)(ws + L.off_zeros), nullptr,
                             nullptr, ws + L.off_ws, L.total - L.off_ws, status, s, wt ? nullptr : pass_done, ctx);
  if (rc) return rc;
  int launches = g_launches;
  cudaError_t e;
  // the count chain and the WM group starts from the matrix levels: rank
  // directory of every level, then the group recurrence level by level
  {
    const int64_t* dz = zeros ? zeros : (int64_t*)(ws + L.off_zeros);
    uint32_t* blk = (uint32_t*)(ws + L.off_blk);
    int64_t* chk = (int64_t*)(ws + L.off_chunk);
    rank_blocks_kernel<<<dim3((unsigned)L.nchunk, (unsigned)w), RK_THREADS, 0, s>>>(temp, nwords, L.nblk, L.nchunk,
                                                                                  blk, chk);
    rank_chunks_kernel<<<w, TAB_THREADS, 0, s>>>(chk, L.nchunk);
    launches += 2;
    RankDir d;
    d.words = temp;
    d.nwords = nwords;
    d.nblk = L.nblk;
    d.nchunk = L.nchunk;
    d.n = n;
    d.blk_pre = blk;
    d.chunk_pre = chk;
    for (int l = 0; l < w; ++l) {
      const int64_t ng = 1ll << l;
      wm_groups_kernel<<<(unsigned)std::min<int64_t>((ng + 255) / 256, (int64_t)sm_count() * 8), 256, 0, s>>>(
          d, l, dz, chain, wmst, bounds);
      ++launches;
    }
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  if (borders && w >= 2) {
    borders_copy_kernel<<<(unsigned)std::min<int64_t>((((1ll << w) - 2) + 255) / 256, (int64_t)sm_count() * 8), 256, 0,
                          s>>>(wt ? bounds : wmst, w, wt ? 1 : 0, borders);
    ++launches;
  }
  if (!wt) {
    if (hist) {
      e = cudaMemcpyAsync(hist, chain + chain_off(w), ((size_t)1 << w) * 8, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return (int)e;
    }
    g_launches = launches;
    return (int)cudaGetLastError();
  }
  // levels 0 and 1 are identical; the others are reordered group by group
  e = cudaMemcpyAsync(level_words, temp, (size_t)std::min(w, 2) * nwords * 8, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return (int)e;
  // one launch per level (measured: all levels in one 2-D grid is slower --
  // 2 (w - 2) concurrent streams of HBM traffic instead of 2)
  int64_t blocks = (nwords + 256 * MERGE_WORDS_PER_LANE - 1) / (256 * MERGE_WORDS_PER_LANE);
  blocks = std::min<int64_t>(blocks, (int64_t)sm_count() * 32);
  for (int k = 2; k < w; ++k) {
    merge_bits_kernel<<<(unsigned)blocks, 256, 0, s>>>(level_words + (int64_t)k * nwords, 0, nwords, n,
                                                        bounds + chain_off(k) + k, wmst + chain_off(k), 1ll << k,
                                                        temp + (int64_t)k * nwords);
    ++launches;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  if (hist) {
    e = cudaMemcpyAsync(hist, chain + chain_off(w), ((size_t)1 << w) * 8, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return (int)e;
  }
  prof_mark(s, WVLT_STAGE_REORDER);
  g_launches = launches;
  if (pass_done) pass_done(ctx, 0, w);
  return 0;
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

int wvlt_profile_enable(int on) {
  g_prof.on = on != 0;
  g_prof.n = 0;
  return 0;
}

int wvlt_profile_read(float* stage_ms, int* stage_ids, int max_stages) {
  Prof& P = g_prof;
  if (!P.on || P.n < 2) return 0;
  cudaError_t e = cudaEventSynchronize(P.ev[P.n - 1]);
  if (e != cudaSuccess) return -(int)e;
  int k = 0;
  for (int i = 0; i + 1 < P.n && k < max_stages; ++i, ++k) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, P.ev[i], P.ev[i + 1]);
    if (stage_ms) stage_ms[k] = ms;
    if (stage_ids) stage_ids[k] = P.ids[i];
  }
  return k;
}

size_t wvlt_workspace_bytes(int64_t n, int sym_bytes, int64_t sigma, int kind) {
  Plan P;
  if (n < 0 || !(sym_bytes == 1 || sym_bytes == 2 || sym_bytes == 4)) return 0;
  if (!make_plan(n, sym_bytes, sigma, kind, &P, true)) return 0;
  Plan P2;
  make_plan(n, sym_bytes, sigma, kind, &P2, false);
  size_t total = std::max(P.total, P2.total);
  WtViaWm L;
  if (P.width > 8 && n > 0 && wt_via_wm_layout(n, sym_bytes, sigma, kind, &L)) total = std::max(total, L.total);
  if (k8_eligible(sym_bytes, P.width, n) && !P.widen_bytes) return std::max(total, k8_layout(n, P.width).total);
  return total;
}

int wvlt_workspace_parts(int64_t n, int sym_bytes, int64_t sigma, int kind, int want_hist, int want_borders,
                         size_t* parts) {
  if (!parts) return WVLT_E_ARG;
  parts[0] = parts[1] = parts[2] = 0;
  if (n < 0 || !(sym_bytes == 1 || sym_bytes == 2 || sym_bytes == 4) || sigma < 1) return WVLT_E_ARG;
  if (kind != WVLT_KIND_WT && kind != WVLT_KIND_WM) return WVLT_E_ARG;
  const bool lean = kind == WVLT_KIND_WM && !want_hist && !want_borders;
  Plan P;
  if (!make_plan(n, sym_bytes, sigma, kind, &P, lean)) return WVLT_E_WIDTH;
  const int w = P.width;
  if (n == 0 || w == 0) return 0;
  // the same path choice as build_device_impl
  WtViaWm L;
  if ((kind == WVLT_KIND_WT || !lean) && w > 8 && wt_via_wm_layout(n, sym_bytes, sigma, kind, &L)) {
    Plan M;
    make_plan(n, sym_bytes, sigma, WVLT_KIND_WM, &M, true);
    parts[0] = (L.off_ws - L.off_zeros) + M.off_buf0;                 // group tables + the matrix build's tables
    parts[1] = 2 * M.buf_bytes + (M.widen_bytes ? align_up((size_t)n * M.widen_bytes, 256) : 0);
    parts[2] = kind == WVLT_KIND_WT ? (size_t)w * (size_t)((n + 63) >> 6) * 8 : 0;  // the matrix before its reorder
    return 0;
  }
  if (k8_eligible(sym_bytes, w, n) && !P.widen_bytes) {
    parts[0] = k8_layout(n, w).total;  // per-tile counts, prefixes, run tables; the level orders stay on chip
    return 0;
  }
  parts[0] = P.off_buf0;
  parts[1] = 2 * P.buf_bytes + (P.widen_bytes ? align_up((size_t)n * P.widen_bytes, 256) : 0);
  return 0;
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
  e = launch_hist_generic(text, sym_bytes, n, w, (unsigned long long*)hist, status, s);
  return (int)e;
}

int wvlt_build_device(const void* text, int sym_bytes, int64_t n, int64_t sigma, int kind, uint64_t* level_words,
                      int64_t* zeros, int64_t* hist, int64_t* borders, void* workspace, size_t workspace_bytes,
                      int32_t* status, void* stream) {
  return build_device_impl(text, sym_bytes, n, sigma, kind, level_words, zeros, hist, borders, workspace,
                           workspace_bytes, status, stream, nullptr, nullptr);
}
}  // extern "C"

namespace {
// The build; `pass_done(ctx, l0, K)` (optional) is called right after pass
// l0..l0+K-1 is enqueued, when those levels' words are final on `stream`.
int build_device_impl(const void* text, int sym_bytes, int64_t n, int64_t sigma, int kind, uint64_t* level_words,
                      int64_t* zeros, int64_t* hist, int64_t* borders, void* workspace, size_t workspace_bytes,
                      int32_t* status, void* stream, void (*pass_done)(void*, int, int), void* ctx) {
  g_launches = 0;
  if (!(sym_bytes == 1 || sym_bytes == 2 || sym_bytes == 4) || n < 0 || sigma < 1) return WVLT_E_ARG;
  if (kind != WVLT_KIND_WT && kind != WVLT_KIND_WM) return WVLT_E_ARG;
  Plan P;
  // lean WM build: no histogram / borders requested -> no K1 histogram and no
  // K2 tables; each pass's tables come from its own tile-count scan
  const bool lean = kind == WVLT_KIND_WM && !hist && !borders;
  if (!make_plan(n, sym_bytes, sigma, kind, &P, lean)) return WVLT_E_WIDTH;
  const int w = P.width;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (status) {
    e = cudaMemsetAsync(status, 0, 4, s);
    if (e != cudaSuccess) return (int)e;
  }
  const int64_t nwords = (n + 63) >> 6;
  if ((kind == WVLT_KIND_WT || !lean) && n > 0 && w > 8 && text && level_words && workspace) {
    WtViaWm L;
    if (wt_via_wm_layout(n, sym_bytes, sigma, kind, &L)) {
      if (workspace_bytes < L.total) return WVLT_E_WORKSPACE;
      return build_wt_via_wm(kind, text, sym_bytes, n, sigma, level_words, zeros, hist, borders,
                             (unsigned char*)workspace, L, status, s, pass_done, ctx);
    }
  }
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
    if (w >= 2 && borders) {
      e = cudaMemsetAsync(borders, 0, (((size_t)1 << w) - 2) * 8, s);
      if (e != cudaSuccess) return (int)e;
    }
    if (w == 0 && n > 0 && status) {  // range check still applies: every symbol must be 0
      e = launch_hist_generic(text, sym_bytes, n, 0, nullptr, status, s);
      if (e != cudaSuccess) return (int)e;
    }
    return 0;
  }
  if (!text || !level_words || !workspace) return WVLT_E_ARG;
  if (k8_eligible(sym_bytes, w, n) && !P.widen_bytes) {
    // byte text, 2 <= w <= 8: every level in one fused pass (k8.cuh)
    if (workspace_bytes < k8_layout(n, w).total) return WVLT_E_WORKSPACE;
    return build_k8((const uint8_t*)text, n, sigma, w, kind, level_words, zeros, hist, borders, workspace, status, s,
                    pass_done, ctx, 0, -1);
  }
  if (workspace_bytes < P.total) return WVLT_E_WORKSPACE;
  unsigned char* ws = (unsigned char*)workspace;
  int64_t* chain = (int64_t*)(ws + P.off_chain);
  int64_t* wtstart = (int64_t*)(ws + P.off_wtstart);
  int64_t* wm_base = (int64_t*)(ws + P.off_wmbase);
  int64_t* corr = (int64_t*)(ws + P.off_corr);
  int64_t* bsum = (int64_t*)(ws + P.off_bsum);
  void* bufs[2] = {ws + P.off_buf0, ws + P.off_buf1};
  int32_t* st_flag = status ? status : (int32_t*)(ws + P.off_scratch);

  g_prof.n = 0;
  prof_mark(s, -1);
  // (the fused passes write / zero their own levels)
  const int fused_lvl = P.k32_w ? P.k32_lvl : P.k16_w ? P.k16_lvl : P.tail_w ? P.tail_lvl : w;
  if (fused_lvl > 0) {
    e = cudaMemsetAsync(level_words, 0, (size_t)fused_lvl * nwords * 8, s);
    if (e != cudaSuccess) return (int)e;
  }
  if (P.npass > 0) {
    e = cudaMemsetAsync(ws + P.off_tcnt[0], 0, P.tcnt_bytes, s);
    if (e != cudaSuccess) return (int)e;
  }
  unsigned long long* hw = (unsigned long long*)(chain + chain_off(w));
  if (!lean) {
    e = cudaMemsetAsync(hw, 0, ((size_t)1 << w) * 8, s);
    if (e != cudaSuccess) return (int)e;
  }
  if (!status) {
    e = cudaMemsetAsync(st_flag, 0, 4, s);
    if (e != cudaSuccess) return (int)e;
  }
  const void* src0 = text;
  if (P.widen_bytes) {
    ++g_launches;
    void* wide = ws + P.off_wide;
    const int blocks = sm_count() * 8;
    if (P.widen_bytes == 2) widen_kernel<uint8_t, uint16_t><<<blocks, 256, 0, s>>>((const uint8_t*)text, (uint16_t*)wide, n);
    else if (sym_bytes == 1) widen_kernel<uint8_t, uint32_t><<<blocks, 256, 0, s>>>((const uint8_t*)text, (uint32_t*)wide, n);
    else widen_kernel<uint16_t, uint32_t><<<blocks, 256, 0, s>>>((const uint16_t*)text, (uint32_t*)wide, n);
    e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    src0 = wide;
  }
  prof_mark(s, WVLT_STAGE_MEMSET);
  if (P.npass == 0) {
    e = cudaSuccess;  // (lean, the fused 2-byte pass first: its digit kernel does the range check)
  } else if (lean) {
    ++g_launches;
    e = launch_digits_fast(src0, P.in_bytes[0], n, w, sigma, P.K[0], P.tile[0], P.ntiles[0],
                           (uint32_t*)(ws + P.off_tcnt[0]), st_flag, s);
  } else {
    g_launches += P.in_bytes[0] == 1 && w <= 8 && P.tile[0] == TILE_U8 && (((uintptr_t)src0) & 15) == 0 ? 1 : 2;
    e = launch_hist_build(src0, P.in_bytes[0], n, w, P.K[0], P.tile[0], P.ntiles[0], hw,
                          (uint32_t*)(ws + P.off_tcnt[0]), st_flag, s);
  }
  if (e != cudaSuccess) return (int)e;
  prof_mark(s, WVLT_STAGE_HIST);

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
  ta.zeros_out = zeros;
  ta.hist_out = hist;
  ta.borders_out = (w >= 2) ? borders : nullptr;
  ta.status = st_flag;
  if (!lean) {
    tables_kernel<<<1, TAB_THREADS, 0, s>>>(ta);
    ++g_launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
  }
  prof_mark(s, WVLT_STAGE_TABLES);

  const void* cur = src0;
  for (int p = 0; p < P.npass; ++p) {
    uint32_t* tcnt = (uint32_t*)(ws + P.off_tcnt[p]);
    int64_t* tpre = (int64_t*)(ws + P.off_tpre[p]);
    e = launch_scan(tcnt, P.K[p], P.ntiles[p], bsum, tpre, s);
    g_launches += 2;
    if (e != cudaSuccess) return (int)e;
    if (lean) {
      ++g_launches;
      wm_pass_tables_kernel<<<1, 32, 0, s>>>(tcnt, tpre, P.ntiles[p], P.K[p], P.lvl[p],
                                             wm_base + (int64_t)p * (KMAX + 1) * NDIG, zeros);
      e = cudaGetLastError();
      if (e != cudaSuccess) return (int)e;
    }
    prof_mark(s, WVLT_STAGE_SCAN0 + p);
    PassArgs pa;
    memset(&pa, 0, sizeof(pa));
    pa.src = cur;
    pa.dst = P.out_bytes[p] ? bufs[p & 1] : nullptr;
    pa.words = level_words;
    pa.nwords = nwords;
    pa.n = n;
    pa.ntiles = P.ntiles[p];
    pa.level = P.lvl[p];
    pa.width = w;
    pa.kind = kind;
    pa.has_out = P.out_bytes[p] ? 1 : 0;
    pa.tcnt = tcnt;
    pa.tpre = tpre;
    if (pa.has_out && p + 1 == P.npass) {
      pa.ntshift = 13;  // output for the fused tail, which counts its own digits
    } else if (pa.has_out) {
      pa.ncnt = (uint32_t*)(ws + P.off_tcnt[p + 1]);
      pa.nntiles = P.ntiles[p + 1];
      pa.ntshift = P.tshift[p + 1];
      pa.nK = P.K[p + 1];
    }
    pa.wm_base = wm_base + (int64_t)p * (KMAX + 1) * NDIG;
    pa.corr = corr;
    for (int j = 0; j <= KMAX; ++j) pa.corr_off[j] = P.corr_off[p][j];
    e = launch_pass(P.in_bytes[p], P.out_bytes[p], P.K[p], pa, P.ntiles[p], s);
    ++g_launches;
    if (e != cudaSuccess) return (int)e;
    prof_mark(s, WVLT_STAGE_PASS0 + p);
    if (pass_done) pass_done(ctx, P.lvl[p], P.K[p]);
    cur = pa.dst;
  }
  int curbuf = P.npass > 0 ? ((P.npass - 1) & 1) : -1;  // bufs[] index holding cur, -1 = the text
  int stage = P.npass;
  if (P.k32_w) {
    const int ob = curbuf == 0 ? 1 : 0;
    uint16_t* out = (uint16_t*)bufs[ob];
    const int64_t lk = P.k32_lvl;
    const uint32_t vmax_ok = (uint32_t)std::min<int64_t>(sigma - 1, 0xFFFFFFFFll);
    const int check = curbuf < 0 && vmax_ok < 0xFFFFFFFFu ? 1 : 0;  // text input: symbols must be < sigma
    const int rc = build_k32((const uint32_t*)cur, n, P.k32_w, level_words + lk * nwords, zeros ? zeros + lk : nullptr,
                             out, (unsigned char*)out + align_up((size_t)n * 2, 256), st_flag, vmax_ok, check, s,
                             pass_done, ctx, (int)lk, stage);
    if (rc) return rc;
    ++stage;
    cur = out;
    curbuf = ob;
  }
  if (P.k16_w) {
    const int ob = curbuf == 0 ? 1 : 0;
    uint8_t* out = (uint8_t*)bufs[ob];
    const int64_t lk = P.k16_lvl;
    const uint32_t vmax_ok = (uint32_t)std::min<int64_t>(sigma - 1, 0xFFFF);
    const int check = curbuf < 0 && vmax_ok < 0xFFFFu ? 1 : 0;  // text input: symbols must be < sigma
    const int rc = build_k16((const uint16_t*)cur, n, P.k16_w, level_words + lk * nwords, zeros ? zeros + lk : nullptr,
                             out, out + align_up((size_t)n, 256), st_flag, vmax_ok, check, s, pass_done, ctx,
                             (int)lk, stage);
    if (rc) return rc;
    ++stage;
    cur = out;
    curbuf = ob;
  }
  if (P.tail_w) {
    const int64_t lt = P.tail_lvl;
    return build_k8((const uint8_t*)cur, n, (int64_t)1 << P.tail_w, P.tail_w, kind, level_words + lt * nwords,
                    zeros ? zeros + lt : nullptr, nullptr, nullptr, bufs[curbuf == 0 ? 1 : 0], st_flag, s, pass_done, ctx,
                    (int)lt, stage);
  }
  return 0;
}

// Pageable host buffers (a numpy array as the reference's callers pass it):
// copies are staged through two page-locked chunks, the host side of each
// chunk spread over several CPU threads (one thread copies ~15 GB/s, or far
// less when it also takes the page faults of fresh output memory; PCIe moves
// ~55 GB/s) and overlapped with the DMA of the neighbouring chunk.
#ifndef STAGE_CHUNK_MB
#define STAGE_CHUNK_MB 32
#endif
constexpr size_t STAGE_CHUNK = (size_t)STAGE_CHUNK_MB << 20;
#ifndef STAGE_MAX_THREADS
#define STAGE_MAX_THREADS 8u
#endif

struct Stager {
  unsigned char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaError_t init() {
    if (buf[0]) return cudaSuccess;
    cudaError_t e = cudaHostAlloc((void**)&buf[0], 2 * STAGE_CHUNK, cudaHostAllocDefault);
    if (e != cudaSuccess) {
      buf[0] = nullptr;
      return e;
    }
    buf[1] = buf[0] + STAGE_CHUNK;
    for (int k = 0; k < 2 && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
    return e;
  }
};
thread_local Stager g_stager;

inline int stage_threads() {
  const unsigned hw = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(STAGE_MAX_THREADS, hw));
}

void par_memcpy(void* dst, const void* src, size_t n, int nt) {
  if (nt <= 1 || n < ((size_t)4 << 20)) {
    memcpy(dst, src, n);
    return;
  }
  const size_t per = ((n + nt - 1) / nt + 4095) & ~(size_t)4095;
  std::vector<std::thread> th;
  for (int t = 1; t < nt && (size_t)t * per < n; ++t)
    th.emplace_back([=] { memcpy((char*)dst + t * per, (const char*)src + t * per, std::min(per, n - t * per)); });
  memcpy(dst, src, std::min(per, n));
  for (auto& x : th) x.join();
}

// Touch every page of a fresh (pageable) output buffer from nt threads, so its
// page faults are taken in parallel while the upload and the build run rather
// than serially inside the final copy.
void prefault_pages(void* p, size_t n, int nt) {
  const size_t page = 4096;
  const size_t per = ((n + nt - 1) / nt + page - 1) & ~(page - 1);
  std::vector<std::thread> th;
  for (int t = 0; t < nt && (size_t)t * per < n; ++t)
    th.emplace_back([=] {
      volatile char* c = (volatile char*)p;
      const size_t e = std::min(n, (size_t)(t + 1) * per);
      for (size_t i = (size_t)t * per; i < e; i += page) c[i] = 0;  // an output buffer: contents are overwritten
    });
  for (auto& x : th) x.join();
}

bool host_is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// pageable host -> device, stream ordered on s (returns once the last chunk is queued)
cudaError_t staged_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  Stager& g = g_stager;
  cudaError_t e = g.init();
  if (e != cudaSuccess) return e;
  const int nt = stage_threads();
  size_t off = 0;
  for (int c = 0; off < bytes; ++c, off += STAGE_CHUNK) {
    const int k = c & 1;
    const size_t sz = std::min(STAGE_CHUNK, bytes - off);
    if (c >= 2 && (e = cudaEventSynchronize(g.ev[k])) != cudaSuccess) return e;  // chunk c - 2 has left buf[k]
    par_memcpy(g.buf[k], (const char*)src + off, sz, nt);
    if ((e = cudaMemcpyAsync((char*)dst + off, g.buf[k], sz, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(g.ev[k], s)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// device -> pageable host after the work queued on s; returns when the data is there
cudaError_t staged_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  Stager& g = g_stager;
  cudaError_t e = g.init();
  if (e != cudaSuccess) return e;
  const int nt = stage_threads();
  const size_t nch = (bytes + STAGE_CHUNK - 1) / STAGE_CHUNK;
  auto issue = [&](size_t c) -> cudaError_t {
    const int k = (int)(c & 1);
    const size_t off = c * STAGE_CHUNK, sz = std::min(STAGE_CHUNK, bytes - off);
    cudaError_t r = cudaMemcpyAsync(g.buf[k], (const char*)src + off, sz, cudaMemcpyDeviceToHost, s);
    return r == cudaSuccess ? cudaEventRecord(g.ev[k], s) : r;
  };
  for (size_t c = 0; c < std::min<size_t>(2, nch); ++c)
    if ((e = issue(c)) != cudaSuccess) return e;
  for (size_t c = 0; c < nch; ++c) {
    const int k = (int)(c & 1);
    const size_t off = c * STAGE_CHUNK, sz = std::min(STAGE_CHUNK, bytes - off);
    if ((e = cudaEventSynchronize(g.ev[k])) != cudaSuccess) return e;
    par_memcpy((char*)dst + off, g.buf[k], sz, nt);
    if (c + 2 < nch && (e = issue(c + 2)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// wvlt_build_host: the level words of a finished pass go device->host on a copy
// stream while the next pass runs.
struct HostCopy {
  cudaStream_t main, copy;
  cudaEvent_t ev[MAXP];
  int nev;
  uint64_t* host;
  const uint64_t* dev;
  int64_t nwords;
  cudaError_t err;
};

void host_copy_pass(void* c, int l0, int K) {
  HostCopy& h = *(HostCopy*)c;
  if (h.err != cudaSuccess || h.nev >= MAXP || h.nwords == 0) return;
  cudaEvent_t e = h.ev[h.nev++];
  h.err = cudaEventRecord(e, h.main);
  if (h.err == cudaSuccess) h.err = cudaStreamWaitEvent(h.copy, e, 0);
  if (h.err == cudaSuccess)
    h.err = cudaMemcpyAsync(h.host + (int64_t)l0 * h.nwords, h.dev + (int64_t)l0 * h.nwords, (size_t)K * h.nwords * 8,
                            cudaMemcpyDeviceToHost, h.copy);
}
}  // namespace

extern "C" {

int wvlt_build_host_borders(const void* host_text, int sym_bytes, int64_t n, int64_t sigma, int kind,
                            uint64_t* host_level_words, int64_t* host_zeros, int64_t* host_hist,
                            int64_t* host_borders, void* dev_text, uint64_t* dev_level_words, void* dev_small,
                            void* workspace, size_t workspace_bytes, void* stream) {
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
  int64_t* dborders = (host_borders && w >= 2) ? small + 1 + w + ((int64_t)1 << w) : nullptr;
  const int64_t nwords = (n + 63) >> 6;
  if (w > 0 && nwords > 0 && !host_level_words) return WVLT_E_ARG;
  // pageable level words: no per-pass streaming, one staged download at the end;
  // their pages are faulted in by helper threads while the text goes up
  const bool words_pinned = !(w > 0 && nwords > 0) || host_is_pinned(host_level_words);
  std::thread prefault;
  if (!words_pinned)
    prefault = std::thread(prefault_pages, (void*)host_level_words, (size_t)w * nwords * 8, stage_threads());
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{prefault};
  if (n > 0) {
    if (!host_text || !dev_text) return WVLT_E_ARG;
    e = host_is_pinned(host_text)
            ? cudaMemcpyAsync(dev_text, host_text, (size_t)n * sym_bytes, cudaMemcpyHostToDevice, s)
            : staged_h2d(dev_text, host_text, (size_t)n * sym_bytes, s);
    if (e != cudaSuccess) return (int)e;
  }
  // level words of each finished pass stream back while the next pass runs
  static thread_local cudaStream_t copy_stream = nullptr;
  static thread_local cudaEvent_t evs[MAXP];
  if (!copy_stream) {
    e = cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return (int)e;
    for (int i = 0; i < MAXP; ++i) {
      e = cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return (int)e;
    }
  }
  HostCopy hc;
  hc.main = s;
  hc.copy = copy_stream;
  for (int i = 0; i < MAXP; ++i) hc.ev[i] = evs[i];
  hc.nev = 0;
  hc.host = host_level_words;
  hc.dev = dev_level_words;
  hc.nwords = (w > 0) ? nwords : 0;
  hc.err = cudaSuccess;
  int rc = build_device_impl(dev_text, sym_bytes, n, sigma, kind, dev_level_words, dzeros, host_hist ? dhist : nullptr,
                             dborders, workspace, workspace_bytes, dstatus, s, words_pinned ? host_copy_pass : nullptr,
                             &hc);
  if (rc) {
    cudaStreamSynchronize(copy_stream);
    return rc;
  }
  if (hc.err != cudaSuccess) return (int)hc.err;
  if (w > 0 && nwords > 0 && !words_pinned) {
    if (prefault.joinable()) prefault.join();
    e = staged_d2h(host_level_words, dev_level_words, (size_t)w * nwords * 8, s);
    if (e != cudaSuccess) return (int)e;
  } else if (w > 0 && nwords > 0 && hc.nev == 0) {  // degenerate shapes: no passes ran
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
  if (dborders) {
    e = cudaMemcpyAsync(host_borders, dborders, (((size_t)1 << w) - 2) * 8, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return (int)e;
  }
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return (int)e;
  e = cudaStreamSynchronize(copy_stream);
  if (e != cudaSuccess) return (int)e;
  return (hstatus & WVLT_STATUS_RANGE) ? WVLT_E_RANGE : 0;
}

int wvlt_build_host(const void* host_text, int sym_bytes, int64_t n, int64_t sigma, int kind,
                    uint64_t* host_level_words, int64_t* host_zeros, int64_t* host_hist, void* dev_text,
                    uint64_t* dev_level_words, void* dev_small, void* workspace, size_t workspace_bytes,
                    void* stream) {
  return wvlt_build_host_borders(host_text, sym_bytes, n, sigma, kind, host_level_words, host_zeros, host_hist,
                                 nullptr, dev_text, dev_level_words, dev_small, workspace, workspace_bytes, stream);
}

// A sequence of independent builds with host buffers, software-pipelined over
// three streams: uploads (H2D of build i+1's text), compute (`stream`: build i)
// and downloads (D2H of build i-1's levels, which start pass by pass as in
// wvlt_build_host).  Device text / levels / small buffers are double-buffered
// (two slots); the workspace is used by the compute stream only.  PCIe is full
// duplex, so in steady state a build costs max(upload, download, compute)
// instead of their sum.
int wvlt_build_host_batch(int count, const void* const* host_texts, const int64_t* ns, int sym_bytes, int64_t sigma,
                          int kind, uint64_t* const* host_level_words, int64_t* host_zeros, int64_t* host_hist,
                          int32_t* host_status, void* dev_text, size_t dev_text_slot_bytes, uint64_t* dev_level_words,
                          size_t dev_words_slot_bytes, void* dev_small, void* workspace, size_t workspace_bytes,
                          void* stream) {
  if (count < 0 || !(sym_bytes == 1 || sym_bytes == 2 || sym_bytes == 4) || sigma < 1) return WVLT_E_ARG;
  if (count == 0) return 0;
  if (!host_texts || !ns || !host_level_words || !host_status || !dev_small) return WVLT_E_ARG;
  const int w = code_width_host(sigma);
  if (w > WVLT_MAX_WIDTH) return WVLT_E_WIDTH;
  for (int i = 0; i < count; ++i) {
    const int64_t n = ns[i];
    if (n < 0 || (size_t)n * sym_bytes > dev_text_slot_bytes) return WVLT_E_ARG;
    if ((size_t)w * ((n + 63) >> 6) * 8 > dev_words_slot_bytes) return WVLT_E_ARG;
    if (n > 0 && (!host_texts[i] || !dev_text)) return WVLT_E_ARG;
    if (w > 0 && n > 0 && (!host_level_words[i] || !dev_level_words)) return WVLT_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  static thread_local cudaStream_t up = nullptr, down = nullptr;
  static thread_local cudaEvent_t ev_up[2], ev_comp[2], ev_down[2], ev_pass[2][MAXP];
  if (!up) {
    e = cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking);
    for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
      e = cudaEventCreateWithFlags(&ev_up[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_comp[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_down[k], cudaEventDisableTiming);
      for (int i = 0; i < MAXP && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&ev_pass[k][i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
      up = nullptr;
      return (int)e;
    }
  }
  const size_t small_slot = ((size_t)1 << w) + w + 1;  // int64 entries: status, zeros, hist
  // the small outputs come back through page-locked staging (a copy into pageable
  // memory would block this thread until the download stream reached it, and
  // with it the enqueueing of the next upload)
  static thread_local int64_t* stage = nullptr;
  static thread_local size_t stage_len = 0;
  const size_t need_stage = (size_t)std::max(count, 64) * small_slot;  // (grown rarely: cudaFreeHost syncs)
  if (stage_len < need_stage) {
    if (stage) cudaFreeHost(stage);
    stage = nullptr;
    stage_len = 0;
    if ((e = cudaHostAlloc((void**)&stage, need_stage * 8, cudaHostAllocDefault)) != cudaSuccess) return (int)e;
    stage_len = need_stage;
  }
  // enqueue build i on the three streams; an error stops the queue, and every
  // stream is drained below before returning (no copy into caller memory may
  // still be in flight)
  auto enqueue = [&](int i) -> int {
    cudaError_t e;
    const int slot = i & 1;
    const int64_t n = ns[i];
    const int64_t nwords = (n + 63) >> 6;
    unsigned char* dtext = (unsigned char*)dev_text + slot * dev_text_slot_bytes;
    uint64_t* dwords = (uint64_t*)((unsigned char*)dev_level_words + slot * dev_words_slot_bytes);
    int64_t* small = (int64_t*)dev_small + slot * small_slot;
    // upload: the slot's text is free once build i-2 has run
    if (i >= 2 && (e = cudaStreamWaitEvent(up, ev_comp[slot], 0)) != cudaSuccess) return (int)e;
    if (n > 0 && (e = cudaMemcpyAsync(dtext, host_texts[i], (size_t)n * sym_bytes, cudaMemcpyHostToDevice, up)) != cudaSuccess)
      return (int)e;
    if ((e = cudaEventRecord(ev_up[slot], up)) != cudaSuccess) return (int)e;
    // compute: after the upload, and after build i-2's levels have left the slot
    if ((e = cudaStreamWaitEvent(s, ev_up[slot], 0)) != cudaSuccess) return (int)e;
    if (i >= 2 && (e = cudaStreamWaitEvent(s, ev_down[slot], 0)) != cudaSuccess) return (int)e;
    HostCopy hc;
    hc.main = s;
    hc.copy = down;
    for (int k = 0; k < MAXP; ++k) hc.ev[k] = ev_pass[slot][k];
    hc.nev = 0;
    hc.host = host_level_words[i];
    hc.dev = dwords;
    hc.nwords = (w > 0) ? nwords : 0;
    hc.err = cudaSuccess;
    int32_t* dstatus = (int32_t*)small;
    int64_t* dzeros = small + 1;
    int64_t* dhist = small + 1 + w;
    int64_t* hh = host_hist ? host_hist + ((size_t)i << w) : nullptr;
    const int brc = build_device_impl(dtext, sym_bytes, n, sigma, kind, dwords, dzeros, hh ? dhist : nullptr, nullptr,
                                      workspace, workspace_bytes, dstatus, s, host_copy_pass, &hc);
    if (brc) return brc;
    if (hc.err != cudaSuccess) return (int)hc.err;
    if ((e = cudaEventRecord(ev_comp[slot], s)) != cudaSuccess) return (int)e;
    // download: whatever the passes did not already send, then the small outputs
    if ((e = cudaStreamWaitEvent(down, ev_comp[slot], 0)) != cudaSuccess) return (int)e;
    if (w > 0 && nwords > 0 && hc.nev == 0 &&
        (e = cudaMemcpyAsync(host_level_words[i], dwords, (size_t)w * nwords * 8, cudaMemcpyDeviceToHost, down)) !=
            cudaSuccess)
      return (int)e;
    // status, zeros and histogram are contiguous in the slot: one small copy
    if ((e = cudaMemcpyAsync(stage + (size_t)i * small_slot, small, (1 + w + (hh ? ((size_t)1 << w) : 0)) * 8,
                             cudaMemcpyDeviceToHost, down)) != cudaSuccess)
      return (int)e;
    if ((e = cudaEventRecord(ev_down[slot], down)) != cudaSuccess) return (int)e;
    return 0;
  };
  int rc = 0;
  for (int i = 0; i < count && !rc; ++i) rc = enqueue(i);
  cudaError_t e1 = cudaStreamSynchronize(up), e2 = cudaStreamSynchronize(s), e3 = cudaStreamSynchronize(down);
  if (rc) return rc;
  if (e1 != cudaSuccess) return (int)e1;
  if (e2 != cudaSuccess) return (int)e2;
  if (e3 != cudaSuccess) return (int)e3;
  int range = 0;
  for (int i = 0; i < count; ++i) {
    const int64_t* st = stage + (size_t)i * small_slot;
    host_status[i] = *(const int32_t*)st;
    if (host_zeros && w > 0) memcpy(host_zeros + (size_t)i * w, st + 1, (size_t)w * 8);
    if (host_hist) memcpy(host_hist + ((size_t)i << w), st + 1 + w, ((size_t)1 << w) * 8);
    if (host_status[i] & WVLT_STATUS_RANGE) range = 1;
  }
  return range ? WVLT_E_RANGE : 0;
}

int wvlt_last_launches(void) { return g_launches; }

int wvlt_merge_bits(uint64_t* dst_words, int64_t word_lo, int64_t word_hi, int64_t n_bits, const int64_t* bounds,
                    const int64_t* src_starts, int64_t ntasks, const uint64_t* src_words, void* stream) {
  if (word_hi < word_lo || word_lo < 0 || n_bits < 0 || ntasks < 0) return WVLT_E_ARG;
  if (word_hi == word_lo) return 0;
  if (!dst_words || (n_bits > 0 && (!bounds || !src_starts || !src_words || ntasks < 1))) return WVLT_E_ARG;
  const int64_t nw = word_hi - word_lo;
  int64_t blocks = (nw + 256 * MERGE_WORDS_PER_LANE - 1) / (256 * MERGE_WORDS_PER_LANE);
  const int64_t cap = (int64_t)sm_count() * 32;
  if (blocks > cap) blocks = cap;
  merge_bits_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dst_words, word_lo, word_hi, n_bits, bounds,
                                                                         src_starts, ntasks, src_words);
  return (int)cudaGetLastError();
}

int wvlt_merge_levels_peer(uint64_t* dst_words, int64_t dst_row_words, int width, int64_t word_lo, int64_t word_hi,
                           int64_t n_bits, const int64_t* bounds, const int64_t* bounds_off, const int64_t* src_starts,
                           const int32_t* src_ranks, const int64_t* task_off, const uint64_t* const* level_src,
                           int nranks, void* stream) {
  if (width < 0 || word_hi < word_lo || word_lo < 0 || n_bits < 0 || nranks < 1 || dst_row_words < word_hi - word_lo)
    return WVLT_E_ARG;
  if (width == 0 || word_hi == word_lo) return 0;
  if (!dst_words || !bounds || !bounds_off || !src_starts || !src_ranks || !task_off || !level_src) return WVLT_E_ARG;
  const int64_t nw = word_hi - word_lo;
  int64_t blocks = (nw + 256 * MERGE_WORDS_PER_LANE - 1) / (256 * MERGE_WORDS_PER_LANE);
  const int64_t cap = std::max<int64_t>(1, (int64_t)sm_count() * 32 / width);
  if (blocks > cap) blocks = cap;
  merge_peer_kernel<<<dim3((unsigned)blocks, (unsigned)width), 256, 0, (cudaStream_t)stream>>>(
      dst_words, dst_row_words, word_lo, word_hi, n_bits, bounds, bounds_off, src_starts, src_ranks, task_off,
      level_src, nranks);
  return (int)cudaGetLastError();
}

int wvlt_peer_plan(const int64_t* rows, int64_t row_stride, int64_t borders_col, const int64_t* local_ns, int nranks,
                   int width, int kind, int64_t* bounds, int64_t* src_starts, int32_t* src_ranks, int64_t* bounds_off,
                   int64_t* task_off, void* stream) {
  if (nranks < 1 || width < 0 || width > WVLT_MAX_WIDTH || (kind != WVLT_KIND_WT && kind != WVLT_KIND_WM))
    return WVLT_E_ARG;
  if (!rows || !local_ns || !bounds || !src_starts || !src_ranks || !bounds_off || !task_off) return WVLT_E_ARG;
  const int64_t items = std::max<int64_t>((1ll << width) - 1, width + 1);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, (int64_t)sm_count() * 8));
  peer_plan_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(rows, row_stride, borders_col, local_ns, nranks, width,
                                                             kind, bounds, src_starts, src_ranks, bounds_off, task_off);
  return (int)cudaGetLastError();
}

}  // extern "C"

#include "support.cuh"
