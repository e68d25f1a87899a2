// K8: the whole build of a byte text with code width 2 <= W <= 8 in ONE fused
// pass.  For a wavelet matrix the symbols of level l with equal l-bit key keep
// their text order (A_l is the stable LSD sort of the text by the key), and
// for the tree the same holds per prefix group, so every level's contribution
// of a text tile is a set of contiguous runs placed by the tile prefix of its
// W-bit digit counts.  One CTA per K8_TILE-symbol tile runs the W-1 stable
// one-bit splits in shared memory and emits all W levels -- no intermediate
// order ever goes back to HBM, no second pass.  Needs per-tile counts of all
// 2^W digits (hist8_kernel) and their prefix over tiles (scan8_* kernels).
// Included from wvlt_b200.cu (same translation unit).

namespace {


// ---- K1: per-tile counts of every W-bit value (tile-major [tile][2^W]) ----
// One warp per tile; lane-private 16-bit counter pairs for (p, p + 2^(W-1)): the
// low half counts both, the high half p + 2^(W-1); zeroed after every tile so
// the per-tile row sums never carry.
constexpr int H8_WARPS = 4;
#ifndef K8_TILE
#define K8_TILE 16384  // symbols per tile of every kernel of the single pass (measured: 8192 and 32768 slower)
#endif
#ifndef K8_CTAS
#define K8_CTAS (K8_TILE == 8192 ? 7 : K8_TILE == 16384 ? 4 : 2)  // pass CTAs per SM (shared memory / registers)
#endif
#ifndef H8_COLS
#define H8_COLS 16  // counter columns per warp (measured: 16 < 32 < 8 ms; more warps per SM)
#endif
#ifndef H8_PLANE_W
#define H8_PLANE_W 3  // up to this width the counts come from bit planes in registers (no shared atomics)
#endif
#ifndef H8_ATOMIC_BATCH
#define H8_ATOMIC_BATCH 2  // hist8: 16-byte loads per pipelined batch when counting by shared atomics
#endif
#ifndef H8_BATCH
#define H8_BATCH 4  // hist16 / hist32: 16-byte loads in flight per lane (measured: 4 < 8 < 16)
#endif

// Clearing the tile's words of the levels a pass ORs into: bulk (TMA) stores
// of a zero row in shared memory, so the clearing goes through the async copy
// engine instead of the LSU pipe (the bottleneck of the counting kernels: one
// shared atomic per symbol).  Rows that are not whole or not 16-byte aligned
// fall back to LSU stores.  The kernel fills the row (zero_row_init) and waits
// for the bulk reads before exiting (zero_row_drain).
template <int TW>
__device__ __forceinline__ uint32_t zero_row_init(uint64_t* s_zero) {
  for (int i = threadIdx.x; i < TW; i += blockDim.x) s_zero[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  return (uint32_t)__cvta_generic_to_shared(s_zero);
}
__device__ __forceinline__ void zero_row_drain(int lane) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncthreads();
}
// levels 1..nlev-1 after `lvl` (row stride nwords), words [w0, w0 + tw)
template <int TW>
__device__ __forceinline__ void clear_level_rows(uint64_t* lvl, int64_t nwords, int64_t w0, int tw, int nlev,
                                                 uint32_t zsrc, int lane) {
  if (tw == TW && !(nwords & 1) && !(reinterpret_cast<uintptr_t>(lvl + w0) & 15)) {
    if (lane == 0) {
      for (int j = 1; j < nlev; ++j)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(lvl + j * nwords + w0),
                     "r"(zsrc), "r"((uint32_t)(TW * 8))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  } else {
    for (int j = 1; j < nlev; ++j) {
      uint64_t* lw = lvl + j * nwords + w0;
      for (int i = lane; i < tw; i += 32) __stcs(reinterpret_cast<unsigned long long*>(lw + i), 0ull);
    }
  }
}

#ifndef H8_PLANE_BATCH
#define H8_PLANE_BATCH 4  // 256-bit loads in flight per lane when counting from bit planes (measured: 4 < 2 < 1 ms)
#endif
// 32 bytes, streaming (read once)
__device__ __forceinline__ void ld256_cs(uint32_t (&r)[8], const uint32_t* p) {
  asm volatile("ld.global.cs.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
// the same 32 bytes from an address that is only 16-byte aligned
__device__ __forceinline__ void ld2x128_cs(uint32_t (&r)[8], const uint32_t* p) {
  const uint4 a = __ldcs(reinterpret_cast<const uint4*>(p)), b = __ldcs(reinterpret_cast<const uint4*>(p) + 1);
  r[0] = a.x, r[1] = a.y, r[2] = a.z, r[3] = a.w, r[4] = b.x, r[5] = b.y, r[6] = b.z, r[7] = b.w;
}
// exchange the bits selected by m with the bits sh above them
__device__ __forceinline__ uint32_t delta_swap(uint32_t x, int sh, uint32_t m) {
  const uint32_t t = ((x >> sh) ^ x) & m;
  return x ^ t ^ (t << sh);
}

// One 16384-symbol tile of the register-plane counting (widths <= H8_PLANE_W): a
// lane takes 32 consecutive symbols per step (one 256-bit load, or two 128-bit
// ones from a text that is only 16-byte aligned) and turns them into W bit
// planes of 32 bits, bit 8k + u = symbol 4u + k (byte k of word u): one shift +
// one LOP3 per word and plane.  The values are counted with one POPC per value
// and 32 symbols; level 0 is the top plane transposed to text order by four
// delta swaps and stored as the lane's own 32-bit half word (coalesced, no
// shuffles).
template <int W, bool WIDE>
__device__ __forceinline__ void hist8_planes_tile(const uint32_t* __restrict__ t32, uint32_t* __restrict__ l0, int lane,
                                                  int check, uint32_t (&acc)[1 << W], uint32_t& hi_or) {
  constexpr int NB = 1 << W;
  constexpr int NIT = K8_TILE / 32 / 32;
  constexpr int NB2 = H8_PLANE_BATCH;
  static_assert(NIT % NB2 == 0, "whole batches");
  uint32_t qn[NB2][8];
#pragma unroll
  for (int k = 0; k < NB2; ++k) {
    if (WIDE) ld256_cs(qn[k], t32 + 8 * (k * 32 + lane));
    else ld2x128_cs(qn[k], t32 + 8 * (k * 32 + lane));
  }
#pragma unroll 1
  for (int it0 = 0; it0 < NIT; it0 += NB2) {
    uint32_t q[NB2][8];
#pragma unroll
    for (int k = 0; k < NB2; ++k)
#pragma unroll
      for (int u = 0; u < 8; ++u) q[k][u] = qn[k][u];
    if (it0 + NB2 < NIT) {
#pragma unroll
      for (int k = 0; k < NB2; ++k) {
        if (WIDE) ld256_cs(qn[k], t32 + 8 * ((it0 + NB2 + k) * 32 + lane));
        else ld2x128_cs(qn[k], t32 + 8 * ((it0 + NB2 + k) * 32 + lane));
      }
    }
#pragma unroll
    for (int k = 0; k < NB2; ++k) {
      uint32_t pl[W], nl[W];
      if (check) hi_or |= (q[k][0] | q[k][1] | q[k][2] | q[k][3]) | (q[k][4] | q[k][5] | q[k][6] | q[k][7]);
#pragma unroll
      for (int b = 0; b < W; ++b) {
        uint32_t x = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          x |= (u >= b ? q[k][u] << (u - b) : q[k][u] >> (b - u)) & (0x01010101u << u);
        pl[b] = x;
        nl[b] = ~x;
      }
#pragma unroll
      for (int v = 0; v < NB; ++v) {
        uint32_t m = (v & 1) ? pl[0] : nl[0];
#pragma unroll
        for (int b = 1; b < W; ++b) m &= ((v >> b) & 1) ? pl[b] : nl[b];
        acc[v] += __popc(m);
      }
      uint32_t t = pl[W - 1];  // bit (k1 k0 u2 u1 u0) -> bit (u2 u1 u0 k1 k0)
      t = delta_swap(t, 12, 0x0000F0F0u);
      t = delta_swap(t, 6, 0x00CC00CCu);
      t = delta_swap(t, 3, 0x0A0A0A0Au);
      t = delta_swap(t, 1, 0x22222222u);
      l0[(it0 + k) * 32 + lane] = t;
    }
  }
}

// It also writes level 0 (the top code bit of every symbol, already in text
// order), so that level can leave for the host while the rest is built.
template <int W>
__global__ void __launch_bounds__(H8_WARPS * 32) hist8_kernel(const uint8_t* __restrict__ text, int64_t n,
                                                             int64_t ntiles, uint32_t vmax_ok, int check,
                                                             uint32_t* __restrict__ tcnt8, uint64_t* __restrict__ level0,
                                                             int64_t nwords, int32_t* __restrict__ status) {
  constexpr int NB = 1 << W;
  constexpr int HALF = NB / 2;
  constexpr int C = H8_COLS;  // counter columns per warp (lanes l and l + C share one)
  constexpr int WORDS = HALF * C;
  extern __shared__ __align__(16) uint32_t s_cols[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* c32 = s_cols + (size_t)wid * WORDS;
  uint32_t* c32w = c32 + (lane & (C - 1));
  for (int i = lane; i < WORDS; i += 32) c32[i] = 0;
  __shared__ __align__(128) uint64_t s_zero[K8_TILE / 64];
  const uint32_t zsrc = zero_row_init<K8_TILE / 64>(s_zero);
  __syncwarp();
  uint32_t vmax = 0;
  uint32_t hi_or = 0;  // (register-plane widths) OR of every word: a bit above the code width = out of range
  const bool aligned = (((uintptr_t)text) & 15) == 0;           // 128-bit loads
  const bool wide = (((uintptr_t)text) & 31) == 0;              // (register-plane widths) 256-bit loads
  const int64_t nwarps = (int64_t)gridDim.x * H8_WARPS;
  for (int64_t t = (int64_t)blockIdx.x * H8_WARPS + wid; t < ntiles; t += nwarps) {
    const int64_t first = t * K8_TILE;
    const int cnt = (int)min((int64_t)K8_TILE, n - first);
    // clear this tile's words of levels 1..W-1 (the pass ORs run-edge words)
    clear_level_rows<K8_TILE / 64>(level0, nwords, first >> 6, (int)min((int64_t)(K8_TILE / 64), nwords - (first >> 6)),
                                   W, zsrc, lane);
    // narrow alphabets count in registers from bit planes, one POPC per value
    constexpr bool PLANES = W <= H8_PLANE_W;
    uint32_t acc[PLANES ? NB : 1];
#pragma unroll
    for (int v = 0; v < (PLANES ? NB : 1); ++v) acc[v] = 0;
    const bool fast = cnt == K8_TILE && aligned;
    if (PLANES && fast) {
      // narrow alphabets: counted from bit planes in registers (hist8_planes_tile)
      const uint32_t* t32 = reinterpret_cast<const uint32_t*>(text + first);
      uint32_t* l0 = reinterpret_cast<uint32_t*>(level0) + (first >> 5);
      if constexpr (PLANES) {
        if (wide) hist8_planes_tile<W, true>(t32, l0, lane, check, acc, hi_or);
        else hist8_planes_tile<W, false>(t32, l0, lane, check, acc, hi_or);
      }
    } else if (!PLANES && fast) {
      const uint4* v4 = reinterpret_cast<const uint4*>(text + first);
      // (the widths that count by shared atomics) software-pipelined: the next
      // batch's loads are in flight while this one is counted
      constexpr int NBAT = H8_ATOMIC_BATCH;
      uint4 qn[NBAT];
#pragma unroll
      for (int k = 0; k < NBAT; ++k) qn[k] = __ldcs(v4 + k * 32 + lane);
#pragma unroll 1
      for (int k0 = 0; k0 < K8_TILE / 16 / 32; k0 += NBAT) {
        uint4 q[NBAT];
#pragma unroll
        for (int k = 0; k < NBAT; ++k) q[k] = qn[k];
        if (k0 + NBAT < K8_TILE / 16 / 32) {
#pragma unroll
          for (int k = 0; k < NBAT; ++k) qn[k] = __ldcs(v4 + (k0 + NBAT + k) * 32 + lane);
        }
#pragma unroll
        for (int k = 0; k < NBAT; ++k) {
          const uint32_t wd[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
          uint32_t m16 = 0;  // level-0 bits of this lane's 16 symbols
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (check) vmax = __vmaxu4(vmax, wd[u]);
            const uint32_t lo = wd[u] & ((uint32_t)(HALF - 1) * 0x01010101u);
            const uint32_t hb = (wd[u] >> (W - 1)) & 0x01010101u;
            m16 |= ((hb * 0x01020408u) >> 24) << (4 * u);
            // increment 0x00010001 for a value with its top bit set, else 1, straight
            // from one PRMT: the low half counts both values of the pair, the high
            // half the upper one
#pragma unroll
            for (int b = 0; b < 4; ++b)
              atomicAdd(c32w + prmt(lo, 0, 0x4440 + b) * C, prmt(hb, 1u, 0x5054 + (b << 8)));
          }
          // lanes 4i..4i+3 hold 64 consecutive symbols: one level-0 word
          const uint32_t m32 = m16 | (__shfl_down_sync(FULL, m16, 1) << 16);
          const uint32_t hi32 = __shfl_down_sync(FULL, m32, 2);
          if ((lane & 3) == 0)
            level0[(first >> 6) + ((k0 + k) * 32 + lane) / 4] = (uint64_t)m32 | ((uint64_t)hi32 << 32);
        }
      }
    } else {
      uint32_t* l0 = reinterpret_cast<uint32_t*>(level0) + (first >> 5);
      for (int i0 = 0; i0 < cnt; i0 += 32) {
        const int i = i0 + lane;
        uint32_t v = 0;
        if (i < cnt) {
          v = text[first + i];
          vmax = max(vmax, v);
          atomicAdd(c32w + (v & (HALF - 1)) * C, ((v >> (W - 1)) & 1u) ? 0x10001u : 1u);
        }
        const uint32_t b = __ballot_sync(FULL, i < cnt && ((v >> (W - 1)) & 1u));
        if (lane == 0) l0[i0 >> 5] = b;
      }
      // a tail tile ending inside a 64-bit word: zero its upper half
      if (lane == 0 && (((first + cnt + 31) >> 5) & 1)) l0[(cnt + 31) >> 5] = 0u;
    }
    __syncwarp();
    // row p (bins p, p + HALF) summed over the 32 lane columns; lane l takes rows
    // l, l + 32, ...; skewed reads keep the 32 lanes on distinct banks
    // (16-byte reads: lane l takes chunk k ^ (l & 7) of its row, so the 8
    // lanes of a wavefront hit 8 different bank quads)
    uint32_t* row_out = tcnt8 + t * NB;
    if (PLANES && fast) {
#pragma unroll
      for (int v = 0; v < (PLANES ? NB : 1); ++v) {
        const uint32_t tot = __reduce_add_sync(FULL, acc[v]);
        if (lane == v) row_out[v] = tot;
        if (check && (uint32_t)v > vmax_ok && tot) vmax = 0xFFu;  // a value in [sigma, 2^W)
      }
      continue;  // the shared counters were not touched
    }
    for (int p = lane; p < HALF; p += 32) {
      const uint4* row = reinterpret_cast<const uint4*>(c32 + p * C);
      uint32_t s = 0;
#pragma unroll
      for (int k = 0; k < C / 4; ++k) {
        const uint4 q = row[k ^ (lane & (C / 4 - 1))];
        s += (q.x + q.y) + (q.z + q.w);
      }
      row_out[p] = (s & 0xFFFFu) - (s >> 16);
      row_out[p + HALF] = s >> 16;
    }
    __syncwarp();
    for (int i = lane * 4; i < WORDS; i += 128) *reinterpret_cast<uint4*>(c32 + i) = make_uint4(0, 0, 0, 0);
    __syncwarp();
  }
  if (check) {
    vmax = max(max(vmax & 0xFFu, (vmax >> 8) & 0xFFu), max((vmax >> 16) & 0xFFu, vmax >> 24));
    if (hi_or & ~((uint32_t)(NB - 1) * 0x01010101u)) vmax = 0xFFu;
    if (vmax > vmax_ok) atomicOr(status, WVLT_STATUS_RANGE);
  }
  zero_row_drain(lane);  // the zero row must outlive the bulk stores that read it
}

// ---- S8: exclusive prefix over tiles of every column of tcnt8 ----
// chunks of S8_CHUNK tiles: per-chunk column sums (thread = column, 16 loads
// in flight), a block-wide scan of each column over the chunks, then the
// per-tile prefixes from the chunk carries.
constexpr int S8_CHUNK = 64;     // tiles per chunk
constexpr int S8_UNROLL = 16;
constexpr int S8_SCAN_THREADS = 512;

__global__ void __launch_bounds__(256) scan8_chunks_kernel(const uint32_t* __restrict__ tcnt8, int64_t ntiles,
                                                          int nb, uint32_t* __restrict__ chunk) {
  const int d = threadIdx.x;
  const int64_t t0 = (int64_t)blockIdx.x * S8_CHUNK, t1 = min(t0 + S8_CHUNK, ntiles);
  uint32_t s = 0;
  for (int64_t t = t0; t < t1; t += S8_UNROLL) {
    uint32_t v[S8_UNROLL];
#pragma unroll
    for (int u = 0; u < S8_UNROLL; ++u) v[u] = t + u < t1 ? __ldcs(tcnt8 + (t + u) * nb + d) : 0u;
#pragma unroll
    for (int u = 0; u < S8_UNROLL; ++u) s += v[u];
  }
  chunk[(int64_t)blockIdx.x * nb + d] = s;
}

// one block per column: exclusive scan of the column over the chunks (in
// place) and the column total
__global__ void __launch_bounds__(S8_SCAN_THREADS) scan8_carry_kernel(uint32_t* __restrict__ chunk, int64_t nchunks,
                                                                     int nb, int64_t* __restrict__ totals) {
  __shared__ uint32_t s_w[S8_SCAN_THREADS / 32];
  const int d = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t carry = 0;
  for (int64_t b0 = 0; b0 < nchunks; b0 += S8_SCAN_THREADS) {
    const int64_t b = b0 + threadIdx.x;
    const uint32_t v = b < nchunks ? chunk[b * nb + d] : 0u;
    const uint32_t incl = warp_incl_scan(v);
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < S8_SCAN_THREADS / 32; ++k) {
      const uint32_t t = s_w[k];
      wpre += k < wid ? t : 0u;
      tot += t;
    }
    if (b < nchunks) chunk[b * nb + d] = carry + wpre + incl - v;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[d] = carry;
}

__global__ void __launch_bounds__(256) scan8_apply_kernel(const uint32_t* __restrict__ tcnt8, int64_t ntiles, int nb,
                                                         const uint32_t* __restrict__ chunk,
                                                         uint32_t* __restrict__ tpre8) {
  const int d = threadIdx.x;
  const int64_t t0 = (int64_t)blockIdx.x * S8_CHUNK, t1 = min(t0 + S8_CHUNK, ntiles);
  uint32_t run = chunk[(int64_t)blockIdx.x * nb + d];
  for (int64_t t = t0; t < t1; t += S8_UNROLL) {
    uint32_t v[S8_UNROLL];
#pragma unroll
    for (int u = 0; u < S8_UNROLL; ++u) v[u] = t + u < t1 ? __ldcs(tcnt8 + (t + u) * nb + d) : 0u;
#pragma unroll
    for (int u = 0; u < S8_UNROLL; ++u) {
      if (t + u < t1) tpre8[(t + u) * nb + d] = run;
      run += v[u];
    }
  }
}

// ---- T8: global placement tables from the digit totals ----
// base[j * 256 + d], 1 <= j < W, d < 2^j an LSD digit: where the group of d
// starts in level j (WM: exclusive prefix of the group sizes in LSD-digit
// order; WT: interval start of the numeric prefix rev(d)).  Also the zero
// counts per level and (optionally) the histogram and the node borders (level
// j at [2^j - 2, 2^(j+1) - 2) indexed by the numeric j-bit prefix: WT interval
// starts, levelstats.py:58-73; WM group starts, wt2wm.py:55-78).
// exclusive scan of get(i), i < cnt <= 256, by one warp (8 entries per lane), written through put
template <typename Get, typename Put>
__device__ __forceinline__ void warp_scan_excl64(int cnt, int lane, Get get, Put put) {
  int64_t v[8], sum = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = lane * 8 + k;
    v[k] = i < cnt ? get(i) : 0;
    sum += v[k];
  }
  int64_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  int64_t run = incl - sum;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = lane * 8 + k;
    if (i < cnt) put(i, run);
    run += v[k];
  }
}

// One CTA (the fused passes keep n < 2^32, so every count fits 32 bits):
// group sizes of every level folded from the digit totals level by level
// (thread = group), zero counts by warp reductions, then one warp per level
// scans the sizes into group starts (warp 7: the WM level-W starts).
__global__ void __launch_bounds__(256) tables8_kernel(const int64_t* __restrict__ totals, int W, int kind,
                                                      int64_t* __restrict__ base, int64_t* __restrict__ zeros,
                                                      int64_t* __restrict__ hist, int64_t* __restrict__ baseW,
                                                      int64_t* __restrict__ borders) {
  __shared__ uint32_t s_tot[256];
  __shared__ uint32_t s_cnt[9][256];  // level j: WM by LSD digit, WT by numeric prefix
  __shared__ uint32_t s_z[8][8];      // [warp][level] partial zero counts
  const int nb = 1 << W;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t tot = 0;
  if (tid < nb) {
    const int64_t t64 = totals[tid];
    tot = (uint32_t)t64;
    s_tot[tid] = tot;
    if (hist) hist[tid] = t64;
    s_cnt[W][kind == WVLT_KIND_WM ? (int)rev_bits((unsigned)tid, W) : tid] = tot;
  }
  for (int l = 0; l < W; ++l) {  // symbols whose level-l bit is 0
    const uint32_t z = __reduce_add_sync(FULL, ((tid >> (W - 1 - l)) & 1) ? 0u : tot);
    if (lane == 0) s_z[wid][l] = z;
  }
  __syncthreads();
  for (int j = W - 1; j >= 1; --j) {
    const int mj = 1 << j;
    if (tid < mj)  // WM: LSD digits d, d + 2^j of level j+1; WT: prefixes 2P, 2P+1
      s_cnt[j][tid] = kind == WVLT_KIND_WM ? s_cnt[j + 1][tid] + s_cnt[j + 1][tid + mj]
                                           : s_cnt[j + 1][2 * tid] + s_cnt[j + 1][2 * tid + 1];
    __syncthreads();
  }
  if (zeros && tid < W) {
    int64_t z = 0;
    for (int w = 0; w < 8; ++w) z += w * 32 < nb ? s_z[w][tid] : 0u;
    zeros[tid] = z;
  }
  const int j = wid + 1;  // warp j - 1: level j
  if (j < W) {
    const uint32_t* c = s_cnt[j];
    int64_t* bj = borders ? borders + ((1 << j) - 2) : nullptr;
    if (kind == WVLT_KIND_WM)
      warp_scan_excl64(1 << j, lane, [&](int d) { return (int64_t)c[d]; }, [&](int d, int64_t v) {
        base[j * 256 + d] = v;
        if (bj) bj[rev_bits((unsigned)d, j)] = v;  // digit d = bit-reversed prefix
      });
    else
      warp_scan_excl64(1 << j, lane, [&](int P) { return (int64_t)c[P]; }, [&](int P, int64_t v) {
        base[j * 256 + rev_bits((unsigned)P, j)] = v;
        if (bj) bj[P] = v;
      });
  } else if (wid == 7 && baseW) {  // WM level-W group starts (the 2-byte pass's output order)
    warp_scan_excl64(nb, lane, [&](int d) { return (int64_t)s_tot[rev_bits((unsigned)d, W)]; },
                     [&](int d, int64_t v) { baseW[d] = v; });
  }
}

// ---- K3 (K8): the fused pass ----
struct Pass8Args {
  const uint8_t* src;
  uint64_t* words;
  int64_t nwords, n, ntiles;
  const uint32_t* tcnt8;
  const uint32_t* tpre8;
  const int64_t* base;  // [8][256]
};

#ifndef K8_EMIT_WORDS
#define K8_EMIT_WORDS 2  // destination words per emission task
#endif

// Runs of levels 1..W-1 flattened: run r = 2^j - 2 + d (j = level, d = LSD digit).
// (positions fit 32 bits: the single-pass path needs n < 2^32)
struct Tables8 {
  uint16_t cnt[256];  // run sizes
  uint16_t ls[256];   // run starts in the tile-local order of its level
  uint32_t gs[256];   // run starts in the global level
  uint32_t lb[256];   // symbols of earlier tiles in the run's group (scratch)
  uint16_t wpre[256]; // emission: destination words before each run (+ total)
  uint16_t cW[264];   // level-W digit counts (scratch, index d + d / 32)
  uint32_t lbW[264];  // level-W tile prefixes (scratch, index d + d / 32)
};

// a tile's count / prefix row into registers (entry e = lane + 32 k)
template <int W>
__device__ __forceinline__ void table8_load(const Pass8Args& a, int64_t tile, int lane, uint32_t (&rc)[8],
                                            uint32_t (&rp)[8]) {
  constexpr int NB = 1 << W;
  const uint32_t* cr = a.tcnt8 + tile * NB;
  const uint32_t* pr = a.tpre8 + tile * NB;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int e = lane + 32 * k;
    rc[k] = e < NB ? __ldcs(cr + e) : 0u;
    rp[k] = e < NB ? __ldcs(pr + e) : 0u;
  }
}

// ... and into the scratch in LSD-digit order
template <int W>
__device__ __forceinline__ void table8_stage(Tables8& tt, int lane, const uint32_t (&rc)[8], const uint32_t (&rp)[8]) {
  constexpr int NB = 1 << W;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int e = lane + 32 * k;
    if (e < NB) {
      const int d = (int)rev_bits((unsigned)e, W);
      // (bit-reversed d: the skew d + d / 32 spreads a warp's stores over the banks)
      tt.cW[d + (d >> 5)] = (uint16_t)rc[k];
      tt.lbW[d + (d >> 5)] = rp[k];
    }
  }
  __syncwarp();
}

template <int W>
__device__ __forceinline__ void table8_compute(Tables8& tt, const uint32_t* s_base, int lane) {
  constexpr int NB = 1 << W;
  constexpr int NR = NB - 2;

  // fold: level j's digit d collects the level j+1 digits d and d + 2^j
#pragma unroll 1
  for (int j = W - 1; j >= 1; --j) {
    const int mj = 1 << j;
    for (int d = lane; d < mj; d += 32) {
      int c;
      uint32_t lb;
      if (j == W - 1) {
        c = tt.cW[d + (d >> 5)] + tt.cW[d + mj + ((d + mj) >> 5)];
        lb = tt.lbW[d + (d >> 5)] + tt.lbW[d + mj + ((d + mj) >> 5)];
      } else {
        const int up = (2 << j) - 2;
        c = tt.cnt[up + d] + tt.cnt[up + d + mj];
        lb = tt.lb[up + d] + tt.lb[up + d + mj];
      }
      const int r = mj - 2 + d;
      tt.cnt[r] = (uint16_t)c;
      tt.lb[r] = lb;
      tt.gs[r] = s_base[r] + lb;
    }
    __syncwarp();
  }
  // one pass over the flattened runs (lane: PER consecutive ones): exclusive
  // prefixes of the run sizes (P) and of the destination words (wpre); a
  // run's tile-local start is P minus P at its level's first run.  (W = 8:
  // each lane's 8 runs move as 16-byte vectors -- scalar accesses at an
  // 8-run stride were 4- to 8-way bank conflicts)
  {
    constexpr int PER = (NR + 31) / 32;
    uint32_t c[PER], g[PER], nw[PER];
    if constexpr (PER == 8) {
      const uint4 cv = reinterpret_cast<const uint4*>(tt.cnt)[lane];
      const uint4 g0 = reinterpret_cast<const uint4*>(tt.gs)[2 * lane], g1 = reinterpret_cast<const uint4*>(tt.gs)[2 * lane + 1];
      const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) c[k] = (cw[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
      g[0] = g0.x; g[1] = g0.y; g[2] = g0.z; g[3] = g0.w;
      g[4] = g1.x; g[5] = g1.y; g[6] = g1.z; g[7] = g1.w;
    } else {
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        c[k] = tt.cnt[lane * PER + k];
        g[k] = tt.gs[lane * PER + k];
      }
    }
    uint32_t sc = 0, sw = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int r = lane * PER + k;
      if (r >= NR) c[k] = 0;  // (scratch beyond the runs)
      // emission tasks of the run: K8_EMIT_WORDS destination words each
      nw[k] = c[k] ? (((g[k] + c[k] - 1) >> 6) - (g[k] >> 6) + K8_EMIT_WORDS) / K8_EMIT_WORDS : 0u;
      sc += c[k];
      sw += nw[k];
    }
    uint32_t pc = warp_incl_scan(sc) - sc, pw = warp_incl_scan(sw) - sw;
    uint32_t P[PER], Wp[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      P[k] = pc;
      Wp[k] = pw;
      pc += c[k];
      pw += nw[k];
    }
    __syncwarp();
    if constexpr (PER == 8) {
      reinterpret_cast<uint4*>(tt.lb)[2 * lane] = make_uint4(P[0], P[1], P[2], P[3]);  // (lb is free once gs is set)
      reinterpret_cast<uint4*>(tt.lb)[2 * lane + 1] = make_uint4(P[4], P[5], P[6], P[7]);
      reinterpret_cast<uint4*>(tt.wpre)[lane] =
          make_uint4(Wp[0] | (Wp[1] << 16), Wp[2] | (Wp[3] << 16), Wp[4] | (Wp[5] << 16), Wp[6] | (Wp[7] << 16));
    } else {
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int r = lane * PER + k;
        if (r < NR) {
          tt.lb[r] = P[k];
          tt.wpre[r] = (uint16_t)Wp[k];
        }
      }
    }
    if (lane == 31) tt.wpre[NR] = (uint16_t)pw;
    __syncwarp();
    uint32_t lsv[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int r = lane * PER + k;
      lsv[k] = r < NR ? P[k] - tt.lb[(1 << (31 - __clz(r + 2))) - 2] : 0u;
    }
    if constexpr (PER == 8) {
      reinterpret_cast<uint4*>(tt.ls)[lane] =
          make_uint4(lsv[0] | (lsv[1] << 16), lsv[2] | (lsv[3] << 16), lsv[4] | (lsv[5] << 16), lsv[6] | (lsv[7] << 16));
    } else {
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int r = lane * PER + k;
        if (r < NR) tt.ls[r] = (uint16_t)lsv[k];
      }
    }
  }
}

// Compact per-tile run table written by tiles8_kernel and bulk-copied into
// the pass kernel's shared memory with the tile: positions fit 32 bits (the
// single-pass path needs n < 2^32), sizes and offsets inside a tile 16 bits.
// Sized by the width: 2^W - 2 runs plus the emission total, rounded so the
// table stays a multiple of 16 bytes (W = 8: 256 entries, 2560 bytes; W = 4:
// 16 entries, 160 bytes).
template <int W>
struct TabW {
  static constexpr int NRP = (((1 << W) - 1) + 7) & ~7;
  uint32_t gs[NRP];   // run starts in the global level
  uint16_t cnt[NRP];  // run sizes
  uint16_t ls[NRP];   // run starts in the tile-local order of the level
  uint16_t wpre[NRP]; // destination words before each run; wpre[NR] = total
};
using Tab8 = TabW<8>;  // the largest (workspace sizing)
static_assert(sizeof(Tab8) == 2560 && sizeof(TabW<2>) % 16 == 0 && sizeof(TabW<5>) % 16 == 0, "bulk-copy granularity");

// Emission of levels 1..W-1 from a tile's level-bit arrays (NC + 4 words per
// level, tile-local order): one destination word per task, the runs of all
// levels flattened (consecutive tasks = consecutive words of one run, so the
// stores of a warp coalesce); whole words stored, run-edge words OR-ed (runs of
// neighbouring tiles share them; the levels were zeroed).
template <int W, int NC>
__device__ __forceinline__ void emit_levels8(const TabW<W>& tt, const uint32_t* bits, uint64_t* words, int64_t nwords,
                                             int tid, int nthreads, uint8_t* coarse) {
  constexpr int NR = (1 << W) - 2;
#ifndef K8_EMIT_G
#define K8_EMIT_G 8  // measured: 8 < 16 < 4 < 32
#endif
  constexpr int G = K8_EMIT_G;  // tasks per coarse map entry
  const int total = tt.wpre[NR];
  // coarse task -> run map (shared scratch): the run of every 16th task, found by
  // one binary search each; a task then walks forward over the few runs that
  // start after its entry (empty runs share prefix values)
  for (int c = tid; c * G < total; c += nthreads) {
    const int q = c * G;
    int r = 0;
#pragma unroll
    for (int s = 128; s >= 1; s >>= 1)
      if (r + s < NR && tt.wpre[r + s] <= q) r += s;
    coarse[c] = (uint8_t)r;
  }
  bar_sync(1, nthreads);
  for (int q = tid; q < total; q += nthreads) {
    int r = coarse[q / G];  // last run with wpre[r] <= q
    while (r + 1 < NR && tt.wpre[r + 1] <= q) ++r;
    const int j = 31 - __clz(r + 2);
    // 32-bit bit positions: the fused passes keep n < 2^32 - 64
    const uint32_t g = tt.gs[r];
    const uint32_t c = tt.cnt[r];
    const uint32_t* L = bits + j * (NC + 4);
    const uint32_t w0 = (g >> 6) + K8_EMIT_WORDS * (uint32_t)(q - tt.wpre[r]);
    const uint32_t wlast = (g + c - 1) >> 6;
    const int ls = tt.ls[r];
    uint64_t* dst0 = words + (int64_t)j * nwords + w0;
#if K8_EMIT_WORDS == 2
    // the task's source bits are contiguous: [ls + lo0 - g, + up to 128) -- five
    // words from three aligned 64-bit loads instead of two 3-word extractions
    const uint32_t wb0 = w0 << 6;
    const uint32_t lo0 = g > wb0 ? g : wb0;
    const int src = ls + (int)(lo0 - g);
    const uint2* L2 = reinterpret_cast<const uint2*>(L) + (src >> 6);
    const uint2 qa = L2[0], qb = L2[1], qc = L2[2];
    const bool odd = (src >> 5) & 1;
    const uint32_t x0 = odd ? qa.y : qa.x, x1 = odd ? qb.x : qa.y, x2 = odd ? qb.y : qb.x, x3 = odd ? qc.x : qb.y,
                   x4 = odd ? qc.y : qc.x;
    const uint32_t sh = src & 31;
    const uint64_t s0 = (uint64_t)__funnelshift_r(x0, x1, sh) | ((uint64_t)__funnelshift_r(x1, x2, sh) << 32);
    const uint64_t s1 = (uint64_t)__funnelshift_r(x2, x3, sh) | ((uint64_t)__funnelshift_r(x3, x4, sh) << 32);
#endif
#pragma unroll
    for (int u = 0; u < K8_EMIT_WORDS; ++u) {
      const uint32_t wd = w0 + u;
      if (wd > wlast) break;
      const uint32_t wb = wd << 6;
      const uint32_t lo = g > wb ? g : wb;
      const uint32_t hi = (g + c) < wb + 64 ? (g + c) : wb + 64;
      const int len = (int)(hi - lo);
#if K8_EMIT_WORDS == 2
      // word 0: source bits [0, len) of s0 s1; word 1: [64 - (lo0 - wb0), + len)
      const uint32_t off = u ? 64u - (lo0 - wb0) : 0u;  // (word 1 starts where word 0's 64 - its offset bits end)
      const uint64_t raw = off == 0 ? s0 : off == 64 ? s1 : ((s0 >> off) | (s1 << (64 - off)));
      const uint64_t v = (len >= 64 ? raw : (raw & ((1ull << len) - 1))) << (lo - wb);
#else
      const uint64_t v = extract_bits(L, ls + (int)(lo - g), len) << (lo - wb);
#endif
      // whole word: plain store; run edge: OR (shared with a neighbouring run), skipped if empty
      asm volatile(
          "{\n\t.reg .pred p, q;\n\tsetp.eq.s32 p, %2, 64;\n\tsetp.ne.and.b64 q, %1, 0, !p;\n\t"
          "@p st.global.b64 [%0], %1;\n\t@q red.global.or.b64 [%0], %1;\n\t}" ::"l"(dst0 + u), "l"(v), "r"(len)
          : "memory");
    }
  }
}

constexpr int T8_WARPS = 8;

// One warp per tile: the tile's run tables (table8_compute) into the compact
// global layout, off the pass kernel's critical path.
template <int W>
__global__ void __launch_bounds__(T8_WARPS * 32) tiles8_kernel(const Pass8Args a, TabW<W>* __restrict__ out) {
  constexpr int NR = (1 << W) - 2;
  extern __shared__ __align__(16) unsigned char t8_smem[];
  __shared__ uint32_t s_base[256];  // global group starts of every run
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int r = threadIdx.x; r < NR; r += T8_WARPS * 32) {
    const int j = 31 - __clz(r + 2);
    s_base[r] = (uint32_t)__ldg(a.base + j * 256 + (r + 2 - (1 << j)));
  }
  __syncthreads();
  Tables8& tt = reinterpret_cast<Tables8*>(t8_smem)[wid];
  const int64_t nw = (int64_t)gridDim.x * T8_WARPS;
  int64_t tile = (int64_t)blockIdx.x * T8_WARPS + wid;
  if (tile >= a.ntiles) return;
  uint32_t rc[8], rp[8];
  table8_load<W>(a, tile, lane, rc, rp);
  for (; tile < a.ntiles; tile += nw) {
    table8_stage<W>(tt, lane, rc, rp);
    if (tile + nw < a.ntiles) table8_load<W>(a, tile + nw, lane, rc, rp);  // next row in flight
    table8_compute<W>(tt, s_base, lane);
    __syncwarp();
    TabW<W>* o = out + tile;
    constexpr int NRP = TabW<W>::NRP;  // (a multiple of 8: every field is whole 16-byte vectors)
    for (int i = lane; i < NRP / 4; i += 32)
      reinterpret_cast<uint4*>(o->gs)[i] = reinterpret_cast<const uint4*>(tt.gs)[i];
    for (int i = lane; i < NRP / 8; i += 32) {
      reinterpret_cast<uint4*>(o->cnt)[i] = reinterpret_cast<const uint4*>(tt.cnt)[i];
      reinterpret_cast<uint4*>(o->ls)[i] = reinterpret_cast<const uint4*>(tt.ls)[i];
      reinterpret_cast<uint4*>(o->wpre)[i] = reinterpret_cast<const uint4*>(tt.wpre)[i];
    }
    __syncwarp();
  }
}

// Threads of the pass kernel: Q 8-symbol runs ("quarters") per thread, the
// tile split into Q regions of T / Q symbols (run k of thread t covers
// [k T/Q + 8 t, k T/Q + 8 t + 8)).  More runs per thread amortize the scan.
#ifndef K8_Q
#define K8_Q 4
#endif

template <int Q>
struct K8Cfg {
  static constexpr int NT = K8_TILE / (8 * Q);
  static constexpr int CTAS = K8_CTAS;
};

template <int W, int Q>
__global__ void __launch_bounds__(K8Cfg<Q>::NT, K8Cfg<Q>::CTAS) level_pass8_kernel(const Pass8Args a, const TabW<W>* __restrict__ tabs) {
  constexpr int T = K8_TILE;
  constexpr int NT = K8Cfg<Q>::NT;
  constexpr int R = T / Q;  // region of run k
  constexpr int NC = T / 32;
  constexpr int NW = NT / 32;
  constexpr int P = Q / 2;  // packed 16|16 scan values
  constexpr uint32_t B1 = 0x01010101u;
  extern __shared__ __align__(128) unsigned char smem[];
  // [stage | ping-pong order buffer | run table | level bits of levels 1..W-1]
  TabW<W>& tt = *reinterpret_cast<TabW<W>*>(smem + 2 * T);
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + 2 * T + sizeof(TabW<W>)) - (NC + 4);  // level j at j (NC+4)
  __shared__ __align__(16) uint32_t s_wtot[2][P][NW];
  __shared__ uint32_t s_lut[256];
  __shared__ __align__(8) uint64_t s_mbar;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint8_t* text = a.src;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * T;
  const int cnt = (int)min((int64_t)T, a.n - base);
  const bool bulk = (((uintptr_t)text) & 15) == 0 && cnt == T;
  if (tid == 0) {
    mbar_init(mbar, 1);
    fence_mbar_init();
    // the run table always comes by bulk copy, the tile when it is whole and aligned
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar),
                 "r"((uint32_t)(sizeof(TabW<W>) + (bulk ? T : 0)))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sbase + 2 * T),
                 "l"(tabs + tile), "r"((uint32_t)sizeof(TabW<W>)), "r"(mbar)
                 : "memory");
    if (bulk)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sbase),
                   "l"(text + base), "r"((uint32_t)T), "r"(mbar)
                   : "memory");
  }
  for (int i = tid; i < 256; i += NT) s_lut[i] = g_sort_lut.sel[i];
  // level W-1 is OR-ed bit by bit from the last split (order W-1 is never
  // materialised as bytes)
  for (int i = tid; i < NC + 4; i += NT) bits[(W - 1) * (NC + 4) + i] = 0u;
  if (!bulk)
    for (int p = tid; p < T; p += NT) smem[p] = p < cnt ? text[base + p] : (uint8_t)0xFF;
  bar_sync(1, NT);  // mbarrier initialised, direct staging done
  mbar_wait(mbar, 0);
  uint8_t* bits8 = reinterpret_cast<uint8_t*>(bits);

#pragma unroll
  for (int j = 0; j < W; ++j) {
    const int sh = W - 1 - j;
    const uint8_t* cur = smem + (size_t)(j & 1) * T;
    uint32_t x[2 * Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      const uint2 qv = reinterpret_cast<const uint2*>(cur + k * R)[tid];
      x[2 * k] = qv.x;
      x[2 * k + 1] = qv.y;
    }
    uint32_t m[Q], ones[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      // one multiply gathers a run's 8 flags (bits at 8i and 8i + 4 -> 24 + i, 28 + i)
      const uint32_t b0 = (x[2 * k] >> sh) & B1, b1 = (x[2 * k + 1] >> sh) & B1;
      m[k] = ((b1 * 16u + b0) * 0x01020408u) >> 24;
      ones[k] = __popc(m[k]);
      if (j > 0) bits8[j * 4 * (NC + 4) + k * (R / 8) + tid] = (uint8_t)m[k];  // level 0: hist8_kernel
    }
    if (j + 1 == W) break;
    uint32_t pk[P], incl[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      pk[p] = ones[2 * p] | (ones[2 * p + 1] << 16);
      incl[p] = warp_incl_scan(pk[p]);
      if (lane == 31) s_wtot[j & 1][p][wid] = incl[p];
    }
    bar_sync(1, NT);
    int opre[Q];
    int run_tot = 0;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint32_t wv = lane < NW ? s_wtot[j & 1][p][lane] : 0u;
      const uint32_t wpre = __reduce_add_sync(FULL, lane < wid ? wv : 0u);
      const uint32_t tot = __reduce_add_sync(FULL, wv);
      const uint32_t ex = wpre + incl[p] - pk[p];
      opre[2 * p] = run_tot + (int)(ex & 0xFFFFu);
      run_tot += (int)(tot & 0xFFFFu);
      opre[2 * p + 1] = run_tot + (int)(ex >> 16);
      run_tot += (int)(tot >> 16);
    }
    const int Z = T - run_tot;
    if (j + 2 == W) {
      // last split: only the next level's bits are needed.  The run's flags of
      // bit sh - 1 in split order (zeros part low, ones part high) are OR-ed
      // into the level W-1 bit array at the two parts' positions.
      uint32_t* LB = bits + (W - 1) * (NC + 4);
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        const uint32_t sel = s_lut[m[k]];
        const uint32_t s0 = prmt(x[2 * k], x[2 * k + 1], sel), s1 = prmt(x[2 * k], x[2 * k + 1], sel >> 16);
        const uint32_t c0 = (s0 >> (sh - 1)) & B1, c1 = (s1 >> (sh - 1)) & B1;
        const uint32_t f = ((c1 * 16u + c0) * 0x01020408u) >> 24;
        const int nz = 8 - (int)ones[k];
        const uint32_t pz = (uint32_t)(k * R + 8 * tid - opre[k]);
        const uint32_t po = (uint32_t)(Z + opre[k]);
        const uint32_t fz = f & ((1u << nz) - 1u), fo = f >> nz;
        if (fz) {
          const uint64_t v = (uint64_t)fz << (pz & 31);
          atomicOr(LB + (pz >> 5), (uint32_t)v);
          if (v >> 32) atomicOr(LB + (pz >> 5) + 1, (uint32_t)(v >> 32));
        }
        if (fo) {
          const uint64_t v = (uint64_t)fo << (po & 31);
          atomicOr(LB + (po >> 5), (uint32_t)v);
          if (v >> 32) atomicOr(LB + (po >> 5) + 1, (uint32_t)(v >> 32));
        }
      }
      break;
    }
    const uint32_t nxt = sbase + (uint32_t)((j + 1) & 1) * T;
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      const int nz = 8 - (int)ones[k];
      const uint32_t za = nxt + (uint32_t)(k * R + 8 * tid - opre[k]);
      const uint32_t oa = nxt + (uint32_t)(Z + opre[k]);
      const uint32_t sel = s_lut[m[k]];  // prmt reads selector bits 0-15
      const uint32_t sv[2] = {prmt(x[2 * k], x[2 * k + 1], sel), prmt(x[2 * k], x[2 * k + 1], sel >> 16)};
      // zeros of run k go to k R + 8 t - opre (its zeros before), ones to Z + opre
      const uint32_t zo = opaque(za);
      const uint32_t oo = opaque(oa - (uint32_t)nz);
      // address selection mostly off the integer ALU pipe (its bound): the
      // carry of (15 - nz) 2^28 + (kk + 1) 2^28 out of 32 bits is [kk >= nz],
      // read as the high word of one mad.wide; then addr = za + flag (oa - za)
      const uint32_t F = (uint32_t)(15 - nz) << 28;
      const uint32_t dz = oo - zo;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t v = sv[kk >> 2];
        const uint32_t vb = (kk & 3) == 0 ? v : (kk & 3) == 1 ? shr_mul<8>(v) : (kk & 3) == 2 ? shr_mul<16>(v) : shr_mul<24>(v);
        uint64_t t;
        asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(t) : "r"(F), "l"((uint64_t)(kk + 1) << 28));
        const uint32_t addr = zo + (uint32_t)(t >> 32) * dz + kk;
        asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(vb) : "memory");
      }
    }
    bar_sync(1, NT);
  }
  bar_sync(1, NT);  // every warp's level bits are stored
  emit_levels8<W, NC>(tt, bits, a.words, a.nwords, tid, NT, smem);  // ping-pong buffers are free now
}

// per-tile run tables, one warp per tile
template <int W>
cudaError_t launch_tiles8(const Pass8Args& a, void* tabs, cudaStream_t s) {
  constexpr size_t sm = (size_t)T8_WARPS * sizeof(Tables8);
  cudaError_t e0 = ensure_smem_attr((const void*)tiles8_kernel<W>, (int)sm);
  if (e0 != cudaSuccess) return e0;
  const int64_t blocks = std::min<int64_t>((a.ntiles + T8_WARPS - 1) / T8_WARPS, (int64_t)sm_count() * 4);
  tiles8_kernel<W><<<(unsigned)blocks, T8_WARPS * 32, sm, s>>>(a, (TabW<W>*)tabs);
  return cudaGetLastError();
}

template <int W>
cudaError_t launch_pass8(const Pass8Args& a, void* tabs, cudaStream_t s) {
  constexpr int T = K8_TILE;
  // level bits of levels 1..W-1 only (level 0 comes from hist8_kernel)
  const size_t smem = 2 * (size_t)T + sizeof(TabW<W>) + (size_t)(W - 1) * (T / 32 + 4) * 4;
  auto kern = level_pass8_kernel<W, K8_Q>;
  cudaError_t e0 = ensure_smem_attr((const void*)kern, (int)smem, true);
  if (e0 != cudaSuccess) return e0;
  kern<<<(unsigned)a.ntiles, K8Cfg<K8_Q>::NT, smem, s>>>(a, (const TabW<W>*)tabs);
  return cudaGetLastError();
}

#ifndef K8_QUAD
#define K8_QUAD 1  // two levels per shared-memory round (k8q.cuh); 0: one level per round
#endif
#include "k8q.cuh"

template <int W>
cudaError_t launch_hist8(const uint8_t* text, int64_t n, int64_t ntiles, uint32_t vmax_ok, int check,
                         uint32_t* tcnt8, uint64_t* level0, int64_t nwords, int32_t* status, cudaStream_t s) {
  constexpr size_t sb = (size_t)H8_WARPS * (1 << (W - 1)) * H8_COLS * 4;
  cudaError_t e0 = ensure_smem_attr((const void*)hist8_kernel<W>, (int)sb);
  if (e0 != cudaSuccess) return e0;
  const int per_sm = (int)std::min<size_t>(8, (size_t)(220 * 1024) / (sb + 1024));
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((ntiles + H8_WARPS - 1) / H8_WARPS,
                                                                 (int64_t)sm_count() * per_sm));
  hist8_kernel<W><<<(unsigned)blocks, H8_WARPS * 32, sb, s>>>(text, n, ntiles, vmax_ok, check, tcnt8, level0,
                                                              nwords, status);
  return cudaGetLastError();
}

// Workspace of the single-pass byte build.
struct K8Layout {
  size_t off_tcnt, off_tpre, off_chunk, off_totals, off_base, off_tabs, total;
  int64_t ntiles, nchunks;
};

inline bool k8_eligible(int sym_bytes, int w, int64_t n) {
  return sym_bytes == 1 && w >= 2 && w <= 8 && n > 0 && n < (1ll << 32) - 64;
}

inline K8Layout k8_layout(int64_t n, int w) {
  K8Layout L;
  const int nb = 1 << w;
  L.ntiles = (n + K8_TILE - 1) / K8_TILE;
  L.nchunks = (L.ntiles + S8_CHUNK - 1) / S8_CHUNK;
  size_t off = 0;
  L.off_tcnt = off;
  off = align_up(off + (size_t)L.ntiles * nb * 4, 256);
  L.off_tpre = off;
  off = align_up(off + (size_t)L.ntiles * nb * 4, 256);
  L.off_chunk = off;
  off = align_up(off + (size_t)L.nchunks * nb * 4, 256);
  L.off_totals = off;
  off = align_up(off + (size_t)nb * 8, 256);
  L.off_base = off;
  off = align_up(off + (size_t)8 * 256 * 8, 256);
  L.off_tabs = off;
  off = align_up(off + (size_t)L.ntiles * sizeof(Tab8), 256);
  L.total = off + 256;  // + status scratch
  return L;
}

// The whole single-pass build (called by build_device_impl).
int build_k8(const uint8_t* text, int64_t n, int64_t sigma, int w, int kind, uint64_t* level_words,
             int64_t* zeros, int64_t* hist, int64_t* borders, void* workspace, int32_t* status, cudaStream_t s,
             void (*pass_done)(void*, int, int), void* ctx, int lvl0, int tail_pass) {
  const K8Layout L = k8_layout(n, w);
  const int nb = 1 << w;
  unsigned char* ws = (unsigned char*)workspace;
  uint32_t* tcnt8 = (uint32_t*)(ws + L.off_tcnt);
  uint32_t* tpre8 = (uint32_t*)(ws + L.off_tpre);
  uint32_t* chunk = (uint32_t*)(ws + L.off_chunk);
  int64_t* totals = (int64_t*)(ws + L.off_totals);
  int64_t* base = (int64_t*)(ws + L.off_base);
  int32_t* st_flag = status ? status : (int32_t*)(ws + L.total - 256);
  const int64_t nwords = (n + 63) >> 6;
  cudaError_t e;
  const bool tail = tail_pass >= 0;  // the fused tail of a wider WM build (levels lvl0..)
  if (!tail) {
    g_prof.n = 0;
    prof_mark(s, -1);
  }
  // level 0 is written whole (every word) by hist8_kernel, which also zeroes
  // levels 1..w-1 (their run-edge words are OR-ed by the pass)
  if (!status) {
    e = cudaMemsetAsync(st_flag, 0, 4, s);
    if (e != cudaSuccess) return (int)e;
  }
  if (!tail) prof_mark(s, WVLT_STAGE_MEMSET);
  const uint32_t vmax_ok = (uint32_t)std::min<int64_t>(sigma - 1, 255);
  const int check = vmax_ok < 255 ? 1 : 0;
  switch (w) {
    case 2: e = launch_hist8<2>(text, n, L.ntiles, vmax_ok, check, tcnt8, level_words, nwords, st_flag, s); break;
    case 3: e = launch_hist8<3>(text, n, L.ntiles, vmax_ok, check, tcnt8, level_words, nwords, st_flag, s); break;
    case 4: e = launch_hist8<4>(text, n, L.ntiles, vmax_ok, check, tcnt8, level_words, nwords, st_flag, s); break;
    case 5: e = launch_hist8<5>(text, n, L.ntiles, vmax_ok, check, tcnt8, level_words, nwords, st_flag, s); break;
    case 6: e = launch_hist8<6>(text, n, L.ntiles, vmax_ok, check, tcnt8, level_words, nwords, st_flag, s); break;
    case 7: e = launch_hist8<7>(text, n, L.ntiles, vmax_ok, check, tcnt8, level_words, nwords, st_flag, s); break;
    default: e = launch_hist8<8>(text, n, L.ntiles, vmax_ok, check, tcnt8, level_words, nwords, st_flag, s); break;
  }
  if (e != cudaSuccess) return (int)e;
  ++g_launches;
  if (!tail) prof_mark(s, WVLT_STAGE_HIST);
  if (pass_done) pass_done(ctx, lvl0, 1);  // level 0 is final: it may leave now
  scan8_chunks_kernel<<<(unsigned)L.nchunks, nb, 0, s>>>(tcnt8, L.ntiles, nb, chunk);
  scan8_carry_kernel<<<nb, S8_SCAN_THREADS, 0, s>>>(chunk, L.nchunks, nb, totals);
  scan8_apply_kernel<<<(unsigned)L.nchunks, nb, 0, s>>>(tcnt8, L.ntiles, nb, chunk, tpre8);
  g_launches += 3;
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  if (!tail) prof_mark(s, WVLT_STAGE_SCAN0);
  tables8_kernel<<<1, 256, 0, s>>>(totals, w, kind, base, zeros, hist, nullptr, borders);
  ++g_launches;
  Pass8Args a;
  a.src = text;
  a.words = level_words;
  a.nwords = nwords;
  a.n = n;
  a.ntiles = L.ntiles;
  a.tcnt8 = tcnt8;
  a.tpre8 = tpre8;
  a.base = base;
  void* tabs = ws + L.off_tabs;  // TabW<w> per tile
  switch (w) {
    case 2: e = launch_tiles8<2>(a, tabs, s); break;
    case 3: e = launch_tiles8<3>(a, tabs, s); break;
    case 4: e = launch_tiles8<4>(a, tabs, s); break;
    case 5: e = launch_tiles8<5>(a, tabs, s); break;
    case 6: e = launch_tiles8<6>(a, tabs, s); break;
    case 7: e = launch_tiles8<7>(a, tabs, s); break;
    default: e = launch_tiles8<8>(a, tabs, s); break;
  }
  if (e != cudaSuccess) return (int)e;
  ++g_launches;
  prof_mark(s, tail ? WVLT_STAGE_SCAN0 + tail_pass : WVLT_STAGE_TABLES);
#if K8_QUAD
#define K8_PASS launch_pass8q
#else
#define K8_PASS launch_pass8
#endif
  switch (w) {
    case 2: e = K8_PASS<2>(a, tabs, s); break;
    case 3: e = K8_PASS<3>(a, tabs, s); break;
    case 4: e = K8_PASS<4>(a, tabs, s); break;
    case 5: e = K8_PASS<5>(a, tabs, s); break;
    case 6: e = K8_PASS<6>(a, tabs, s); break;
    case 7: e = K8_PASS<7>(a, tabs, s); break;
    default: e = K8_PASS<8>(a, tabs, s); break;
  }
#undef K8_PASS
  if (e != cudaSuccess) return (int)e;
  ++g_launches;
  prof_mark(s, WVLT_STAGE_PASS0 + (tail ? tail_pass : 0));
  if (pass_done) pass_done(ctx, lvl0 + 1, w - 1);
  return 0;
}

size_t k8_workspace_total(int64_t n, int w) { return k8_layout(n, w).total; }

}  // namespace
