// Fused pass for the first levels of a 2-byte WM build (10..16 live bits).
//
// The W = live - 8 levels whose digit is the high byte come from one
// shared-memory tile, as in the byte pass (k8.cuh): a split splits a run's
// 2-byte elements into a high-byte and a low-byte register pair, sorts both
// with the same PRMT selector (computed from the high bytes' flags), re-pairs
// them and stores one 16-bit element per symbol (measured: 8% faster than two
// byte planes).  After the W-th split the tile is in level-W order; each digit
// group's low bytes leave as one contiguous run of a byte text, which the
// fused byte tail (build_k8) turns into the last 8 levels.  No 2-byte
// intermediate order ever goes back to HBM.
// Included from wvlt_b200.cu after k8.cuh (same translation unit).

namespace {

#ifndef K16_TILE
#define K16_TILE 16384  // symbols per tile (run sizes / offsets fit 16 bits; measured: 8192 slower)
#endif
constexpr int K16_Q = 4;        // 8-symbol runs per thread
constexpr int K16_NT = K16_TILE / (8 * K16_Q);
#ifndef K16_CTAS
#define K16_CTAS (K16_TILE == 8192 ? 4 : 2)
#endif

// ---- K1: per-tile counts of the W-bit high-byte digit, range check, level l0 ----
// One warp per tile, the byte kernel's counter pairs; the level-l0 bits are
// the top digit bit of every symbol; the tile's words of levels l0+1..l0+W-1
// are zeroed here (the pass ORs their run-edge words).
#ifndef H16_PIPE_BATCH
#define H16_PIPE_BATCH 2  // 16-byte loads per pipelined batch of the counting kernel (measured: 2 <= 4)
#endif
template <int W>
__global__ void __launch_bounds__(H8_WARPS * 32) hist16_kernel(const uint16_t* __restrict__ src, int64_t n,
                                                              int64_t ntiles, uint32_t vmax_ok, int check,
                                                              uint32_t* __restrict__ tcnt8,
                                                              uint64_t* __restrict__ level0, int64_t nwords,
                                                              int32_t* __restrict__ status) {
  constexpr int NB = 1 << W;
  constexpr int HALF = NB / 2;
  constexpr int C = H8_COLS;  // counter columns per warp (lanes l and l + C share one)
  constexpr int WORDS = HALF * C;
  constexpr uint32_t B1 = 0x01010101u;
  extern __shared__ __align__(16) uint32_t s_cols[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* c32 = s_cols + (size_t)wid * WORDS;
  uint32_t* c32w = c32 + (lane & (C - 1));
  for (int i = lane; i < WORDS; i += 32) c32[i] = 0;
  __shared__ __align__(128) uint64_t s_zero[K16_TILE / 64];
  const uint32_t zsrc = zero_row_init<K16_TILE / 64>(s_zero);
  __syncwarp();
  uint32_t vmax = 0;
  const bool aligned = (((uintptr_t)src) & 15) == 0;
  const int64_t nwarps = (int64_t)gridDim.x * H8_WARPS;
  for (int64_t t = (int64_t)blockIdx.x * H8_WARPS + wid; t < ntiles; t += nwarps) {
    const int64_t first = t * K16_TILE;
    const int cnt = (int)min((int64_t)K16_TILE, n - first);
    // clear this tile's words of levels l0+1..l0+W-1 (the pass ORs run-edge words)
    clear_level_rows<K16_TILE / 64>(level0, nwords, first >> 6, (int)min((int64_t)(K16_TILE / 64), nwords - (first >> 6)), W,
                                    zsrc, lane);
    if (cnt == K16_TILE && aligned) {
      const uint4* v4 = reinterpret_cast<const uint4*>(src + first);  // 8 symbols per 16 bytes
      // software-pipelined: the next batch's loads are in flight while this one is counted
      constexpr int NBAT = H16_PIPE_BATCH;
      uint4 qn[NBAT];
#pragma unroll
      for (int k = 0; k < NBAT; ++k) qn[k] = __ldcs(v4 + k * 32 + lane);
#pragma unroll 1
      for (int k0 = 0; k0 < K16_TILE / 8 / 32; k0 += NBAT) {
        uint4 q[NBAT];
#pragma unroll
        for (int k = 0; k < NBAT; ++k) q[k] = qn[k];
        if (k0 + NBAT < K16_TILE / 8 / 32) {
#pragma unroll
          for (int k = 0; k < NBAT; ++k) qn[k] = __ldcs(v4 + (k0 + NBAT + k) * 32 + lane);
        }
#pragma unroll
        for (int k = 0; k < NBAT; ++k) {
          if (check) {
            vmax = __vmaxu2(vmax, q[k].x);
            vmax = __vmaxu2(vmax, q[k].y);
            vmax = __vmaxu2(vmax, q[k].z);
            vmax = __vmaxu2(vmax, q[k].w);
          }
          // the high bytes (the digits) of symbols 0-3 and 4-7
          const uint32_t hw[2] = {prmt(q[k].x, q[k].y, 0x7531), prmt(q[k].z, q[k].w, 0x7531)};
          uint32_t m8 = 0;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const uint32_t lo = hw[u] & ((uint32_t)(HALF - 1) * B1);
            const uint32_t hb = (hw[u] >> (W - 1)) & B1;
            m8 |= ((hb * 0x01020408u) >> 24) << (4 * u);
#pragma unroll
            for (int b = 0; b < 4; ++b)
              atomicAdd(c32w + prmt(lo, 0, 0x4440 + b) * C, prmt(hb, 1u, 0x5054 + (b << 8)));
          }
          // lanes 8i..8i+7 hold 64 consecutive symbols: one level-l0 word
          uint32_t m32 = m8 | (__shfl_down_sync(FULL, m8, 1) << 8);
          m32 |= __shfl_down_sync(FULL, m32, 2) << 16;
          const uint32_t hi32 = __shfl_down_sync(FULL, m32, 4);
          if ((lane & 7) == 0)
            level0[(first >> 6) + ((k0 + k) * 32 + lane) / 8] = (uint64_t)m32 | ((uint64_t)hi32 << 32);
        }
      }
    } else {
      uint32_t* l0 = reinterpret_cast<uint32_t*>(level0) + (first >> 5);
      for (int i0 = 0; i0 < cnt; i0 += 32) {
        const int i = i0 + lane;
        uint32_t v = 0;
        if (i < cnt) {
          v = src[first + i];
          vmax = max(vmax, v);
          const uint32_t d = v >> 8;
          atomicAdd(c32w + (d & (HALF - 1)) * C, ((d >> (W - 1)) & 1u) ? 0x10001u : 1u);
        }
        const uint32_t b = __ballot_sync(FULL, i < cnt && (((v >> 8) >> (W - 1)) & 1u));
        if (lane == 0) l0[i0 >> 5] = b;
      }
      if (lane == 0 && (((first + cnt + 31) >> 5) & 1)) l0[(cnt + 31) >> 5] = 0u;
    }
    __syncwarp();
    uint32_t* row_out = tcnt8 + t * NB;
    for (int p = lane; p < HALF; p += 32) {
      const uint4* row = reinterpret_cast<const uint4*>(c32 + p * C);
      uint32_t s = 0;
#pragma unroll
      for (int k = 0; k < C / 4; ++k) {
        const uint4 qq = row[k ^ (lane & (C / 4 - 1))];
        s += (qq.x + qq.y) + (qq.z + qq.w);
      }
      row_out[p] = (s & 0xFFFFu) - (s >> 16);
      row_out[p + HALF] = s >> 16;
    }
    __syncwarp();
    for (int i = lane * 4; i < WORDS; i += 128) *reinterpret_cast<uint4*>(c32 + i) = make_uint4(0, 0, 0, 0);
    __syncwarp();
  }
  if (check) {
    vmax = max(vmax & 0xFFFFu, vmax >> 16);
    if (vmax > vmax_ok) atomicOr(status, WVLT_STATUS_RANGE);
  }
  zero_row_drain(lane);  // the zero row must outlive the bulk stores that read it
}

// ---- K3: the fused 2-byte pass ----
struct Pass16Args {
  const uint16_t* src;
  uint8_t* out;           // low bytes in level-W order (the byte tail's text)
  uint64_t* words;        // level l0 (levels l0+1.. follow at nwords strides)
  int64_t nwords, n, ntiles;
  const uint32_t* tcnt8;  // [tile][2^W] digit counts
  const uint32_t* tpre8;  // [tile][2^W] digit prefixes over earlier tiles
  const int64_t* baseW;   // [2^W] level-W group starts, LSD-digit order
};

template <int W>
__global__ void __launch_bounds__(K16_NT, K16_CTAS) level_pass16_kernel(const Pass16Args a,
                                                                        const TabW<W>* __restrict__ tabs) {
  constexpr int T = K16_TILE;
  constexpr int NT = K16_NT;
  constexpr int Q = K16_Q;
  constexpr int R = T / Q;
  constexpr int NC = T / 32;
  constexpr int NW = NT / 32;
  constexpr int NB = 1 << W;
  constexpr int P = Q / 2;
  constexpr uint32_t B1 = 0x01010101u;
  extern __shared__ __align__(128) unsigned char smem[];
  // [buffer 0: staged tile, then orders 2, 4, .. (2-byte elements)
  //  | buffer 1: orders 1, 3, .. | run table | level bits of levels 1..W-1]
  TabW<W>& tt = *reinterpret_cast<TabW<W>*>(smem + 4 * T);
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + 4 * T + sizeof(TabW<W>)) - (NC + 4);
  __shared__ __align__(16) uint32_t s_wtot[2][P][NW];
  __shared__ uint32_t s_tmp[NW];
  __shared__ uint32_t s_lut[256];
  __shared__ uint32_t s_gW[NB];
  __shared__ uint16_t s_cW[NB], s_lsW[NB];
  __shared__ __align__(8) uint64_t s_mbar;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * T;
  const int cnt = (int)min((int64_t)T, a.n - base);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
  const bool bulk = (((uintptr_t)a.src) & 15) == 0 && cnt == T;
  if (tid == 0) {
    mbar_init(mbar, 1);
    fence_mbar_init();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar),
                 "r"((uint32_t)(sizeof(TabW<W>) + (bulk ? 2 * T : 0)))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sbase + 4 * T),
                 "l"(tabs + tile), "r"((uint32_t)sizeof(TabW<W>)), "r"(mbar)
                 : "memory");
    if (bulk)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sbase),
                   "l"(a.src + base), "r"((uint32_t)(2 * T)), "r"(mbar)
                   : "memory");
  }
  for (int i = tid; i < 256; i += NT) s_lut[i] = g_sort_lut.sel[i];
  // level-W groups of this tile: sizes, global starts (LSD digit d = rev(e))
  uint32_t cw = 0;
  if (tid < NB) {
    const int d = (int)rev_bits((unsigned)tid, W);
    cw = __ldg(a.tcnt8 + tile * NB + tid);
    s_cW[d] = (uint16_t)cw;
    s_gW[d] = (uint32_t)(__ldg(a.baseW + d) + (int64_t)__ldg(a.tpre8 + tile * NB + tid));
  }
  if (!bulk) {
    uint16_t* st = reinterpret_cast<uint16_t*>(smem);
    for (int p = tid; p < T; p += NT) st[p] = p < cnt ? a.src[base + p] : (uint16_t)0xFFFF;
  }
  bar_sync(1, NT);  // mbarrier initialised, direct staging done, level-W sizes stored
  {
    // tile-local level-W group starts: exclusive prefix of s_cW in LSD order
    const uint32_t v = tid < NB ? (uint32_t)s_cW[tid] : 0u;
    const uint32_t incl = warp_incl_scan(v);
    if (lane == 31) s_tmp[wid] = incl;
    bar_sync(1, NT);
    const uint32_t wv = lane < NW ? s_tmp[lane] : 0u;
    const uint32_t wpre = __reduce_add_sync(FULL, lane < wid ? wv : 0u);
    if (tid < NB) s_lsW[tid] = (uint16_t)(wpre + incl - v);
  }
  mbar_wait(mbar, 0);
  uint8_t* bits8 = reinterpret_cast<uint8_t*>(bits);

#pragma unroll
  for (int j = 0; j < W; ++j) {
    const int sh = W - 1 - j;
    uint32_t x[2 * Q], y[2 * Q];  // high / low bytes of the thread's runs
    {
      const unsigned char* cur = smem + (size_t)(j & 1) * 2 * T;
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        const uint4 qv = reinterpret_cast<const uint4*>(cur + 2 * (k * R))[tid];
        x[2 * k] = prmt(qv.x, qv.y, 0x7531);
        x[2 * k + 1] = prmt(qv.z, qv.w, 0x7531);
        y[2 * k] = prmt(qv.x, qv.y, 0x6420);
        y[2 * k + 1] = prmt(qv.z, qv.w, 0x6420);
      }
    }
    uint32_t m[Q], ones[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      const uint32_t b0 = (x[2 * k] >> sh) & B1, b1 = (x[2 * k + 1] >> sh) & B1;
      m[k] = ((b1 * 16u + b0) * 0x01020408u) >> 24;
      ones[k] = __popc(m[k]);
      if (j > 0) bits8[j * 4 * (NC + 4) + k * (R / 8) + tid] = (uint8_t)m[k];  // level 0: hist16_kernel
    }
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
    // order j + 1 into buffer (j + 1) & 1
    const uint32_t nxt = sbase + (uint32_t)((j + 1) & 1) * 2 * T;
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      const uint32_t sel = s_lut[m[k]];
      const uint32_t h0 = prmt(x[2 * k], x[2 * k + 1], sel), h1 = prmt(x[2 * k], x[2 * k + 1], sel >> 16);
      const uint32_t l0 = prmt(y[2 * k], y[2 * k + 1], sel), l1 = prmt(y[2 * k], y[2 * k + 1], sel >> 16);
      const uint32_t e[4] = {prmt(l0, h0, 0x5140), prmt(l0, h0, 0x7362), prmt(l1, h1, 0x5140), prmt(l1, h1, 0x7362)};
      const int nz = 8 - (int)ones[k];
      const uint32_t za = opaque(nxt + 2u * (uint32_t)(k * R + 8 * tid - opre[k]));
      const uint32_t oa = opaque(nxt + 2u * (uint32_t)(Z + opre[k] - nz));
      const uint32_t F = (uint32_t)(15 - nz) << 28;
      const uint32_t dz = oa - za;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint64_t t;
        asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(t) : "r"(F), "l"((uint64_t)(kk + 1) << 28));
        const uint32_t addr = za + (uint32_t)(t >> 32) * dz + 2 * kk;
        const uint32_t v = (kk & 1) ? (e[kk >> 1] >> 16) : e[kk >> 1];
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
      }
    }
    bar_sync(1, NT);
  }
  // levels 1..W-1 as flattened destination-word tasks (as in the byte pass)
  emit_levels8<W, NC>(tt, bits, a.words, a.nwords, tid, NT, smem + (size_t)((W + 1) & 1) * 2 * T);
  // the low bytes of each level-W group: one contiguous run of the byte text
  const uint8_t* lo = smem + (size_t)(W & 1) * 2 * T;
  constexpr int LS = 2;  // low byte of element p at byte 2 p
  for (int r = wid; r < NB; r += NW) {
    const int c = s_cW[r];
    if (!c) continue;
    uint8_t* dst = a.out + s_gW[r];
    const uint8_t* sp = lo + LS * s_lsW[r];
    for (int i = lane; i < c; i += 32) dst[i] = sp[LS * i];
  }
}

template <int W>
cudaError_t launch_hist16(const uint16_t* src, int64_t n, int64_t ntiles, uint32_t vmax_ok, int check,
                          uint32_t* tcnt8, uint64_t* level0, int64_t nwords, int32_t* status, cudaStream_t s) {
  constexpr size_t sb = (size_t)H8_WARPS * (1 << (W - 1)) * H8_COLS * 4;
  cudaError_t e0 = ensure_smem_attr((const void*)hist16_kernel<W>, (int)sb);
  if (e0 != cudaSuccess) return e0;
  const int per_sm = (int)std::min<size_t>(8, (size_t)(220 * 1024) / (sb + 1024));
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((ntiles + H8_WARPS - 1) / H8_WARPS,
                                                                 (int64_t)sm_count() * per_sm));
  hist16_kernel<W><<<(unsigned)blocks, H8_WARPS * 32, sb, s>>>(src, n, ntiles, vmax_ok, check, tcnt8, level0,
                                                               nwords, status);
  return cudaGetLastError();
}

template <int W>
cudaError_t launch_pass16(const Pass16Args& a, const void* tabs, cudaStream_t s) {
  constexpr int T = K16_TILE;
  const size_t smem = 4 * (size_t)T + sizeof(TabW<W>) + (size_t)(W - 1) * (T / 32 + 4) * 4;
  auto kern = level_pass16_kernel<W>;
  cudaError_t e0 = ensure_smem_attr((const void*)kern, (int)smem, true);
  if (e0 != cudaSuccess) return e0;
  kern<<<(unsigned)a.ntiles, K16_NT, smem, s>>>(a, (const TabW<W>*)tabs);
  return cudaGetLastError();
}

}  // namespace
#ifndef K16_QUAD
#define K16_QUAD 1  // even widths: two levels per shared-memory round (k16q.cuh)
#endif
#include "k16q.cuh"
namespace {

// Workspace of the 2-byte fused pass (its tables; the byte output is separate).
struct K16Layout {
  size_t off_tcnt, off_tpre, off_chunk, off_totals, off_base, off_baseW, off_tabs, total;
  int64_t ntiles, nchunks;
};

inline K16Layout k16_layout(int64_t n, int w, int tile = K16_TILE) {
  K16Layout L;
  const int nb = 1 << w;
  L.ntiles = (n + tile - 1) / tile;
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
  L.off_baseW = off;
  off = align_up(off + (size_t)256 * 8, 256);
  L.off_tabs = off;
  off = align_up(off + (size_t)L.ntiles * sizeof(Tab8), 256);
  L.total = off;
  return L;
}

// Levels lvl0 .. lvl0 + W - 1 of a WM build from a 2-byte text with 8 + W live
// bits (2 <= W <= 8); the low bytes leave in level-(lvl0 + W) order in `out`.
int build_k16(const uint16_t* src, int64_t n, int W, uint64_t* level_words, int64_t* zeros, uint8_t* out,
              void* workspace, int32_t* st_flag, uint32_t vmax_ok, int check, cudaStream_t s,
              void (*pass_done)(void*, int, int), void* ctx, int lvl0, int stage_pass) {
  const K16Layout L = k16_layout(n, W);
  const int nb = 1 << W;
  unsigned char* ws = (unsigned char*)workspace;
  uint32_t* tcnt8 = (uint32_t*)(ws + L.off_tcnt);
  uint32_t* tpre8 = (uint32_t*)(ws + L.off_tpre);
  uint32_t* chunk = (uint32_t*)(ws + L.off_chunk);
  int64_t* totals = (int64_t*)(ws + L.off_totals);
  int64_t* base = (int64_t*)(ws + L.off_base);
  int64_t* baseW = (int64_t*)(ws + L.off_baseW);
  void* tabs = ws + L.off_tabs;  // TabW<W> per tile
  const int64_t nwords = (n + 63) >> 6;
  cudaError_t e;
  switch (W) {
#define WVLT_K16H(WW) \
  case WW: e = launch_hist16<WW>(src, n, L.ntiles, vmax_ok, check, tcnt8, level_words, nwords, st_flag, s); break;
    WVLT_K16H(2) WVLT_K16H(3) WVLT_K16H(4) WVLT_K16H(5) WVLT_K16H(6) WVLT_K16H(7) WVLT_K16H(8)
#undef WVLT_K16H
    default: return WVLT_E_ARG;
  }
  if (e != cudaSuccess) return (int)e;
  ++g_launches;
  if (pass_done) pass_done(ctx, lvl0, 1);
  scan8_chunks_kernel<<<(unsigned)L.nchunks, nb, 0, s>>>(tcnt8, L.ntiles, nb, chunk);
  scan8_carry_kernel<<<nb, S8_SCAN_THREADS, 0, s>>>(chunk, L.nchunks, nb, totals);
  scan8_apply_kernel<<<(unsigned)L.nchunks, nb, 0, s>>>(tcnt8, L.ntiles, nb, chunk, tpre8);
  tables8_kernel<<<1, 256, 0, s>>>(totals, W, WVLT_KIND_WM, base, zeros, nullptr, baseW, nullptr);
  g_launches += 4;
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  Pass8Args t;
  t.src = nullptr;
  t.words = level_words;
  t.nwords = nwords;
  t.n = n;
  t.ntiles = L.ntiles;
  t.tcnt8 = tcnt8;
  t.tpre8 = tpre8;
  t.base = base;
  switch (W) {
#define WVLT_K16T(WW) \
  case WW: e = launch_tiles8<WW>(t, tabs, s); break;
    WVLT_K16T(2) WVLT_K16T(3) WVLT_K16T(4) WVLT_K16T(5) WVLT_K16T(6) WVLT_K16T(7) WVLT_K16T(8)
#undef WVLT_K16T
  }
  if (e != cudaSuccess) return (int)e;
  ++g_launches;
  prof_mark(s, WVLT_STAGE_SCAN0 + stage_pass);
  Pass16Args a;
  a.src = src;
  a.out = out;
  a.words = level_words;
  a.nwords = nwords;
  a.n = n;
  a.ntiles = L.ntiles;
  a.tcnt8 = tcnt8;
  a.tpre8 = tpre8;
  a.baseW = baseW;
  switch (W) {
#define WVLT_K16P(WW) \
  case WW: e = (K16_QUAD && (WW % 2 == 0)) ? launch_pass16q<(WW % 2 == 0 ? WW : 2)>(a, tabs, s) : launch_pass16<WW>(a, tabs, s); break;
    WVLT_K16P(2) WVLT_K16P(3) WVLT_K16P(4) WVLT_K16P(5) WVLT_K16P(6) WVLT_K16P(7) WVLT_K16P(8)
#undef WVLT_K16P
  }
  if (e != cudaSuccess) return (int)e;
  ++g_launches;
  prof_mark(s, WVLT_STAGE_PASS0 + stage_pass);
  if (pass_done) pass_done(ctx, lvl0 + 1, W - 1);
  return 0;
}

size_t k16_workspace_total(int64_t n, int w) { return k16_layout(n, w).total; }

}  // namespace
