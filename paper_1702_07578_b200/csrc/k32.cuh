// Fused pass for the first levels of a 4-byte WM build (18..24 live bits).
//
// The W = live - 16 levels whose digit is byte 2 of every symbol come from one
// shared-memory tile of 4-byte elements (as k16.cuh does for 2-byte ones): a
// split transposes a run's 8 elements into three byte planes (digit, low and
// high payload byte), sorts the planes with one PRMT selector from the digit
// flags, transposes back and stores one 4-byte element per symbol.  The last
// split keeps only the 2-byte payload; after it every level-W digit group's
// payloads leave as one contiguous run of the 2-byte text the fused 2-byte pass
// (build_k16) continues with.  Included from wvlt_b200.cu after k16.cuh.

namespace {

#ifndef K32_TILE
#define K32_TILE 8192
#endif
constexpr int K32_Q = 4;  // 8-symbol runs per thread
constexpr int K32_NT = K32_TILE / (8 * K32_Q);
#ifndef K32_CTAS
#define K32_CTAS 3
#endif

// ---- K1: per-tile counts of the W-bit digit (byte 2), range check, level l0 ----
#ifndef H32_PIPE_BATCH
#define H32_PIPE_BATCH 2  // 16-byte loads per pipelined batch of the counting kernel (measured: 2 < 4)
#endif
template <int W>
__global__ void __launch_bounds__(H8_WARPS * 32) hist32_kernel(const uint32_t* __restrict__ src, int64_t n,
                                                              int64_t ntiles, uint32_t vmax_ok, int check,
                                                              uint32_t* __restrict__ tcnt8,
                                                              uint64_t* __restrict__ level0, int64_t nwords,
                                                              int32_t* __restrict__ status) {
  constexpr int NB = 1 << W;
  constexpr int HALF = NB / 2;
  constexpr int C = H8_COLS;
  constexpr int WORDS = HALF * C;
  constexpr uint32_t B1 = 0x01010101u;
  extern __shared__ __align__(16) uint32_t s_cols[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* c32 = s_cols + (size_t)wid * WORDS;
  uint32_t* c32w = c32 + (lane & (C - 1));
  for (int i = lane; i < WORDS; i += 32) c32[i] = 0;
  __shared__ __align__(128) uint64_t s_zero[K32_TILE / 64];
  const uint32_t zsrc = zero_row_init<K32_TILE / 64>(s_zero);
  __syncwarp();
  uint32_t vmax = 0;
  const bool aligned = (((uintptr_t)src) & 15) == 0;
  const int64_t nwarps = (int64_t)gridDim.x * H8_WARPS;
  for (int64_t t = (int64_t)blockIdx.x * H8_WARPS + wid; t < ntiles; t += nwarps) {
    const int64_t first = t * K32_TILE;
    const int cnt = (int)min((int64_t)K32_TILE, n - first);
    // clear this tile's words of levels l0+1..l0+W-1 (the pass ORs run-edge words)
    clear_level_rows<K32_TILE / 64>(level0, nwords, first >> 6, (int)min((int64_t)(K32_TILE / 64), nwords - (first >> 6)), W,
                                    zsrc, lane);
    if (cnt == K32_TILE && aligned) {
      const uint4* v4 = reinterpret_cast<const uint4*>(src + first);  // 4 symbols per 16 bytes
      // software-pipelined: the next batch's loads are in flight while this one is counted
      constexpr int NBAT = H32_PIPE_BATCH;
      uint4 qn[NBAT];
#pragma unroll
      for (int k = 0; k < NBAT; ++k) qn[k] = __ldcs(v4 + k * 32 + lane);
#pragma unroll 1
      for (int k0 = 0; k0 < K32_TILE / 4 / 32; k0 += NBAT) {
        uint4 q[NBAT];
#pragma unroll
        for (int k = 0; k < NBAT; ++k) q[k] = qn[k];
        if (k0 + NBAT < K32_TILE / 4 / 32) {
#pragma unroll
          for (int k = 0; k < NBAT; ++k) qn[k] = __ldcs(v4 + (k0 + NBAT + k) * 32 + lane);
        }
#pragma unroll
        for (int k = 0; k < NBAT; ++k) {
          if (check) vmax = max(max(vmax, max(q[k].x, q[k].y)), max(q[k].z, q[k].w));
          // byte 2 (the digit) of the four symbols
          const uint32_t d4 = prmt(prmt(q[k].x, q[k].y, 0x0062), prmt(q[k].z, q[k].w, 0x0062), 0x5410);
          const uint32_t lo = d4 & ((uint32_t)(HALF - 1) * B1);
          const uint32_t hb = (d4 >> (W - 1)) & B1;
          const uint32_t m4 = (hb * 0x01020408u) >> 24;
#pragma unroll
          for (int b = 0; b < 4; ++b)
            atomicAdd(c32w + prmt(lo, 0, 0x4440 + b) * C, prmt(hb, 1u, 0x5054 + (b << 8)));
          // lanes 16i..16i+15 hold 64 consecutive symbols: one level-l0 word
          uint32_t m = m4 | (__shfl_down_sync(FULL, m4, 1) << 4);
          m |= __shfl_down_sync(FULL, m, 2) << 8;
          m |= __shfl_down_sync(FULL, m, 4) << 16;
          const uint32_t hi32 = __shfl_down_sync(FULL, m, 8);
          if ((lane & 15) == 0)
            level0[(first >> 6) + ((k0 + k) * 32 + lane) / 16] = (uint64_t)m | ((uint64_t)hi32 << 32);
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
          const uint32_t d = (v >> 16) & 0xFFu;
          atomicAdd(c32w + (d & (HALF - 1)) * C, ((d >> (W - 1)) & 1u) ? 0x10001u : 1u);
        }
        const uint32_t b = __ballot_sync(FULL, i < cnt && (((v >> 16) >> (W - 1)) & 1u));
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
  if (check && vmax > vmax_ok) atomicOr(status, WVLT_STATUS_RANGE);
  zero_row_drain(lane);  // the zero row must outlive the bulk stores that read it
}

// ---- K3: the fused 4-byte pass ----
struct Pass32Args {
  const uint32_t* src;
  uint16_t* out;          // 2-byte payloads in level-W order (the 2-byte pass's text)
  uint64_t* words;        // level l0 (levels l0+1.. follow at nwords strides)
  int64_t nwords, n, ntiles;
  const uint32_t* tcnt8;
  const uint32_t* tpre8;
  const int64_t* baseW;
};

// four elements -> byte planes 0, 1, 2 (one byte per element each)
__device__ __forceinline__ void planes4(uint32_t e0, uint32_t e1, uint32_t e2, uint32_t e3, uint32_t& p0,
                                        uint32_t& p1, uint32_t& p2) {
  const uint32_t a = prmt(e0, e1, 0x5140), b = prmt(e2, e3, 0x5140);  // (e0.0 e1.0 e0.1 e1.1), (e2 e3 ..)
  const uint32_t c = prmt(e0, e1, 0x7362), d = prmt(e2, e3, 0x7362);  // bytes 2, 3
  p0 = prmt(a, b, 0x5410);
  p1 = prmt(a, b, 0x7632);
  p2 = prmt(c, d, 0x5410);
}

template <int W>
__global__ void __launch_bounds__(K32_NT, K32_CTAS) level_pass32_kernel(const Pass32Args a,
                                                                        const TabW<W>* __restrict__ tabs) {
  constexpr int T = K32_TILE;
  constexpr int NT = K32_NT;
  constexpr int Q = K32_Q;
  constexpr int R = T / Q;
  constexpr int NC = T / 32;
  constexpr int NW = NT / 32;
  constexpr int NB = 1 << W;
  constexpr int P = Q / 2;
  constexpr uint32_t B1 = 0x01010101u;
  extern __shared__ __align__(128) unsigned char smem[];
  // [buffer 0: staged tile, then orders 2, 4, .. (4-byte elements; the last
  //  order 2-byte payloads) | buffer 1: orders 1, 3, .. | run table | level bits]
  TabW<W>& tt = *reinterpret_cast<TabW<W>*>(smem + 8 * T);
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + 8 * T + sizeof(TabW<W>)) - (NC + 4);
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
                 "r"((uint32_t)(sizeof(TabW<W>) + (bulk ? 4 * T : 0)))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sbase + 8 * T),
                 "l"(tabs + tile), "r"((uint32_t)sizeof(TabW<W>)), "r"(mbar)
                 : "memory");
    if (bulk)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sbase),
                   "l"(a.src + base), "r"((uint32_t)(4 * T)), "r"(mbar)
                   : "memory");
  }
  for (int i = tid; i < 256; i += NT) s_lut[i] = g_sort_lut.sel[i];
  if (tid < NB) {
    const int d = (int)rev_bits((unsigned)tid, W);
    s_cW[d] = (uint16_t)__ldg(a.tcnt8 + tile * NB + tid);
    s_gW[d] = (uint32_t)(__ldg(a.baseW + d) + (int64_t)__ldg(a.tpre8 + tile * NB + tid));
  }
  if (!bulk) {
    uint32_t* st = reinterpret_cast<uint32_t*>(smem);
    for (int p = tid; p < T; p += NT) st[p] = p < cnt ? a.src[base + p] : 0x00FFFFFFu;
  }
  bar_sync(1, NT);
  {
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
    uint32_t p0[2 * Q], p1[2 * Q], x[2 * Q];  // byte planes: payload low / high, digit
    {
      const unsigned char* cur = smem + (size_t)(j & 1) * 4 * T;
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        const uint4 q0 = reinterpret_cast<const uint4*>(cur + 4 * (k * R))[2 * tid];
        const uint4 q1 = reinterpret_cast<const uint4*>(cur + 4 * (k * R))[2 * tid + 1];
        planes4(q0.x, q0.y, q0.z, q0.w, p0[2 * k], p1[2 * k], x[2 * k]);
        planes4(q1.x, q1.y, q1.z, q1.w, p0[2 * k + 1], p1[2 * k + 1], x[2 * k + 1]);
      }
    }
    uint32_t m[Q], ones[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      const uint32_t b0 = (x[2 * k] >> sh) & B1, b1 = (x[2 * k + 1] >> sh) & B1;
      m[k] = ((b1 * 16u + b0) * 0x01020408u) >> 24;
      ones[k] = __popc(m[k]);
      if (j > 0) bits8[j * 4 * (NC + 4) + k * (R / 8) + tid] = (uint8_t)m[k];  // level 0: hist32_kernel
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
    const uint32_t nxt = sbase + (uint32_t)((j + 1) & 1) * 4 * T;
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      const uint32_t sel = s_lut[m[k]];
      const uint32_t a0 = prmt(p0[2 * k], p0[2 * k + 1], sel), a1 = prmt(p0[2 * k], p0[2 * k + 1], sel >> 16);
      const uint32_t c0 = prmt(p1[2 * k], p1[2 * k + 1], sel), c1 = prmt(p1[2 * k], p1[2 * k + 1], sel >> 16);
      // payload pairs (low, high) of the sorted elements 0-1, 2-3, 4-5, 6-7
      const uint32_t u[4] = {prmt(a0, c0, 0x5140), prmt(a0, c0, 0x7362), prmt(a1, c1, 0x5140), prmt(a1, c1, 0x7362)};
      const int nz = 8 - (int)ones[k];
      const uint32_t F = (uint32_t)(15 - nz) << 28;
      if (j + 1 < W) {
        const uint32_t d0 = prmt(x[2 * k], x[2 * k + 1], sel), d1 = prmt(x[2 * k], x[2 * k + 1], sel >> 16);
        // elements (payload | digit << 16)
        const uint32_t e[8] = {prmt(u[0], d0, 0x0410), prmt(u[0], d0, 0x0532), prmt(u[1], d0, 0x0610),
                               prmt(u[1], d0, 0x0732), prmt(u[2], d1, 0x0410), prmt(u[2], d1, 0x0532),
                               prmt(u[3], d1, 0x0610), prmt(u[3], d1, 0x0732)};
        const uint32_t za = opaque(nxt + 4u * (uint32_t)(k * R + 8 * tid - opre[k]));
        const uint32_t oa = opaque(nxt + 4u * (uint32_t)(Z + opre[k] - nz));
        const uint32_t dz = oa - za;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          uint64_t t;
          asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(t) : "r"(F), "l"((uint64_t)(kk + 1) << 28));
          const uint32_t addr = za + (uint32_t)(t >> 32) * dz + 4 * kk;
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(e[kk]) : "memory");
        }
      } else {
        // last split: only the 2-byte payloads (level-W order) are kept
        const uint32_t za = opaque(nxt + 2u * (uint32_t)(k * R + 8 * tid - opre[k]));
        const uint32_t oa = opaque(nxt + 2u * (uint32_t)(Z + opre[k] - nz));
        const uint32_t dz = oa - za;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          uint64_t t;
          asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(t) : "r"(F), "l"((uint64_t)(kk + 1) << 28));
          const uint32_t addr = za + (uint32_t)(t >> 32) * dz + 2 * kk;
          const uint32_t v = (kk & 1) ? (u[kk >> 1] >> 16) : u[kk >> 1];
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
        }
      }
    }
    bar_sync(1, NT);
  }
  emit_levels8<W, NC>(tt, bits, a.words, a.nwords, tid, NT, smem + (size_t)((W + 1) & 1) * 4 * T);
  // each level-W digit group's payloads: one contiguous run of the 2-byte text
  const uint16_t* pay = reinterpret_cast<const uint16_t*>(smem + (size_t)(W & 1) * 4 * T);
  for (int r = wid; r < NB; r += NW) {
    const int c = s_cW[r];
    if (!c) continue;
    uint16_t* dst = a.out + s_gW[r];
    const uint16_t* sp = pay + s_lsW[r];
    for (int i = lane; i < c; i += 32) dst[i] = sp[i];
  }
}

template <int W>
cudaError_t launch_hist32(const uint32_t* src, int64_t n, int64_t ntiles, uint32_t vmax_ok, int check,
                          uint32_t* tcnt8, uint64_t* level0, int64_t nwords, int32_t* status, cudaStream_t s) {
  constexpr size_t sb = (size_t)H8_WARPS * (1 << (W - 1)) * H8_COLS * 4;
  cudaError_t e0 = ensure_smem_attr((const void*)hist32_kernel<W>, (int)sb);
  if (e0 != cudaSuccess) return e0;
  const int per_sm = (int)std::min<size_t>(8, (size_t)(220 * 1024) / (sb + 1024));
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((ntiles + H8_WARPS - 1) / H8_WARPS,
                                                                 (int64_t)sm_count() * per_sm));
  hist32_kernel<W><<<(unsigned)blocks, H8_WARPS * 32, sb, s>>>(src, n, ntiles, vmax_ok, check, tcnt8, level0,
                                                               nwords, status);
  return cudaGetLastError();
}

template <int W>
cudaError_t launch_pass32(const Pass32Args& a, const void* tabs, cudaStream_t s) {
  constexpr int T = K32_TILE;
  const size_t smem = 8 * (size_t)T + sizeof(TabW<W>) + (size_t)(W - 1) * (T / 32 + 4) * 4;
  auto kern = level_pass32_kernel<W>;
  cudaError_t e0 = ensure_smem_attr((const void*)kern, (int)smem, true);
  if (e0 != cudaSuccess) return e0;
  kern<<<(unsigned)a.ntiles, K32_NT, smem, s>>>(a, (const TabW<W>*)tabs);
  return cudaGetLastError();
}

// Levels lvl0 .. lvl0 + W - 1 of a WM build from a 4-byte text with 16 + W live
// bits (2 <= W <= 8); the 2-byte payloads leave in level-(lvl0 + W) order in `out`.
int build_k32(const uint32_t* src, int64_t n, int W, uint64_t* level_words, int64_t* zeros, uint16_t* out,
              void* workspace, int32_t* st_flag, uint32_t vmax_ok, int check, cudaStream_t s,
              void (*pass_done)(void*, int, int), void* ctx, int lvl0, int stage_pass) {
  const K16Layout L = k16_layout(n, W, K32_TILE);
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
#define WVLT_K32H(WW) \
  case WW: e = launch_hist32<WW>(src, n, L.ntiles, vmax_ok, check, tcnt8, level_words, nwords, st_flag, s); break;
    WVLT_K32H(2) WVLT_K32H(3) WVLT_K32H(4) WVLT_K32H(5) WVLT_K32H(6) WVLT_K32H(7) WVLT_K32H(8)
#undef WVLT_K32H
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
#define WVLT_K32T(WW) \
  case WW: e = launch_tiles8<WW>(t, tabs, s); break;
    WVLT_K32T(2) WVLT_K32T(3) WVLT_K32T(4) WVLT_K32T(5) WVLT_K32T(6) WVLT_K32T(7) WVLT_K32T(8)
#undef WVLT_K32T
  }
  if (e != cudaSuccess) return (int)e;
  ++g_launches;
  prof_mark(s, WVLT_STAGE_SCAN0 + stage_pass);
  Pass32Args a;
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
#define WVLT_K32P(WW) \
  case WW: e = launch_pass32<WW>(a, tabs, s); break;
    WVLT_K32P(2) WVLT_K32P(3) WVLT_K32P(4) WVLT_K32P(5) WVLT_K32P(6) WVLT_K32P(7) WVLT_K32P(8)
#undef WVLT_K32P
  }
  if (e != cudaSuccess) return (int)e;
  ++g_launches;
  prof_mark(s, WVLT_STAGE_PASS0 + stage_pass);
  if (pass_done) pass_done(ctx, lvl0 + 1, W - 1);
  return 0;
}

size_t k32_workspace_total(int64_t n, int w) { return k16_layout(n, w, K32_TILE).total; }

}  // namespace
