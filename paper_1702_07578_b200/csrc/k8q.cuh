// K8Q: the fused byte pass with TWO levels per shared-memory round.
//
// Same contract as level_pass8_kernel (k8.cuh): one CTA per K8_TILE-symbol
// tile, every level's tile-local bits in shared memory, emitted at the end as
// whole destination words.  What changes is how the tile-local orders are
// produced.  A round starting at order A_j (bytes in shared memory):
//
//   * L_j   = the b_j flags of A_j                       (one byte per 8-symbol run)
//   * A_j+2 = A_j stably sorted by the class c = 2 b_j+1 + b_j: ONE 4-way byte
//             scatter instead of two 2-way ones (A_j+1 is never materialised)
//   * L_j+1 = b_j+1 over A_j+1 = [b_j+1 of A_j's b_j-zeros] ++ [... of its ones]:
//             each run already sorts its 8 bytes by b_j (PRMT) for the scatter,
//             so its contribution is the run's sorted b_j+1 flags g split at its
//             zero count z -- two bit pieces.  They are concatenated after the
//             round by threads that own 4 CONSECUTIVE runs (lane-sequential
//             shifts into a 32-bit accumulator per stream, then one OR per
//             stream word into the level's bit array), instead of a bit scatter
//             per run.
//
// Per two levels this halves the byte scatters (the shared-memory store
// wavefronts that bound the one-level-per-round kernel), at the price of a
// second PRMT sort, a 3-class count scan and the concatenation.  The last
// round of an even width only emits L_W-2 and L_W-1 (no scatter), the last of
// an odd width only L_W-1.
//
// 4-way store addressing: the class-sorted run's byte kk goes to
// D[c(kk)] + kk, with the four per-run bases D (16-bit offsets inside the
// destination buffer, < T <= 32768) packed in two registers; one PRMT builds a
// byte's selector from its 2-bit class (nibbles 2c', 2c'+1, and 9 = the sign
// of a high byte < 0x80, i.e. zero, for the upper half), one PRMT looks the
// base up.  The buffer's shared-window address rides in the store's
// uniform-register + immediate operands.
//
// Included from k8.cuh (same translation unit, anonymous namespace).

#ifndef K8Q_LUT
// copies of the sort LUT, interleaved (entry e of copy c at e K8Q_LUT + c, lane
// l reads copy l % K8Q_LUT): a warp's 32 random lookups spread over 32 / K8Q_LUT
// lanes per copy, each copy on its own banks
#define K8Q_LUT 1  // (measured: 4 interleaved copies slower, 2.85 vs 2.82 ms on c2)
#endif

template <int W>
struct Q8Smem {
  static constexpr int T = K8_TILE;
  static constexpr int NC = T / 32;
  static constexpr size_t bits = 2 * (size_t)T;                             // levels 1..W-1, NC + 4 words each
  static constexpr size_t gbuf = bits + (size_t)(W - 1) * (NC + 4) * 4;    // 2 x T/8 run flag bytes
  static constexpr size_t za = gbuf + 2 * (size_t)(T / 8);                  // T/32 u16: zero prefix per 4 half-runs
  static constexpr size_t tot = za + (size_t)(T / 32) * 2;                  // [2 regions][warps] uint2 warp totals
  static constexpr size_t lut = tot + 2 * (size_t)(T / 1024) * 8;          // K8Q_LUT interleaved copies of the 256 sort selectors
  static constexpr size_t mbar = lut + 1024 * K8Q_LUT;                     // tile, then run table
  static constexpr size_t total = mbar + 16;
  // the run table (needed by the emission only) lands in the final round's
  // unused destination buffer, above everything that round keeps there
  static constexpr int JL = (W & 1) ? W - 3 : W - 2;
  static constexpr size_t tab = (size_t)(((JL >> 1) + 1) & 1) * T + 12288;
};

// The 8 flags of bit `sh` of a run's bytes (x0: bytes 0-3, x1: bytes 4-7).
// `bits` gets the flag bits in place (for POPC); the return value holds the
// 8-bit mask in its low byte with garbage above (`flags_lo` cleans it): one
// multiply gathers the flags (bits 8i and 8i + 4 -> bit i), the high word of a
// second one shifts them down, so only the two masks use the integer ALU.
__device__ __forceinline__ uint32_t run_flags8(uint32_t x0, uint32_t x1, int sh, uint32_t& bits) {
  const uint32_t M = 0x01010101u << sh;
  // flag of byte i at bit 8i + p, of byte 4 + i at bit 8i + 4 + p (p = sh, or
  // sh - 4 with bytes 0-3 moved down by a multiply so nothing leaves the word)
  const int p = sh >= 4 ? sh - 4 : sh;
  bits = sh >= 4 ? __umulhi(x0 & M, 1u << 28) + (x1 & M) : (x1 & M) * 16u + (x0 & M);
  if (p == 0) return (bits * 0x01020408u) >> 24;
  return __umulhi(bits, 0x01020408u << (8 - p));
}
__device__ __forceinline__ uint32_t flags_lo(uint32_t f) { return f & 0xFFu; }

// ((1 << width) - 1) << pos (width 0 or pos 32: 0)
__device__ __forceinline__ uint32_t bmsk(uint32_t pos, uint32_t width) {
  uint32_t d;
  asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(d) : "r"(pos), "r"(width));
  return d;
}
// shared OR of v, predicated on v != 0 (no branch)
__device__ __forceinline__ void red_or_nz(uint32_t saddr, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q red.shared.or.b32 [%0], %1;\n\t}" ::"r"(saddr), "r"(v)
               : "memory");
}
// OR a bit string v (its length implied: bits above it are zero) into the
// shared bit array at shared address L, bit pos
__device__ __forceinline__ void or_bits32(uint32_t L, uint32_t pos, uint32_t v) {
  const uint64_t t = (uint64_t)v << (pos & 31);
  const uint32_t a = L + (pos >> 5) * 4u;
  red_or_nz(a, (uint32_t)t);
  red_or_nz(a + 4u, (uint32_t)(t >> 32));
}

template <int W>
__global__ void __launch_bounds__(K8_TILE / 32, K8_CTAS) level_pass8q_kernel(const Pass8Args a,
                                                                            const TabW<W>* __restrict__ tabs) {
  constexpr int T = K8_TILE;
  constexpr int RUN = 16;              // bytes per thread run: two 8-symbol halves, each sorted by PRMT
  constexpr int QR = 2;                // runs per thread, one per region
  constexpr int NT = T / (RUN * QR);
  constexpr int RG = T / QR;           // region of run k: [k RG, (k + 1) RG)
  constexpr int HR = RG / 8;           // 8-symbol half-runs per region
  constexpr int NC = T / 32;
  constexpr int NW = NT / 32;
  using L = Q8Smem<W>;
  // the class-sorted runs stay in registers across the round's barrier where they
  // fit the 32 registers without spills (measured: W = 8 2.82 -> 2.80 ms; W = 4, 5, 7 spill)
  constexpr bool KEEP_U = W == 8 || W == 6;
  static_assert(NW <= 32 && T <= 32768, "16-bit store bases (offsets inside the destination buffer)");
  extern __shared__ __align__(128) unsigned char smem[];
  TabW<W>& tt = *reinterpret_cast<TabW<W>*>(smem + L::tab);
  static_assert(T == 16384 && 12288 + sizeof(TabW<W>) <= (size_t)T, "run table slot");
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + L::bits) - (NC + 4);  // level j at j (NC + 4)
  uint8_t* bits8 = reinterpret_cast<uint8_t*>(bits);
  uint16_t* za16 = reinterpret_cast<uint16_t*>(smem + L::za);  // per 4th half-run: b_j zeros before it
  uint2* s_tot = reinterpret_cast<uint2*>(smem + L::tot);
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem + L::lut);
  const uint32_t* my_lut = s_lut + (threadIdx.x % K8Q_LUT);  // this lane's copy

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint8_t* text = a.src;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t mbar = sb + (uint32_t)L::mbar, mbar_tab = mbar + 8u;
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * T;
  const int cnt = (int)min((int64_t)T, a.n - base);
  const bool bulk = (((uintptr_t)text) & 15) == 0 && cnt == T;
  if (tid == 0) {
    mbar_init(mbar, 1);
    mbar_init(mbar_tab, 1);
    fence_mbar_init();
    if (bulk) bulk_load(sb, text + base, (uint32_t)T, mbar);
    else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
    if (L::JL == 0) bulk_load(sb + (uint32_t)L::tab, tabs + tile, (uint32_t)sizeof(TabW<W>), mbar_tab);
  }
  for (int i = tid; i < 256 * K8Q_LUT; i += NT) s_lut[i] = g_sort_lut.sel[i / K8Q_LUT];
  // the levels filled by OR-ing bit strings (odd levels: the skipped level of
  // every round) start at zero
#pragma unroll
  for (int j = 1; j < W; ++j)
    if ((j & 1) || ((W & 1) && j == W - 1 && W >= 3)) {  // (odd W: the last round ORs level W-1 too)
      uint4* b4 = reinterpret_cast<uint4*>(bits + j * (NC + 4));  // (NC + 4) words: 16-byte aligned rows
      for (int i = tid; i < (NC + 4) / 4; i += NT) b4[i] = make_uint4(0u, 0u, 0u, 0u);
    }
  if (!bulk)
    for (int p = tid; p < T; p += NT) smem[p] = p < cnt ? text[base + p] : (uint8_t)0xFF;
  bar_sync(1, NT);
  mbar_wait(mbar, 0);

  // level 0's flags (hist8_kernel emits level 0) are only needed for round 0's
  // concatenation: they go to a scratch that is free until later -- level W-1's
  // array (re-zeroed after use: W-1 is an OR-ed level for every W >= 4), for
  // W = 2 the second flag buffer, for W = 3 the stage buffer round 0 leaves unused
  uint8_t* const m0b = W == 2 ? smem + L::gbuf + T / 8 : W == 3 ? smem + T : bits8 + (W - 1) * 4 * (NC + 4);

#pragma unroll
  for (int j = 0; j < W; j += 2) {
    const int sh = W - 1 - j;
    if (j == L::JL && j > 0 && tid == 0)  // the run table into the buffer the final round leaves unused
      bulk_load(sb + (uint32_t)L::tab, tabs + tile, (uint32_t)sizeof(TabW<W>), mbar_tab);
    uint8_t* const cur = smem + (size_t)((j >> 1) & 1) * T;
    uint8_t* const mb = j == 0 ? m0b : bits8 + j * 4 * (NC + 4);
    // odd width: the last round starts at A_W-3 and emits three levels without a
    // scatter -- L_W-2 and L_W-1 are concatenated from the runs' 2- and 4-class pieces
    const bool triple = (W & 1) && j + 3 == W;
    const bool quad = j + 2 < W && !triple;
    uint8_t* const gb = smem + L::gbuf + (size_t)((j >> 1) & 1) * (T / 8);
    // (triple round: the unused destination buffer holds its run flags h and
    // the class prefixes of every 4th half-run; for W = 3 after round 0's m0 bytes)
    uint8_t* const nxtb = smem + (size_t)(((j >> 1) + 1) & 1) * T;
    uint8_t* const hb = nxtb + T / 8;
    uint2* const cpre = reinterpret_cast<uint2*>(nxtb + 2 * (T / 8));
    uint32_t cA[QR], cB[QR], ff[QR], ee[QR];  // per run: class counts of its halves (bytes), 10-bit sums, scan
    uint4 ukeep[QR];  // (KEEP_U) the class-sorted runs across the barrier
    uint32_t ones[QR];
#pragma unroll
    for (int k = 0; k < QR; ++k) {
      const uint4 qv = reinterpret_cast<const uint4*>(cur + k * RG)[tid];
      uint32_t xw[4] = {qv.x, qv.y, qv.z, qv.w};
      uint32_t cb[2] = {0u, 0u}, f10 = 0u, o = 0u;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r8 = k * HR + 2 * tid + h;  // the half's 8-symbol run
        uint32_t mbits, gbits;
        const uint32_t m = run_flags8(xw[2 * h], xw[2 * h + 1], sh, mbits);
        mb[r8] = (uint8_t)m;
        const uint32_t sel = my_lut[flags_lo(m) * K8Q_LUT];
        const uint32_t s0 = prmt(xw[2 * h], xw[2 * h + 1], sel), s1 = prmt(xw[2 * h], xw[2 * h + 1], sel >> 16);
        const uint32_t g = run_flags8(s0, s1, sh - 1, gbits);
        gb[r8] = (uint8_t)g;
        if (quad || triple) {
          const uint32_t sel2 = my_lut[flags_lo(g) * K8Q_LUT];
          xw[2 * h] = prmt(s0, s1, sel2);
          xw[2 * h + 1] = prmt(s0, s1, sel2 >> 16);
          if (triple) {
            uint32_t hbits;
            hb[r8] = (uint8_t)run_flags8(xw[2 * h], xw[2 * h + 1], sh - 2, hbits);  // b_j+2 in class order
          }
          // class counts n0..n3 (c = 2 b_j+1 + b_j): z = n0 + n1 (b_j zeros),
          // n2 = the zeros' b_j+1 ones, n3 = the ones' b_j+1 ones; as bytes and
          // as three 10-bit fields (n0 | n1 << 10 | n2 << 20), both mod 2^32
          const uint32_t z = 8u - __popc(mbits);
          const uint32_t n2 = __popc(g & ((1u << z) - 1u));
          const uint32_t n3 = __popc(gbits) - n2;
          cb[h] = z * 0xFFFFFF01u + 0x800u + n2 * 0xFFFFu + n3 * 0xFFFF00u;
          f10 += z * (1u - 1024u) + 8u * 1024u + n2 * ((1u << 20) - 1u) - n3 * 1024u;
        } else {
          o += __popc(mbits);
        }
      }
      if (quad) {
        if (KEEP_U) ukeep[k] = make_uint4(xw[0], xw[1], xw[2], xw[3]);
        else  // the class-sorted halves go back to the run's own slot (read again after the barrier)
          reinterpret_cast<uint4*>(cur + k * RG)[tid] = make_uint4(xw[0], xw[1], xw[2], xw[3]);
      }
      if (quad || triple) {
        cA[k] = cb[0];
        cB[k] = cb[1];
        ff[k] = f10;
        ee[k] = warp_incl_scan(f10);  // 10-bit fields: at most 32 x 16 per class
      } else {
        ones[k] = o;
      }
    }
    uint32_t Zt;  // the tile's b_j zeros: where L_j+1's ones stream starts
    uint32_t C1 = 0, C2 = 0, C3 = 0;  // class starts of A_j+2 (triple round: L_j+2's streams)
    if (quad || triple) {
      if (lane == 31) {  // warp totals per region: (n0 | n1 << 16, n2)
#pragma unroll
        for (int k = 0; k < QR; ++k)
          s_tot[k * NW + wid] = make_uint2((ee[k] & 0x3FFu) | (((ee[k] >> 10) & 0x3FFu) << 16), ee[k] >> 20);
      }
      bar_sync(1, NT);
      // (lane l < NW holds warp l's totals; per-lane sums over the regions
      // turn every prefix into one REDUX)
      uint32_t sx = 0, sy = 0;
#pragma unroll
      for (int k = 0; k < QR; ++k) {
        const uint2 v = lane < NW ? s_tot[k * NW + lane] : make_uint2(0u, 0u);
        sx += v.x;
        sy += v.y;
      }
      const uint32_t TA = __reduce_add_sync(FULL, sx), TB = __reduce_add_sync(FULL, sy);
      C1 = TA & 0xFFFFu;
      C2 = C1 + (TA >> 16);
      C3 = C2 + TB;
      Zt = (TA & 0xFFFFu) + TB;  // classes 0 and 2: b_j = 0
      const uint32_t dst = sb + (uint32_t)(((j >> 1) + 1) & 1) * T;  // destination buffer (store immediates)
      uint32_t ax = 0, ay = 0;  // this lane's warp over the regions before
#pragma unroll
      for (int k = 0; k < QR; ++k) {
        const uint2 v = lane < NW ? s_tot[k * NW + lane] : make_uint2(0u, 0u);
        const uint32_t A = __reduce_add_sync(FULL, ax + (lane < wid ? v.x : 0u));
        const uint32_t B = __reduce_add_sync(FULL, ay + (lane < wid ? v.y : 0u));
        ax += v.x;
        ay += v.y;
        // the run's class prefixes: regions / warps before + this lane's exclusive scan
        const uint32_t e = ee[k] - ff[k];
        const uint32_t P0 = (A & 0xFFFFu) + (e & 0x3FFu);
        const uint32_t P1 = (A >> 16) + ((e >> 10) & 0x3FFu);
        const uint32_t P2 = B + (e >> 20);
        const uint32_t P3 = (uint32_t)(k * RG + RUN * tid) - P0 - P1 - P2;
        if ((tid & 1) == 0) {  // half-run 2t of the region is a 4th half-run: the concatenation's offsets
          const int q4 = (k * HR + 2 * tid) >> 2;
          if (triple) cpre[q4] = make_uint2(P0 | (P2 << 16), P1 | (P3 << 16));
          else za16[q4] = (uint16_t)(P0 + P2);  // b_j zeros before it
        }
        if (triple) continue;  // no scatter
        // the run's class bases as 16-bit pairs (classes 0|2, 1|3); a half's
        // class c byte kk goes to base_c + (half 1: half 0's class-c count) - S_c + kk
        const uint32_t BA = P0 | ((C2 + P2) << 16), BB = (C1 + P1) | ((C3 + P3) << 16);
        const uint4 uk = KEEP_U ? ukeep[k] : reinterpret_cast<const uint4*>(cur + k * RG)[tid];
        const uint32_t uw[4] = {uk.x, uk.y, uk.z, uk.w};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t sv = (h ? cB[k] : cA[k]) * 0x01010100u;  // class starts inside the half
          const uint32_t DA = BA - prmt(sv, 0u, 0x4240u) + (h ? prmt(cA[k], 0u, 0x4240u) : 0u);
          const uint32_t DB = BB - prmt(sv, 0u, 0x4341u) + (h ? prmt(cA[k], 0u, 0x4341u) : 0u);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint32_t w = uw[2 * h + hh];
            const uint32_t x = w >> (sh - 1);
            // PRMT selectors of bytes 0, 2 and 1, 3: nibbles 2c', 2c'+1 pick the
            // byte's 16-bit base (c' = 2 b_j + b_j+1), 0x99 zero-fills the top half
            // (0x22 c' has no bit of 0x10 / 0x99 set: OR adds them, no constant register)
            const uint32_t s02 = ((x & 0x00030003u) * 0x22u) | 0x99109910u;
            const uint32_t s13 = __umulhi(x & 0x03000300u, 0x22000000u) | 0x99109910u;
            const uint32_t a0 = prmt(DA, DB, s02), a1 = prmt(DA, DB, s13);
            const uint32_t a2 = prmt(DA, DB, __umulhi(s02, 0x10000u)), a3 = prmt(DA, DB, __umulhi(s13, 0x10000u));
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(a0 + dst + (uint32_t)(4 * hh)), "r"(w) : "memory");
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(a1 + dst + (uint32_t)(4 * hh + 1)), "r"(__umulhi(w, 1u << 24)) : "memory");
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(a2 + dst + (uint32_t)(4 * hh + 2)), "r"(__umulhi(w, 1u << 16)) : "memory");
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(a3 + dst + (uint32_t)(4 * hh + 3)), "r"(__umulhi(w, 1u << 8)) : "memory");
          }
        }
      }
    } else {
      // last round of an even width: a 2-way count scan for L_W-1's pieces
      // (two runs per thread, one per region, packed 16|16)
      static_assert(QR == 2, "one packed scan for the two regions");
      const uint32_t pk = ones[0] | (ones[1] << 16);
      const uint32_t incl = warp_incl_scan(pk);
      if (lane == 31) s_tot[wid].x = incl;
      bar_sync(1, NT);
      const uint32_t wv = lane < NW ? s_tot[lane].x : 0u;
      const uint32_t ex = __reduce_add_sync(FULL, lane < wid ? wv : 0u) + incl - pk;
      const uint32_t tot = __reduce_add_sync(FULL, wv);
      if ((tid & 1) == 0) {  // zeros before the run = its position - the ones before it
        za16[(2 * tid) >> 2] = (uint16_t)((uint32_t)(RUN * tid) - (ex & 0xFFFFu));
        za16[(HR + 2 * tid) >> 2] = (uint16_t)((uint32_t)(RG + RUN * tid) - ((tot & 0xFFFFu) + (ex >> 16)));
      }
      Zt = (uint32_t)T - (tot & 0xFFFFu) - (tot >> 16);
    }
    // (the run table's slot was last read here: order that before the bulk copy of the next round)
    if (j + 2 == L::JL) fence_proxy_async_smem();
    bar_sync(1, NT);
    // L_j+1 from the half-runs' flag pieces: thread t owns half-runs 4t .. 4t+3
    {
      const uint32_t gw = reinterpret_cast<const uint32_t*>(gb)[tid];
      uint32_t* mwp = reinterpret_cast<uint32_t*>(mb) + tid;
      const uint32_t mw = *mwp;
      if (j == 0 && W >= 4) *mwp = 0u;  // level W-1 (OR-ed later) lent its array
      const uint2 cp = triple ? cpre[tid] : make_uint2(0u, 0u);
      const uint32_t zpos = triple ? (cp.x & 0xFFFFu) + (cp.x >> 16) : za16[tid];
      uint32_t accz = 0, acco = 0, fz = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // run 4t + i: its zeros' flags (bits [8i, 8i + z) of gw) go to fz, its
        // ones' flags (bits [8i + z, 8i + 8)) to the 8i - fz ones before it
        const uint32_t z = 8u - __popc(mw & (0xFFu << (8 * i)));
        const uint32_t zm = bmsk(8u * i, z);
        accz |= (gw & zm) >> (8u * i - fz);
        acco |= (gw & (0xFFu << (8 * i)) & ~zm) >> (z + fz);
        fz += z;
      }
      const uint32_t Lw = sb + (uint32_t)((const unsigned char*)(bits + (j + 1) * (NC + 4)) - smem);
      or_bits32(Lw, zpos, accz);
      or_bits32(Lw, Zt + 32u * tid - zpos, acco);
      if (triple) {
        // L_j+2 = b_j+2 over A_j+2: each half-run's class-sorted b_j+2 flags h,
        // split into its four class pieces, appended to the four class streams
        const uint32_t hw = reinterpret_cast<const uint32_t*>(hb)[tid];
        uint32_t acc[4] = {0u, 0u, 0u, 0u}, f[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t g = (gw >> (8 * i)) & 0xFFu;
          const uint32_t z = 8u - __popc(mw & (0xFFu << (8 * i)));
          const uint32_t n2 = __popc(g & ((1u << z) - 1u)), n3 = __popc(g) - n2;
          const uint32_t n[4] = {z - n2, 8u - z - n3, n2, n3};
          const uint32_t st[4] = {0u, z - n2, 8u - n2 - n3, 8u - n3};  // class starts in the sorted run
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            acc[c] |= (hw & bmsk(8u * i + st[c], n[c])) >> (8u * i + st[c] - f[c]);
            f[c] += n[c];
          }
        }
        const uint32_t L2 = sb + (uint32_t)((const unsigned char*)(bits + (j + 2) * (NC + 4)) - smem);
        or_bits32(L2, cp.x & 0xFFFFu, acc[0]);
        or_bits32(L2, C1 + (cp.y & 0xFFFFu), acc[1]);
        or_bits32(L2, C2 + (cp.x >> 16), acc[2]);
        or_bits32(L2, C3 + (cp.y >> 16), acc[3]);
        break;
      }
    }
  }
  bar_sync(1, NT);  // every level's bits are in place
  mbar_wait(mbar_tab, 0);
  emit_levels8<W, NC>(tt, bits, a.words, a.nwords, tid, NT, smem);  // (coarse map: stage buffer 0's first bytes)
}

template <int W>
cudaError_t launch_pass8q(const Pass8Args& a, void* tabs, cudaStream_t s) {
  constexpr size_t smem = Q8Smem<W>::total;
  static_assert((smem + 1024) * K8_CTAS <= 228 * 1024, "K8_CTAS CTAs per SM must fit the shared memory");
  auto kern = level_pass8q_kernel<W>;
  cudaError_t e0 = ensure_smem_attr((const void*)kern, (int)smem, true);
  if (e0 != cudaSuccess) return e0;
  kern<<<(unsigned)a.ntiles, K8_TILE / 32, smem, s>>>(a, (const TabW<W>*)tabs);
  return cudaGetLastError();
}
