// K16Q: the fused 2-byte pass (k16.cuh) with TWO levels per shared-memory round,
// the byte pass's k8q.cuh scheme on 2-byte elements, for even widths W.
//
// A round from A_j: every 8-element half of a thread's 16-element run is split
// into its high-byte and low-byte planes; both planes are sorted by the b_j
// flags of the high bytes and then by their b_j+1 flags with the same PRMT
// selectors, so the half is in A_j+2 class order (c = 2 b_j+1 + b_j); the
// planes are re-paired and ONE 4-way scatter of 16-bit elements writes A_j+2.
// L_j is the b_j flags, L_j+1 comes from the halves' sorted b_j+1 flags by the
// concatenation of k8q.cuh.  Every round scatters (the last one writes A_W,
// whose level-W groups' low bytes leave as the byte tail's text), so W / 2
// 4-way scatters replace W 2-way ones.  Odd widths keep level_pass16_kernel.
//
// Store addressing as in k8q.cuh: the four per-half class bases, doubled (byte
// offsets of 2-byte elements inside the destination buffer, < 2 T = 32768),
// packed in two registers; the element's class (two bits of its high byte)
// builds a PRMT selector that picks its base.
//
// Included from wvlt_b200.cu after k16.cuh (same translation unit).

namespace {

template <int W>
struct Q16Smem {
  static constexpr int T = K16_TILE;
  static constexpr int NC = T / 32;
  static constexpr int NB = 1 << W;
  static constexpr size_t bits = 4 * (size_t)T;                             // after the two 2-byte order buffers
  static constexpr size_t gbuf = bits + (size_t)(W - 1) * (NC + 4) * 4;    // 2 x T/8 half-run flag bytes
  static constexpr size_t za = gbuf + 2 * (size_t)(T / 8);                  // T/32 u16: zero prefix per 4 half-runs
  static constexpr size_t tot = za + (size_t)(T / 32) * 2;                  // [2 regions][warps] uint2
  static constexpr size_t lut = tot + 2 * (size_t)(T / 1024) * 8;
  static constexpr size_t gW = lut + 1024;                                  // level-W groups: global starts (u32)
  static constexpr size_t cW = gW + 4 * (size_t)NB;                        // sizes (u16)
  static constexpr size_t lsW = cW + 2 * (size_t)NB;                       // tile-local starts (u16)
  static constexpr size_t tmp = lsW + 2 * (size_t)NB;                      // warp sums (u32)
  static constexpr size_t tab = (tmp + 4 * (size_t)(T / 1024) + 15) & ~(size_t)15;  // TabW<W>
  static constexpr size_t mbar = tab + sizeof(TabW<W>);
  static constexpr size_t total = mbar + 16;
};

template <int W>
__global__ void __launch_bounds__(K16_TILE / 32, K16_CTAS) level_pass16q_kernel(const Pass16Args a,
                                                                              const TabW<W>* __restrict__ tabs) {
  static_assert((W & 1) == 0 && W >= 2, "even widths");
  constexpr int T = K16_TILE;
  constexpr int RUN = 16;              // elements per thread run: two 8-element halves
  constexpr int QR = 2;                // runs per thread, one per region
  constexpr int NT = T / (RUN * QR);
  constexpr int RG = T / QR;           // elements per region
  constexpr int HR = RG / 8;           // 8-element half-runs per region
  constexpr int NC = T / 32;
  constexpr int NW = NT / 32;
  constexpr int NB = 1 << W;
  using L = Q16Smem<W>;
  static_assert(NW <= 32 && 2 * T <= 32768, "16-bit store bases (byte offsets inside the destination buffer)");
  extern __shared__ __align__(128) unsigned char smem[];
  TabW<W>& tt = *reinterpret_cast<TabW<W>*>(smem + L::tab);
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + L::bits) - (NC + 4);  // level j at j (NC + 4)
  uint8_t* bits8 = reinterpret_cast<uint8_t*>(bits);
  uint16_t* za16 = reinterpret_cast<uint16_t*>(smem + L::za);
  uint2* s_tot = reinterpret_cast<uint2*>(smem + L::tot);
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem + L::lut);
  uint32_t* s_gW = reinterpret_cast<uint32_t*>(smem + L::gW);
  uint16_t* s_cW = reinterpret_cast<uint16_t*>(smem + L::cW);
  uint16_t* s_lsW = reinterpret_cast<uint16_t*>(smem + L::lsW);
  uint32_t* s_tmp = reinterpret_cast<uint32_t*>(smem + L::tmp);

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * T;
  const int cnt = (int)min((int64_t)T, a.n - base);
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t mbar = sb + (uint32_t)L::mbar;
  const bool bulk = (((uintptr_t)a.src) & 15) == 0 && cnt == T;
  if (tid == 0) {
    mbar_init(mbar, 1);
    fence_mbar_init();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar),
                 "r"((uint32_t)(sizeof(TabW<W>) + (bulk ? 2 * T : 0)))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sb + (uint32_t)L::tab),
                 "l"(tabs + tile), "r"((uint32_t)sizeof(TabW<W>)), "r"(mbar)
                 : "memory");
    if (bulk)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sb),
                   "l"(a.src + base), "r"((uint32_t)(2 * T)), "r"(mbar)
                   : "memory");
  }
  for (int i = tid; i < 256; i += NT) s_lut[i] = g_sort_lut.sel[i];
#pragma unroll
  for (int j = 1; j < W; j += 2) {  // the OR-ed levels (the skipped level of every round) start at zero
    uint4* b4 = reinterpret_cast<uint4*>(bits + j * (NC + 4));
    for (int i = tid; i < (NC + 4) / 4; i += NT) b4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  // level-W groups of this tile: sizes, global starts (LSD digit d = rev(e))
  if (tid < NB) {
    const int d = (int)rev_bits((unsigned)tid, W);
    s_cW[d] = (uint16_t)__ldg(a.tcnt8 + tile * NB + tid);
    s_gW[d] = (uint32_t)(__ldg(a.baseW + d) + (int64_t)__ldg(a.tpre8 + tile * NB + tid));
  }
  if (!bulk) {
    uint16_t* st = reinterpret_cast<uint16_t*>(smem);
    for (int p = tid; p < T; p += NT) st[p] = p < cnt ? a.src[base + p] : (uint16_t)0xFFFF;
  }
  bar_sync(1, NT);
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

  // level 0's flags (hist16_kernel emits level 0) for round 0's concatenation:
  // level W-1's array (an OR-ed level, re-zeroed after use), for W = 2 the
  // second flag buffer
  uint8_t* const m0b = W == 2 ? smem + L::gbuf + T / 8 : bits8 + (W - 1) * 4 * (NC + 4);

#pragma unroll
  for (int j = 0; j < W; j += 2) {
    const int sh = W - 1 - j;
    const unsigned char* cur = smem + (size_t)((j >> 1) & 1) * 2 * T;
    uint8_t* const mb = j == 0 ? m0b : bits8 + j * 4 * (NC + 4);
    uint8_t* const gb = smem + L::gbuf + (size_t)((j >> 1) & 1) * (T / 8);
    uint32_t cA[QR], cB[QR], ff[QR], ee[QR];
    uint32_t hi[QR][4], lo[QR][4];  // the class-sorted runs: high / low byte planes (halves 0, 1)
#pragma unroll
    for (int k = 0; k < QR; ++k) {
      uint32_t cb[2] = {0u, 0u}, f10 = 0u;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 qv = reinterpret_cast<const uint4*>(cur + 2 * (k * RG))[2 * tid + h];
        const uint32_t x0 = prmt(qv.x, qv.y, 0x7531), x1 = prmt(qv.z, qv.w, 0x7531);
        const uint32_t y0 = prmt(qv.x, qv.y, 0x6420), y1 = prmt(qv.z, qv.w, 0x6420);
        const int r8 = k * HR + 2 * tid + h;
        uint32_t mbits, gbits;
        const uint32_t m = run_flags8(x0, x1, sh, mbits);
        mb[r8] = (uint8_t)m;
        const uint32_t sel = s_lut[flags_lo(m)];
        const uint32_t s0 = prmt(x0, x1, sel), s1 = prmt(x0, x1, sel >> 16);
        const uint32_t t0 = prmt(y0, y1, sel), t1 = prmt(y0, y1, sel >> 16);
        const uint32_t g = run_flags8(s0, s1, sh - 1, gbits);
        gb[r8] = (uint8_t)g;
        const uint32_t sel2 = s_lut[flags_lo(g)];
        hi[k][2 * h] = prmt(s0, s1, sel2);
        hi[k][2 * h + 1] = prmt(s0, s1, sel2 >> 16);
        lo[k][2 * h] = prmt(t0, t1, sel2);
        lo[k][2 * h + 1] = prmt(t0, t1, sel2 >> 16);
        const uint32_t z = 8u - __popc(mbits);
        const uint32_t n2 = __popc(g & ((1u << z) - 1u));
        const uint32_t n3 = __popc(gbits) - n2;
        cb[h] = z * 0xFFFFFF01u + 0x800u + n2 * 0xFFFFu + n3 * 0xFFFF00u;
        f10 += z * (1u - 1024u) + 8u * 1024u + n2 * ((1u << 20) - 1u) - n3 * 1024u;
      }
      cA[k] = cb[0];
      cB[k] = cb[1];
      ff[k] = f10;
      ee[k] = warp_incl_scan(f10);
    }
    if (lane == 31) {
#pragma unroll
      for (int k = 0; k < QR; ++k)
        s_tot[k * NW + wid] = make_uint2((ee[k] & 0x3FFu) | (((ee[k] >> 10) & 0x3FFu) << 16), ee[k] >> 20);
    }
    bar_sync(1, NT);
    uint32_t sx = 0, sy = 0;
#pragma unroll
    for (int k = 0; k < QR; ++k) {
      const uint2 v = lane < NW ? s_tot[k * NW + lane] : make_uint2(0u, 0u);
      sx += v.x;
      sy += v.y;
    }
    const uint32_t TA = __reduce_add_sync(FULL, sx), TB = __reduce_add_sync(FULL, sy);
    const uint32_t C1 = TA & 0xFFFFu, C2 = C1 + (TA >> 16), C3 = C2 + TB;
    const uint32_t Zt = (TA & 0xFFFFu) + TB;  // b_j zeros (classes 0 and 2)
    const uint32_t dst = sb + (uint32_t)(((j >> 1) + 1) & 1) * 2 * T;
    uint32_t ax = 0, ay = 0;
#pragma unroll
    for (int k = 0; k < QR; ++k) {
      const uint2 v = lane < NW ? s_tot[k * NW + lane] : make_uint2(0u, 0u);
      const uint32_t A = __reduce_add_sync(FULL, ax + (lane < wid ? v.x : 0u));
      const uint32_t B = __reduce_add_sync(FULL, ay + (lane < wid ? v.y : 0u));
      ax += v.x;
      ay += v.y;
      const uint32_t e = ee[k] - ff[k];
      const uint32_t P0 = (A & 0xFFFFu) + (e & 0x3FFu);
      const uint32_t P1 = (A >> 16) + ((e >> 10) & 0x3FFu);
      const uint32_t P2 = B + (e >> 20);
      const uint32_t P3 = (uint32_t)(k * RG + RUN * tid) - P0 - P1 - P2;
      if ((tid & 1) == 0) za16[(k * HR + 2 * tid) >> 2] = (uint16_t)(P0 + P2);
      const uint32_t BA = P0 | ((C2 + P2) << 16), BB = (C1 + P1) | ((C3 + P3) << 16);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t sv = (h ? cB[k] : cA[k]) * 0x01010100u;
        // element bases (elements), doubled into byte offsets (each 16-bit lane < 2^15)
        const uint32_t DA = 2u * (BA - prmt(sv, 0u, 0x4240u) + (h ? prmt(cA[k], 0u, 0x4240u) : 0u));
        const uint32_t DB = 2u * (BB - prmt(sv, 0u, 0x4341u) + (h ? prmt(cA[k], 0u, 0x4341u) : 0u));
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t hw = hi[k][2 * h + hh], lw = lo[k][2 * h + hh];
          const uint32_t x = hw >> (sh - 1);
          const uint32_t s02 = ((x & 0x00030003u) * 0x22u) | 0x99109910u;
          const uint32_t s13 = __umulhi(x & 0x03000300u, 0x22000000u) | 0x99109910u;
          const uint32_t a0 = prmt(DA, DB, s02), a1 = prmt(DA, DB, s13);
          const uint32_t a2 = prmt(DA, DB, __umulhi(s02, 0x10000u)), a3 = prmt(DA, DB, __umulhi(s13, 0x10000u));
          const uint32_t e01 = prmt(lw, hw, 0x5140), e23 = prmt(lw, hw, 0x7362);  // elements 4hh .. 4hh + 3
          const uint32_t kk = 8u * hh;  // byte offset of element 4 hh inside the half
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a0 + dst + kk), "h"((unsigned short)e01) : "memory");
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a1 + dst + kk + 2u), "h"((unsigned short)(e01 >> 16)) : "memory");
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a2 + dst + kk + 4u), "h"((unsigned short)e23) : "memory");
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a3 + dst + kk + 6u), "h"((unsigned short)(e23 >> 16)) : "memory");
        }
      }
    }
    bar_sync(1, NT);
    // L_j+1 from the half-runs' flag pieces (k8q.cuh): thread t owns half-runs 4t .. 4t+3
    {
      const uint32_t gw = reinterpret_cast<const uint32_t*>(gb)[tid];
      uint32_t* mwp = reinterpret_cast<uint32_t*>(mb) + tid;
      const uint32_t mw = *mwp;
      if (j == 0 && W >= 4) *mwp = 0u;  // level W-1 (OR-ed later) lent its array
      const uint32_t zpos = za16[tid];
      uint32_t accz = 0, acco = 0, fz = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t z = 8u - __popc(mw & (0xFFu << (8 * i)));
        const uint32_t zm = bmsk(8u * i, z);
        accz |= (gw & zm) >> (8u * i - fz);
        acco |= (gw & (0xFFu << (8 * i)) & ~zm) >> (z + fz);
        fz += z;
      }
      const uint32_t Lw = sb + (uint32_t)((const unsigned char*)(bits + (j + 1) * (NC + 4)) - smem);
      or_bits32(Lw, zpos, accz);
      or_bits32(Lw, Zt + 32u * tid - zpos, acco);
    }
  }
  bar_sync(1, NT);  // every level's bits and the level-W order are in place
  // levels 1..W-1 (the order buffer not holding A_W is the emission's scratch)
  emit_levels8<W, NC>(tt, bits, a.words, a.nwords, tid, NT, smem + (size_t)(((W >> 1) + 1) & 1) * 2 * T);
  // the low bytes of each level-W group: one contiguous run of the byte text
  const uint8_t* lob = smem + (size_t)((W >> 1) & 1) * 2 * T;
  for (int r = wid; r < NB; r += NW) {
    const int c = s_cW[r];
    if (!c) continue;
    uint8_t* dstp = a.out + s_gW[r];
    const uint8_t* sp = lob + 2 * s_lsW[r];
    for (int i = lane; i < c; i += 32) dstp[i] = sp[2 * i];
  }
}

template <int W>
cudaError_t launch_pass16q(const Pass16Args& a, const void* tabs, cudaStream_t s) {
  constexpr size_t smem = Q16Smem<W>::total;
  static_assert((smem + 1024) * K16_CTAS <= 228 * 1024, "K16_CTAS CTAs per SM must fit the shared memory");
  auto kern = level_pass16q_kernel<W>;
  cudaError_t e0 = ensure_smem_attr((const void*)kern, (int)smem, true);
  if (e0 != cudaSuccess) return e0;
  kern<<<(unsigned)a.ntiles, K16_TILE / 32, smem, s>>>(a, (const TabW<W>*)tabs);
  return cudaGetLastError();
}

}  // namespace
