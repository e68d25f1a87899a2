// Consumers of a built structure: rank/select directories of the
// level bit vectors and batched access / rank / select queries on the device.
// Included at the end of wvlt_b200.cu (same translation unit: shares the scan
// kernels and warp helpers).
//
// Directory layout is the reference's RankSelectBitVector (bitvec.py:118-163):
// per 2048-bit superblock the zeros before it, per 256-bit block the zeros
// before it relative to its superblock, and the positions of every 8192nd one
// and zero (select samples).  Query algorithms follow bitvec.py:178-263 and
// structures.py:107-256.

namespace {

constexpr int RS_SB_BITS = 2048;
constexpr int RS_SB_WORDS = RS_SB_BITS / 64;  // 32: one word per lane
constexpr int RS_BLK_BITS = 256;
constexpr int RS_BLK_PER_SB = RS_SB_BITS / RS_BLK_BITS;
constexpr int64_t RS_SAMPLE = 8192;
constexpr int RS_WARPS = 8;  // superblocks per CTA in the directory kernels

struct RsShape {
  int64_t nwords, nsuper, nblocks, nsamp;
};

__host__ __device__ inline RsShape rs_shape(int64_t length) {
  RsShape s;
  s.nwords = (length + 63) >> 6;
  s.nsuper = (length + RS_SB_BITS - 1) / RS_SB_BITS;
  s.nblocks = (length + RS_BLK_BITS - 1) / RS_BLK_BITS;
  s.nsamp = (length + RS_SAMPLE - 1) / RS_SAMPLE;  // capacity per bit value
  return s;
}

// 0-based position of the k-th (1-based) set bit of a 64-bit word (k <= popc).
__device__ __forceinline__ int select_in_word64(uint64_t word, int k) {
  int pos = 0;
#pragma unroll
  for (int half = 32; half >= 1; half >>= 1) {
    const uint64_t low = word & ((1ull << half) - 1ull);
    const int c = __popcll(low);
    if (k > c) {
      k -= c;
      word >>= half;
      pos += half;
    } else {
      word = low;
    }
  }
  return pos;
}

// Pass 1: one warp per RS_SB_PER_WARP superblocks (lane = word, all loads in
// flight first): word popcounts, block zeros relative to the superblock,
// superblock one counts.
constexpr int RS_SB_PER_WARP = 8;  // (measured: 8 < 16 < 4: directory of c2 0.476 < 0.489 < 0.504 ms)
__global__ void __launch_bounds__(RS_WARPS * 32) rs_blocks_kernel(const uint64_t* __restrict__ words, int64_t length,
                                                                 int64_t* __restrict__ block_zeros,
                                                                 uint32_t* __restrict__ sup_ones) {
  const RsShape sh = rs_shape(length);
  const int v = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t sb0 = ((int64_t)blockIdx.x * RS_WARPS + (threadIdx.x >> 5)) * RS_SB_PER_WARP;
  if (sb0 >= sh.nsuper) return;
  uint64_t word[RS_SB_PER_WARP];
#pragma unroll
  for (int u = 0; u < RS_SB_PER_WARP; ++u) {
    const int64_t w = (sb0 + u) * RS_SB_WORDS + lane;
    word[u] = w < sh.nwords ? __ldcs(reinterpret_cast<const unsigned long long*>(words) + (int64_t)v * sh.nwords + w)
                            : 0ull;
  }
#pragma unroll
  for (int u = 0; u < RS_SB_PER_WARP; ++u) {
    const int64_t sb = sb0 + u;
    if (sb >= sh.nsuper) break;
    const uint32_t pc = (uint32_t)__popcll(word[u]);
    const uint32_t incl = warp_incl_scan(pc);
    const uint32_t excl = incl - pc;
    if ((lane & 3) == 0) {
      const int64_t b = sb * RS_BLK_PER_SB + (lane >> 2);
      if (b < sh.nblocks)
        block_zeros[(int64_t)v * sh.nblocks + b] = (int64_t)(lane >> 2) * RS_BLK_BITS - (int64_t)excl;
    }
    if (lane == 31) sup_ones[(int64_t)v * sh.nsuper + sb] = incl;
  }
}

// Pass 2 (after the scan of superblock one counts into `super_zeros`): turn
// the exclusive one prefixes into zero prefixes, record the select samples
// (at most one per bit value per superblock: 2048 < 8192) and the vector's one
// total.  A warp takes 32 superblocks, one per lane; only the superblocks that
// hold a sample are revisited word by word, cooperatively.
__global__ void __launch_bounds__(RS_WARPS * 32) rs_samples_kernel(const uint64_t* __restrict__ words, int64_t length,
                                                                  const uint32_t* __restrict__ sup_ones,
                                                                  int64_t* __restrict__ super_zeros,
                                                                  int64_t* __restrict__ samples1,
                                                                  int64_t* __restrict__ samples0,
                                                                  int64_t* __restrict__ ones_out) {
  const RsShape sh = rs_shape(length);
  const int v = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t sb0 = ((int64_t)blockIdx.x * RS_WARPS + (threadIdx.x >> 5)) * 32;
  if (sb0 >= sh.nsuper) return;
  const int64_t sb = sb0 + lane;
  const bool in = sb < sh.nsuper;
  int64_t cum1 = 0;
  uint32_t ones = 0;
  if (in) {
    cum1 = super_zeros[(int64_t)v * sh.nsuper + sb];  // ones before sb (scan output)
    ones = sup_ones[(int64_t)v * sh.nsuper + sb];
    super_zeros[(int64_t)v * sh.nsuper + sb] = sb * RS_SB_BITS - cum1;
    if (sb == sh.nsuper - 1) ones_out[v] = cum1 + ones;
  }
  const int64_t sb_bits = in ? min((int64_t)RS_SB_BITS, length - sb * RS_SB_BITS) : 0;
  // does a sample (ordinal 8192 k + 1) of ones / zeros fall into this superblock?
  int64_t kx[2];
  int needx[2];
  bool has[2];
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    const int64_t before = x ? cum1 : sb * RS_SB_BITS - cum1;
    const int64_t inside = x ? (int64_t)ones : sb_bits - (int64_t)ones;
    kx[x] = (before + RS_SAMPLE - 1) / RS_SAMPLE;
    has[x] = in && inside > 0 && kx[x] * RS_SAMPLE <= before + inside - 1;
    needx[x] = has[x] ? (int)(kx[x] * RS_SAMPLE - before + 1) : 0;
  }
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    uint32_t todo = __ballot_sync(FULL, has[x]);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const int64_t s = sb0 + src;
      const int need = __shfl_sync(FULL, needx[x], src);
      const int64_t k = __shfl_sync(FULL, kx[x], src);
      const int64_t w = s * RS_SB_WORDS + lane;
      uint64_t word = w < sh.nwords ? words[(int64_t)v * sh.nwords + w] : 0ull;
      if (!x) {
        const int64_t wbits = min((int64_t)64, max((int64_t)0, length - w * 64));
        word = ~word & (wbits >= 64 ? ~0ull : ((1ull << wbits) - 1ull));
      }
      const uint32_t pc = (uint32_t)__popcll(word);
      const uint32_t incl = warp_incl_scan(pc);
      const uint32_t excl = incl - pc;
      if ((int)excl < need && need <= (int)incl)
        (x ? samples1 : samples0)[(int64_t)v * sh.nsamp + k] = w * 64 + select_in_word64(word, need - (int)excl);
    }
  }
}

// Device view of one level's directory.
struct RsLevel {
  const uint64_t* words;
  const int64_t* super_zeros;
  const int64_t* block_zeros;
  const int64_t* samples1;
  const int64_t* samples0;
  int64_t ones;
};

struct RsArgs {
  const uint64_t* words;  // level-major, nwords per level
  const int64_t* super_zeros;
  const int64_t* block_zeros;
  const int64_t* samples1;
  const int64_t* samples0;
  const int64_t* ones;
  int64_t length;
};

__device__ __forceinline__ RsLevel rs_level(const RsArgs& a, const RsShape& sh, int l) {
  RsLevel L;
  L.words = a.words + (int64_t)l * sh.nwords;
  L.super_zeros = a.super_zeros + (int64_t)l * sh.nsuper;
  L.block_zeros = a.block_zeros + (int64_t)l * sh.nblocks;
  L.samples1 = a.samples1 + (int64_t)l * sh.nsamp;
  L.samples0 = a.samples0 + (int64_t)l * sh.nsamp;
  L.ones = a.ones[l];
  return L;
}

// rank1(i): ones in [0, i) (bitvec.py:190-207)
__device__ __forceinline__ int64_t rs_rank1(const RsLevel& L, const RsShape& sh, int64_t i) {
  if (i <= 0) return 0;
  const int64_t k = min(i >> 8, sh.nblocks - 1);
  int64_t r = (k << 8) - (L.super_zeros[k >> 3] + L.block_zeros[k]);
  const int64_t stop = i >> 6;
  for (int64_t w = k << 2; w < stop; ++w) r += __popcll(L.words[w]);
  const int rem = (int)(i & 63);
  if (rem) r += __popcll(L.words[stop] & ((1ull << rem) - 1ull));
  return r;
}

__device__ __forceinline__ int64_t rs_rank(const RsLevel& L, const RsShape& sh, int x, int64_t i) {
  const int64_t r1 = rs_rank1(L, sh, i);
  return x ? r1 : i - r1;
}

__device__ __forceinline__ int rs_get(const RsLevel& L, int64_t i) { return (int)((L.words[i >> 6] >> (i & 63)) & 1ull); }

// occurrences of x before superblock boundary s << 11 (bitvec.py:209-215)
__device__ __forceinline__ int64_t rs_count_before(const RsLevel& L, const RsShape& sh, int64_t length, int x,
                                                   int64_t s) {
  if (s >= sh.nsuper) return x ? L.ones : length - L.ones;
  const int64_t zeros = L.super_zeros[s];
  return x ? (s << 11) - zeros : zeros;
}

// select(x, j): 0-based position of the j-th occurrence, -1 when absent (bitvec.py:217-263)
__device__ int64_t rs_select(const RsLevel& L, const RsShape& sh, int64_t length, int x, int64_t j) {
  const int64_t total = x ? L.ones : length - L.ones;
  if (j < 1 || j > total) return -1;
  const int64_t* samples = x ? L.samples1 : L.samples0;
  const int64_t nsamp = (total + RS_SAMPLE - 1) / RS_SAMPLE;
  const int64_t si = (j - 1) / RS_SAMPLE;
  int64_t lo = samples[si] >> 11;
  int64_t hi = si + 1 < nsamp ? (samples[si + 1] >> 11) : sh.nsuper - 1;
  while (lo < hi) {  // last superblock whose boundary holds fewer than j occurrences
    const int64_t mid = (lo + hi + 1) >> 1;
    if (rs_count_before(L, sh, length, x, mid) < j) lo = mid;
    else hi = mid - 1;
  }
  const int64_t s = lo;
  int64_t k = s << 3;
  const int64_t last_block = min((s << 3) + RS_BLK_PER_SB, sh.nblocks) - 1;
  const int64_t sz = L.super_zeros[s];
  while (k < last_block) {
    const int64_t nz = sz + L.block_zeros[k + 1];
    const int64_t cnt = x ? ((k + 1) << 8) - nz : nz;
    if (cnt < j) ++k;
    else break;
  }
  const int64_t bz = sz + L.block_zeros[k];
  int64_t need = j - (x ? (k << 8) - bz : bz);
  const int64_t last_word = (length - 1) >> 6;
  for (int64_t w = k << 2;; ++w) {
    uint64_t word = L.words[w];
    const int width = (w == last_word && (length & 63)) ? (int)(length & 63) : 64;
    if (!x) word = ~word & (width == 64 ? ~0ull : ((1ull << width) - 1ull));
    const int c = __popcll(word);
    if (need > c) {
      need -= c;
      continue;
    }
    return (w << 6) + select_in_word64(word, (int)need);
  }
}



struct QueryArgs {
  RsArgs rs;
  const int64_t* zeros;  // WM zero counts
  int kind, op, width;
  const int64_t* sym;    // symbol per query (rank / select), or null
  int64_t sym_scalar;    // used when sym is null
  const int64_t* arg;    // i (access, rank) or j (select)
  int64_t* out;
  int64_t count;
};

// One thread per query: the level walks of structures.py:107-256.
__global__ void __launch_bounds__(256) query_kernel(const QueryArgs a) {
  const RsShape sh = rs_shape(a.rs.length);
  const int64_t n = a.rs.length;
  const int W = a.width;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < a.count;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = a.sym ? a.sym[q] : a.sym_scalar;
    const int64_t arg = a.arg[q];
    int64_t res = 0;
    if (a.op == WVLT_Q_BITRANK) {  // ones of level c in [0, arg)
      res = (c >= 0 && c < W) ? rs_rank1(rs_level(a.rs, sh, (int)c), sh, arg) : 0;
    } else if (a.kind == WVLT_KIND_WM) {
      if (a.op == WVLT_Q_ACCESS) {
        int64_t value = 0, pos = arg;
        for (int l = 0; l < W; ++l) {
          const RsLevel L = rs_level(a.rs, sh, l);
          const int b = rs_get(L, pos);
          value = (value << 1) | b;
          pos = b ? a.zeros[l] + rs_rank1(L, sh, pos) : pos - rs_rank1(L, sh, pos);
        }
        res = W ? value : 0;
      } else {
        int64_t s = 0, e = a.op == WVLT_Q_RANK ? arg : n;
        for (int l = 0; l < W; ++l) {
          const RsLevel L = rs_level(a.rs, sh, l);
          if ((c >> (W - 1 - l)) & 1) {
            s = a.zeros[l] + rs_rank1(L, sh, s);
            e = a.zeros[l] + rs_rank1(L, sh, e);
          } else {
            s = s - rs_rank1(L, sh, s);
            e = e - rs_rank1(L, sh, e);
          }
        }
        if (a.op == WVLT_Q_RANK) {
          res = W ? e - s : arg;
        } else if (W == 0) {
          res = arg <= n ? arg - 1 : -1;
        } else if (arg > e - s) {
          res = -1;
        } else {
          int64_t pos = s + arg - 1;
          for (int l = W - 1; l >= 0 && pos >= 0; --l) {
            const RsLevel L = rs_level(a.rs, sh, l);
            pos = ((c >> (W - 1 - l)) & 1) ? rs_select(L, sh, n, 1, pos - a.zeros[l] + 1)
                                           : rs_select(L, sh, n, 0, pos + 1);
          }
          res = pos;
        }
      }
    } else {  // tree: interval walks
      if (a.op == WVLT_Q_ACCESS) {
        int64_t value = 0, s = 0, e = n, pos = arg;
        for (int l = 0; l < W; ++l) {
          const RsLevel L = rs_level(a.rs, sh, l);
          const int64_t rs1 = rs_rank1(L, sh, s), re1 = rs_rank1(L, sh, e), rp1 = rs_rank1(L, sh, pos);
          const int64_t z = (e - re1) - (s - rs1);
          if (rs_get(L, pos)) {
            value = (value << 1) | 1;
            pos = s + z + (rp1 - rs1);
            s += z;
          } else {
            value <<= 1;
            pos = s + ((pos - rp1) - (s - rs1));
            e = s + z;
          }
        }
        res = W ? value : 0;
      } else if (a.op == WVLT_Q_RANK) {
        int64_t s = 0, e = n, k = arg;
        for (int l = 0; l < W; ++l) {
          const RsLevel L = rs_level(a.rs, sh, l);
          const int64_t rs1 = rs_rank1(L, sh, s), re1 = rs_rank1(L, sh, e);
          const int64_t z = (e - re1) - (s - rs1);
          if ((c >> (W - 1 - l)) & 1) {
            k = rs_rank1(L, sh, s + k) - rs1;
            s += z;
          } else {
            k = (s + k - rs_rank1(L, sh, s + k)) - (s - rs1);
            e = s + z;
          }
        }
        res = W ? k : arg;
      } else {
        if (W == 0) {
          res = arg <= n ? arg - 1 : -1;
        } else {
          int64_t starts[WVLT_MAX_WIDTH];
          int64_t s = 0, e = n;
          for (int l = 0; l < W; ++l) {
            const RsLevel L = rs_level(a.rs, sh, l);
            starts[l] = s;
            const int64_t rs1 = rs_rank1(L, sh, s), re1 = rs_rank1(L, sh, e);
            const int64_t z = (e - re1) - (s - rs1);
            if ((c >> (W - 1 - l)) & 1) s += z;
            else e = s + z;
          }
          if (arg > e - s) {
            res = -1;
          } else {
            int64_t off = arg - 1;
            for (int l = W - 1; l >= 0; --l) {
              const RsLevel L = rs_level(a.rs, sh, l);
              const int bit = (int)((c >> (W - 1 - l)) & 1);
              const int64_t p = rs_select(L, sh, n, bit, rs_rank(L, sh, bit, starts[l]) + off + 1);
              off = p - starts[l];
            }
            res = off;
          }
        }
      }
    }
    a.out[q] = res;
  }
}

}  // namespace

extern "C" {

size_t wvlt_rank_select_workspace_bytes(int64_t nvec, int64_t length) {
  if (nvec < 0 || length < 0) return 0;
  const RsShape sh = rs_shape(length);
  const int64_t nblk = (sh.nsuper + SCAN_TILE - 1) / SCAN_TILE;
  return align_up((size_t)nvec * sh.nsuper * 4, 256) + align_up((size_t)nvec * (nblk + 1) * 8, 256) + 256;
}

int wvlt_rank_select_build(const uint64_t* words, int64_t nvec, int64_t length, int64_t* super_zeros,
                           int64_t* block_zeros, int64_t* samples1, int64_t* samples0, int64_t* ones,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (nvec < 0 || length < 0 || nvec > 65535) return WVLT_E_ARG;
  if (nvec == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (length == 0) {
    cudaError_t e = cudaMemsetAsync(ones, 0, (size_t)nvec * 8, s);
    return (int)e;
  }
  if (!words || !super_zeros || !block_zeros || !samples1 || !samples0 || !ones || !workspace) return WVLT_E_ARG;
  if (workspace_bytes < wvlt_rank_select_workspace_bytes(nvec, length)) return WVLT_E_WORKSPACE;
  const RsShape sh = rs_shape(length);
  uint32_t* sup_ones = (uint32_t*)workspace;
  int64_t* bsum = (int64_t*)((unsigned char*)workspace + align_up((size_t)nvec * sh.nsuper * 4, 256));
  const int64_t per_cta = (int64_t)RS_WARPS * RS_SB_PER_WARP;
  const dim3 gb((unsigned)((sh.nsuper + per_cta - 1) / per_cta), (unsigned)nvec);
  rs_blocks_kernel<<<gb, RS_WARPS * 32, 0, s>>>(words, length, block_zeros, sup_ones);
  const int64_t nblk = (sh.nsuper + SCAN_TILE - 1) / SCAN_TILE;
  const dim3 gs((unsigned)nblk, (unsigned)nvec);
  scan_reduce_kernel<<<gs, SCAN_THREADS, 0, s>>>(sup_ones, sh.nsuper, nblk, bsum);
  scan_apply_kernel<<<gs, SCAN_THREADS, 0, s>>>(sup_ones, sh.nsuper, nblk, bsum, super_zeros);
  const dim3 gsm((unsigned)((sh.nsuper + RS_WARPS * 32 - 1) / (RS_WARPS * 32)), (unsigned)nvec);
  rs_samples_kernel<<<gsm, RS_WARPS * 32, 0, s>>>(words, length, sup_ones, super_zeros, samples1, samples0, ones);
  return (int)cudaGetLastError();
}

int wvlt_query(int kind, int op, const uint64_t* level_words, int64_t n, int width, const int64_t* zeros,
               const int64_t* super_zeros, const int64_t* block_zeros, const int64_t* samples1,
               const int64_t* samples0, const int64_t* ones, const int64_t* sym, int64_t sym_scalar,
               const int64_t* arg, int64_t* out, int64_t count, void* stream) {
  if (kind != WVLT_KIND_WT && kind != WVLT_KIND_WM) return WVLT_E_ARG;
  if (op < WVLT_Q_ACCESS || op > WVLT_Q_BITRANK || width < 0 || width > WVLT_MAX_WIDTH || n < 0 || count < 0)
    return WVLT_E_ARG;
  if (count == 0) return 0;
  if (!arg || !out || (width > 0 && n > 0 && (!level_words || !super_zeros || !block_zeros || !samples1 ||
                                              !samples0 || !ones)))
    return WVLT_E_ARG;
  if (kind == WVLT_KIND_WM && width > 0 && !zeros) return WVLT_E_ARG;
  QueryArgs q;
  q.rs.words = level_words;
  q.rs.super_zeros = super_zeros;
  q.rs.block_zeros = block_zeros;
  q.rs.samples1 = samples1;
  q.rs.samples0 = samples0;
  q.rs.ones = ones;
  q.rs.length = n;
  q.zeros = zeros;
  q.kind = kind;
  q.op = op;
  q.width = n > 0 ? width : 0;
  q.sym = sym;
  q.sym_scalar = sym_scalar;
  q.arg = arg;
  q.out = out;
  q.count = count;
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)sm_count() * 16);
  query_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(q);
  return (int)cudaGetLastError();
}

}  // extern "C"
