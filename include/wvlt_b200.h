/*
 * wvlt_b200.h -- C ABI of the B200 wavelet tree / wavelet matrix construction path.
 *
 * The reference (`wvlt`, Python + numba) has no C ABI: its operator layer is
 * the set of numba kernels in pkg/src/wvlt/_kernels.py, each of which takes
 * preallocated arrays, mutates them in place and returns nothing
 * (_kernels.py:1-13).  The entry points below replace those kernels and the
 * per-level orchestration in construct.py with sm_100a CUDA, keeping the same
 * conventions:
 *
 *   - every buffer is allocated by the caller (Python/torch or any other host
 *     runtime); the library never allocates device memory;
 *   - plain pointers and sizes only, no torch types;
 *   - everything is stream ordered on the `stream` argument (a cudaStream_t,
 *     NULL = legacy default stream);
 *   - return value 0 = success, > 0 = a cudaError_t, < 0 = a WVLT_E* contract
 *     error.  wvlt_error_string() names both.
 *
 * Output layout is the reference's BitVector layout (bitvec.py:3-8): level l
 * of a build over n symbols is ceil(n/64) uint64 words, bit j at word j>>6,
 * in-word position j&63 (LSB first), unused high bits of the last word zero.
 * All levels are packed back to back: level l starts at word l*ceil(n/64).
 */
#ifndef WVLT_B200_H
#define WVLT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WVLT_ABI_VERSION 1

/* structure kinds, same codes as the wire format (structures.py:24) */
#define WVLT_KIND_WT 0
#define WVLT_KIND_WM 1

/* contract errors (negative so they never collide with cudaError_t) */
#define WVLT_E_ARG (-1)        /* bad argument (null pointer, bad kind, bad sym_bytes, ...) */
#define WVLT_E_WIDTH (-2)      /* code width above WVLT_MAX_WIDTH */
#define WVLT_E_WORKSPACE (-3)  /* workspace smaller than wvlt_workspace_bytes() */
#define WVLT_E_RANGE (-4)      /* a symbol lies outside [0, sigma) (host-buffer entry only) */

/* largest supported code width ceil(lg sigma); the histogram fold chain is 2^(w+1) int64 */
#define WVLT_MAX_WIDTH 28

/* Bit in *status set by the device build when a symbol lies outside [0, sigma). */
#define WVLT_STATUS_RANGE 1

int wvlt_abi_version(void);
const char* wvlt_error_string(int code);

/* ceil(lg sigma), 0 for sigma <= 1.  Replaces bitperm.code_width (bitperm.py:18-22). */
int wvlt_code_width(int64_t sigma);

/* Device workspace needed by wvlt_build_device for this problem (bytes). */
size_t wvlt_workspace_bytes(int64_t n, int sym_bytes, int64_t sigma, int kind);

/*
 * What one build's workspace holds, by the reference ledger's categories
 * (construct.AllocationLog, construct.py:48-127): parts[0] "positions" (count
 * chains, node borders, placement tables, per-tile counts / prefixes / run
 * tables), parts[1] "symbols" (level-order buffers in HBM; 0 for a byte text,
 * whose fused pass keeps every order in shared memory), parts[2]
 * "partial_bits" (a wide-alphabet tree's matrix before the reorder).  Bytes;
 * want_hist / want_borders as the build requests them.
 */
int wvlt_workspace_parts(int64_t n, int sym_bytes, int64_t sigma, int kind, int want_hist, int want_borders,
                         size_t* parts);

/*
 * Symbol histogram, padded to 2^width bins, plus the range check.
 * Replaces hist_and_msb_bits / full_histogram (_kernels.py:23-42) and
 * levelstats.symbol_histogram (levelstats.py:30-47).
 *   text      device, n symbols of sym_bytes (1, 2 or 4) bytes, unsigned
 *   hist      device int64[2^width], overwritten
 *   status    device int32, WVLT_STATUS_RANGE is OR-ed in on a bad symbol (may be NULL)
 */
int wvlt_histogram(const void* text, int sym_bytes, int64_t n, int64_t sigma, int64_t* hist,
                   int32_t* status, void* stream);

/*
 * Full device-resident build of one wavelet tree (kind WVLT_KIND_WT) or wavelet
 * matrix (WVLT_KIND_WM).  Replaces build_by_prefix_counting / build_by_prefix_sorting
 * (construct.py:292-387) and their kernels hist_and_msb_bits, fold_pairs,
 * starts_identity, starts_ordered, sort_level_pass, scatter_by_prefix and
 * write_bits_from_symbols (_kernels.py:23-193).
 *   text         device, n symbols (sym_bytes = 1, 2 or 4), values must lie in [0, sigma);
 *                any address works, but only a 16-byte aligned one (32 for sigma <= 8) gets
 *                the vector / bulk loads -- several times slower otherwise
 *   level_words  device uint64[width * ceil(n/64)], fully overwritten
 *   zeros        device int64[width] or NULL: WM zero counts Z[l] (construct.py:273-288);
 *                for kind WT the same per-level zero counts are written
 *   hist         device int64[2^width] or NULL: the padded symbol histogram
 *   borders      device int64[max(2^width - 2, 0)] or NULL: node borders, level l
 *                (1 <= l < width) at [2^l - 2, 2^(l+1) - 2), indexed by l-bit prefix.
 *                WT: interval_starts(fold^(w-l)(hist)) (levelstats.py:58-73);
 *                WM: the same with bit-reversed order, i.e. wt2wm.interval_start_table
 *                (wt2wm.py:55-78)
 *   workspace    device, >= wvlt_workspace_bytes(n, sym_bytes, sigma, kind) bytes
 *   status       device int32 or NULL; set to 0 then WVLT_STATUS_RANGE on a bad symbol
 * When status reports a bad symbol the level words are unspecified (the caller
 * raises, like construct._validated, construct.py:183-187).
 * A WM build with hist == NULL and borders == NULL computes no histogram at all:
 * its per-level tables and zero counts come from the tile digit counts of each
 * pass (the output is identical).
 */
int wvlt_build_device(const void* text, int sym_bytes, int64_t n, int64_t sigma, int kind,
                      uint64_t* level_words, int64_t* zeros, int64_t* hist, int64_t* borders,
                      void* workspace, size_t workspace_bytes, int32_t* status, void* stream);

/*
 * Same build with HOST input and HOST outputs: copies text host->device,
 * builds, copies level words / zeros / histogram device->host and synchronizes
 * `stream`.  Device buffers are caller-provided (dev_text: n*sym_bytes bytes,
 * dev_level_words: width*ceil(n/64)*8 bytes, dev_small: (2^width + width + 1)*8 bytes).
 * Page-locked host buffers get direct DMA; pageable ones are staged through
 * page-locked chunks by several host threads (the output pages are faulted in
 * while the text goes up).  host_zeros and
 * host_hist may be NULL (host_hist == NULL selects the histogram-free WM build).  Returns WVLT_E_RANGE when a symbol is out of range.
 * This is the call a reference-side binding (ctypes / cgo / JNI) would make
 * in place of construct.build_structure (construct.py:150-164).
 */
int wvlt_build_host(const void* host_text, int sym_bytes, int64_t n, int64_t sigma, int kind,
                    uint64_t* host_level_words, int64_t* host_zeros, int64_t* host_hist,
                    void* dev_text, uint64_t* dev_level_words, void* dev_small,
                    void* workspace, size_t workspace_bytes, void* stream);

/*
 * wvlt_build_host plus the node borders (layout of wvlt_build_device's
 * `borders`) copied to host_borders (int64[max(2^width - 2, 0)], may be NULL).
 * With host_borders, dev_small must hold (2^(width+1) + width - 1) int64.
 * This is the drop-in's call: the reference's structures expose the node
 * borders (levelstats.interval_starts, levelstats.py:58-73, for the tree;
 * wt2wm.interval_start_table, wt2wm.py:55-78, for the matrix).
 */
int wvlt_build_host_borders(const void* host_text, int sym_bytes, int64_t n, int64_t sigma, int kind,
                            uint64_t* host_level_words, int64_t* host_zeros, int64_t* host_hist,
                            int64_t* host_borders, void* dev_text, uint64_t* dev_level_words, void* dev_small,
                            void* workspace, size_t workspace_bytes, void* stream);

/*
 * `count` independent builds with host buffers (same sym_bytes, sigma and kind;
 * text i has ns[i] symbols), software-pipelined over three streams: the text of
 * build i+1 goes host->device while build i runs on `stream` and build i-1's
 * level words come back (pass by pass, as in wvlt_build_host).  PCIe is full
 * duplex, so in steady state a build costs max(upload, download, compute)
 * instead of their sum -- the serving form of wvlt_build_host for a queue of
 * texts.  Device buffers hold two slots each: dev_text 2 x dev_text_slot_bytes,
 * dev_level_words 2 x dev_words_slot_bytes, dev_small 2 x (2^width + width + 1)
 * int64.  Outputs: host_level_words[i] (width x ceil(ns[i]/64) words),
 * host_zeros + i*width (may be NULL), host_hist + i*2^width (may be NULL: the
 * histogram-free WM build), host_status[i] (nonzero flags: build i saw a symbol
 * out of range).  Synchronizes before returning; returns WVLT_E_RANGE if any
 * build saw an out-of-range symbol.  The overlap needs page-locked texts and
 * level-word buffers; pageable ones are accepted (the copies then serialise).
 */
int wvlt_build_host_batch(int count, const void* const* host_texts, const int64_t* ns, int sym_bytes,
                          int64_t sigma, int kind, uint64_t* const* host_level_words, int64_t* host_zeros,
                          int64_t* host_hist, int32_t* host_status, void* dev_text, size_t dev_text_slot_bytes,
                          uint64_t* dev_level_words, size_t dev_words_slot_bytes, void* dev_small,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Number of this library's kernels the calling thread's last build launched. */
int wvlt_last_launches(void);

/*
 * Stream ordered bit intervals into whole destination words: destination bit
 * range [bounds[t], bounds[t+1]) receives source bits starting at src_starts[t],
 * for t < ntasks; the tasks tile [0, n_bits).  Writes destination words
 * [word_lo, word_hi) whole (zero padding included).  Replaces gather_bits
 * (_kernels.py:196-232), used by the domain-decomposed merge
 * (construct.py:497-507) -- here the multi-GPU merge -- and by convert_wt_to_wm
 * (wt2wm.py:225).
 */
int wvlt_merge_bits(uint64_t* dst_words, int64_t word_lo, int64_t word_hi, int64_t n_bits,
                    const int64_t* bounds, const int64_t* src_starts, int64_t ntasks,
                    const uint64_t* src_words, void* stream);

/*
 * Multi-GPU merge over peer memory (one launch for every level): destination
 * row l (dst_words + l * dst_row_words) receives global words [word_lo, word_hi)
 * of level l, assembled straight from the source ranks' local levels --
 * level_src[l * nranks + r] points at rank r's local level l words, a
 * peer-mapped (NVLink P2P / symmetric-memory) device pointer.  Level l's tasks
 * are t in [task_off[l], task_off[l+1]): destination bits
 * [b[t'], b[t'+1]) with b = bounds + bounds_off[l] and t' = t - task_off[l]
 * come from rank src_ranks[t] starting at local bit src_starts[t]; they cover
 * the owned bit range.  bounds_off / task_off / bounds / src_* / level_src are
 * device arrays.  Replaces the all-to-all + gather_bits pair of the
 * domain-decomposed merge (construct.py:497-507, _kernels.py:196-232) when the
 * ranks' memories are peer-accessible.
 */
int wvlt_merge_levels_peer(uint64_t* dst_words, int64_t dst_row_words, int width, int64_t word_lo, int64_t word_hi,
                           int64_t n_bits, const int64_t* bounds, const int64_t* bounds_off, const int64_t* src_starts,
                           const int32_t* src_ranks, const int64_t* task_off, const uint64_t* const* level_src,
                           int nranks, void* stream);

/*
 * The merge plan of wvlt_merge_levels_peer for every level and every owner, on
 * the device, from the all-gathered per-rank build outputs (replaces
 * construct._merge_plan, construct.py:516-543, and its host-side use in the
 * domain-decomposed build, construct.py:490-507).  Rank r's row starts at
 * rows + r * row_stride; its node borders (wvlt_build_device `borders` layout:
 * level l at [2^l - 2, 2^(l+1) - 2), indexed by prefix) start at column
 * borders_col.  local_ns[r] = rank r's symbol count.  Level l gets
 * nranks * 2^l tasks ((group in interval order) x rank, group-major, empty
 * tasks kept): task_off[l] = nranks (2^l - 1), bounds_off[l] = task_off[l] + l;
 * bounds / src_starts / src_ranks must hold nranks (2^width - 1) + width,
 * nranks (2^width - 1) and nranks (2^width - 1) entries, task_off width + 1 and
 * bounds_off width.  All arrays are device memory; no host work.
 */
int wvlt_peer_plan(const int64_t* rows, int64_t row_stride, int64_t borders_col, const int64_t* local_ns, int nranks,
                   int width, int kind, int64_t* bounds, int64_t* src_starts, int32_t* src_ranks, int64_t* bounds_off,
                   int64_t* task_off, void* stream);

/*
 * Rank/select directories of nvec bit vectors of `length` bits stored back to
 * back (ceil(length/64) words each, the level layout above).  Replaces
 * RankSelectBitVector._build (bitvec.py:135-163), same arrays per vector:
 *   super_zeros  int64[nvec][ceil(length/2048)]  zeros before each 2048-bit superblock
 *   block_zeros  int64[nvec][ceil(length/256)]   zeros before each 256-bit block, relative
 *                                                to its superblock
 *   samples1/0   int64[nvec][ceil(length/8192)]  position of the (8192k+1)-th one / zero;
 *                                                the first ceil(count/8192) entries are valid
 *   ones         int64[nvec]                     ones per vector
 * workspace: >= wvlt_rank_select_workspace_bytes(nvec, length) bytes.
 */
size_t wvlt_rank_select_workspace_bytes(int64_t nvec, int64_t length);
int wvlt_rank_select_build(const uint64_t* words, int64_t nvec, int64_t length, int64_t* super_zeros,
                           int64_t* block_zeros, int64_t* samples1, int64_t* samples0, int64_t* ones,
                           void* workspace, size_t workspace_bytes, void* stream);

/* query operations of wvlt_query */
#define WVLT_Q_ACCESS 0 /* out[q] = symbol at position arg[q] */
#define WVLT_Q_RANK 1   /* out[q] = occurrences of symbol c in [0, arg[q]) */
#define WVLT_Q_SELECT 2 /* out[q] = position of the arg[q]-th (1-based) c, or -1 when absent */
#define WVLT_Q_BITRANK 3 /* out[q] = ones of level c in bit positions [0, arg[q]) (0 <= c < width) */

/*
 * Batched queries on a built structure with its level directories (one
 * thread per query): access / rank / select of LevelWiseWaveletTree and
 * WaveletMatrix (structures.py:107-256).  The symbol c of query q is sym[q],
 * or sym_scalar when sym is NULL.  Arguments must be in range (access:
 * 0 <= i < n; rank: 0 <= i <= n, 0 <= c < 2^width; select: j >= 1) -- the
 * caller validates, as the reference's _check_* helpers do.
 */
int wvlt_query(int kind, int op, const uint64_t* level_words, int64_t n, int width, const int64_t* zeros,
               const int64_t* super_zeros, const int64_t* block_zeros, const int64_t* samples1,
               const int64_t* samples0, const int64_t* ones, const int64_t* sym, int64_t sym_scalar,
               const int64_t* arg, int64_t* out, int64_t count, void* stream);

/*
 * Optional per-stage timing (CUDA events on the build stream) of the calling
 * thread's wvlt_build_device calls.  Stage ids: WVLT_STAGE_MEMSET (output and
 * look-back reset), WVLT_STAGE_HIST (K1), WVLT_STAGE_TABLES (K2),
 * WVLT_STAGE_SCAN0 + p (tile-prefix scan of pass p), WVLT_STAGE_PASS0 + p
 * (fused level pass p).  wvlt_profile_read synchronizes
 * on the last event and returns the number of stages written.
 */
#define WVLT_STAGE_MEMSET 0
#define WVLT_STAGE_HIST 1
#define WVLT_STAGE_TABLES 2
#define WVLT_STAGE_PASS0 3
#define WVLT_STAGE_SCAN0 64
#define WVLT_STAGE_REORDER 60 /* WT of a wide alphabet: matrix levels reordered into tree order */
int wvlt_profile_enable(int on);
int wvlt_profile_read(float* stage_ms, int* stage_ids, int max_stages);

#ifdef __cplusplus
}
#endif

#endif /* WVLT_B200_H */
