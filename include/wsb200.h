/*
 * wsb200.h -- C ABI of the B200-native batched pairwise-alignment library (libwsb200.so).
 *
 * This is the drop-in boundary for the reference's batch hot path.  Every entry point is plain C: pointers and
 * sizes only, no C++/torch types.  Functions return 0 on success or a negative wsb_status; they never throw.
 *
 * What each entry point replaces in the reference (pkg/src/waveseq/):
 *   wsb_score_batch      batch.run_batch in score_only mode: the worker pool over _run_unit -> engine_score /
 *                        engine_score_packed (batch.py:167-247, engine.py:383-400, 512-597), i.e. the numba kernels
 *                        K.run_linear32 / run_merged32 / run_exact32 / run_linear16 / run_merged16
 *                        (engine.py:333-363, 574-585; _kernels.py:181-201, 337-357, 502-524, 684-698, 843-858).
 *   wsb_traceback_batch  batch.run_batch in traceback mode (batch.py:174-175); CIGARs follow the full-matrix walk
 *                        refdp.ref_traceback (refdp.py:158-235), see DESIGN.md "CIGAR oracle".
 *   wsb_batch_*          the same two calls split into upload / run / download so a caller can keep the sequence
 *                        pools resident in HBM (BatchJob's queries/subjects/pairs, batch.py:68-89).
 *   wsb_plan_shards      the cell-count balanced replacement of _plan_units/_chunk_units (batch.py:118-164) used to
 *                        shard one job over several GPUs (one wsb_ctx per GPU, no collective).
 *
 * Sequence pools: one byte per symbol, 0..3 = A,C,G,T, 4 (or any value >= 4) = flagged / non-ACGT
 * (core.py:63-118; engine._encode_q5, engine.py:203-207).  Sequence k of a pool occupies
 * codes[off[k] .. off[k] + len[k]).  A pair p aligns query pair_q[p] (rows, CIGAR 'I' consumes it) against
 * subject pair_s[p] (columns, CIGAR 'D' consumes it).
 *
 * Results are written by pair index, so they do not depend on scheduling, variant or GPU count
 * (batch.py:206, tests/test_batch.py:89-99).
 */
#ifndef WSB200_H
#define WSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wsb_ctx wsb_ctx;     /* one per GPU: device, streams, scratch.  Not re-entrant. */
typedef struct wsb_batch wsb_batch; /* device-resident sequence pools + pair list + result buffers */

typedef struct wsb_scheme {
    int32_t match;      /* ScoringScheme.match_score   (core.py:125) */
    int32_t mismatch;   /* ScoringScheme.mismatch_score */
    int32_t gap_open;   /* alpha >= 0: cost of the first symbol of a gap run */
    int32_t gap_extend; /* beta >= 0: cost of each further symbol (affine only) */
    int32_t gap_model;  /* WSB_GAP_LINEAR | WSB_GAP_AFFINE */
} wsb_scheme;

enum wsb_align_type { WSB_GLOBAL = 0, WSB_LOCAL = 1, WSB_SEMIGLOBAL = 2 }; /* engine._ATYPE, engine.py:34 */
enum wsb_gap_model { WSB_GAP_LINEAR = 0, WSB_GAP_AFFINE = 1 };

/* Arithmetic variant of the score kernels.  AUTO picks, per pair, the packed half2 kernel when every DP value is an
 * exactly representable fp16 integer (|v| <= 2048) and the scheme allows the merged gap state
 * (engine.merged_state_exact, engine.py:71-94), else the int32 kernel.  Forcing F16X2 makes out-of-range pairs fail
 * with WSB_E_RANGE in their status slot (the reference's PackedRangeOverflow, engine.py:530-534). */
enum wsb_variant { WSB_VARIANT_AUTO = 0, WSB_VARIANT_F16X2 = 1, WSB_VARIANT_I32 = 2, WSB_VARIANT_S16X2 = 3 };
/* S16X2 (opt-in, experimental): routed like AUTO, but short local alignments (reads that fit one 152-column stage,
 * scheme within one byte) take the packed int16 DPX kernel of score_short16.cuh instead of the half2 kernel -- two
 * alignments per thread, exact in 16-bit integers; pairs with a flagged subject symbol are re-scored by the half2
 * kernel inside the same call.  Results are identical; AUTO does not pick it yet because it is currently slower
 * (DESIGN.md 4.6). */

enum wsb_status {
    WSB_OK = 0,
    WSB_E_CUDA = -1,     /* CUDA runtime / launch failure; see wsb_last_error */
    WSB_E_ARG = -2,      /* bad argument (null pointer, index out of range, unknown enum) */
    WSB_E_NOMEM = -3,    /* host or device allocation failed */
    WSB_E_LENGTH = -4,   /* max_step*(m+n) >= 2^29  (core.check_length_bounds, core.py:191-195) */
    WSB_E_RANGE = -5,    /* pair does not fit the forced packed variant (PackedRangeOverflow) */
    WSB_E_SCHEME = -6,   /* forced packed variant with an affine scheme the merged state cannot represent */
    WSB_E_CAPACITY = -7, /* caller-provided CIGAR buffer too small */
    WSB_E_NODEVICE = -8  /* no CUDA device */
};

const char* wsb_strerror(int status);
const char* wsb_version(void);
int wsb_device_count(int* count);

int wsb_ctx_create(int device, wsb_ctx** out);
void wsb_ctx_destroy(wsb_ctx* ctx);
const char* wsb_last_error(const wsb_ctx* ctx);
int wsb_ctx_sm_count(const wsb_ctx* ctx);
/* Host threads that pack large one-byte-per-symbol pools (>= 262144 pairs and >= 32 MB: the piecewise upload) into the 2-bit
 * layout before they cross the bus -- a quarter of the bytes; the kernels of a piece start as soon as its slice is expanded on
 * the device.  Flagged symbols have no 2-bit code: a slice that holds one travels as plain bytes.  threads = 0 switches the
 * packing off (pools go up as they are: the better choice when several GPUs, each behind its own PCIe link, share the host
 * cores), -1 restores the default (WSB_HOST_PACK_THREADS, else min(16, cores - 1)).  No counterpart in the reference (its
 * workers read host memory in place, batch.py:213-240). */
int wsb_ctx_set_host_pack_threads(wsb_ctx* ctx, int threads);
const char* wsb_host_pack_isa(void);   /* "avx512bw", "bmi2" or "plain": the packing body the running CPU selected */

/* ---- resident-batch API ---- */

/* Copy the pools and the pair list to the device (async on the ctx stream) and build the execution plan inputs
 * (per-pair lengths).  Host arrays may be pageable or pinned; they are not referenced after the call returns. */
int wsb_batch_create(wsb_ctx* ctx, const uint8_t* q_codes, const int64_t* q_off, const int32_t* q_len, int64_t n_q,
                     const uint8_t* s_codes, const int64_t* s_off, const int32_t* s_len, int64_t n_s,
                     const int32_t* pair_q, const int32_t* pair_s, int64_t n_pairs, wsb_batch** out);
/* Same, but returns while the copies are still in flight on the context's copy stream: the host arrays must stay
 * valid and unchanged until the first wsb_batch_score / wsb_batch_traceback on the batch has been followed by a fetch
 * (or until wsb_batch_destroy).  Large batches are uploaded in up to eight pieces and the first score call launches
 * piece by piece, so the transfer of later pieces overlaps the kernels of earlier ones (pinned host memory makes the
 * copies truly asynchronous; pageable memory is staged by the driver). */
int wsb_batch_create_async(wsb_ctx* ctx, const uint8_t* q_codes, const int64_t* q_off, const int32_t* q_len, int64_t n_q,
                           const uint8_t* s_codes, const int64_t* s_off, const int32_t* s_len, int64_t n_s,
                           const int32_t* pair_q, const int32_t* pair_s, int64_t n_pairs, wsb_batch** out);
/* Same as wsb_batch_create_async for pools kept in the reference's 2-bit layout (Sequence.data, core.py:78-87: four
 * symbols per byte, low bits first), here over the concatenated pool: symbol k of the pool sits in bits 2*(k%4) of byte
 * k/4.  Flagged (non-ACGT) symbols, stored as code 0 in the packed data like the reference does (core.py:101-114), are
 * listed by pool position in q_flag_pos / s_flag_pos.  A quarter of the bytes cross the bus; the pools are expanded to
 * one byte per symbol on the device, slice by slice. */
int wsb_batch_create_packed_async(wsb_ctx* ctx, const uint8_t* q_packed, const int64_t* q_flag_pos, int64_t n_q_flags,
                                  const int64_t* q_off, const int32_t* q_len, int64_t n_q, const uint8_t* s_packed,
                                  const int64_t* s_flag_pos, int64_t n_s_flags, const int64_t* s_off, const int32_t* s_len,
                                  int64_t n_s, const int32_t* pair_q, const int32_t* pair_s, int64_t n_pairs, wsb_batch** out);
/* Regular batch without metadata arrays: n_pairs reads of q_len symbols back to back in the query pool, n_pairs reads
 * of s_len symbols in the subject pool, pair i = (read i, read i).  Give each pool either as bytes (x_codes) or in the
 * 2-bit layout (x_packed, no flagged symbols), the other pointer null; both pools in the same form.  Offsets, lengths
 * and the pair list are generated on the device and nothing is scanned on the host. */
int wsb_batch_create_uniform_async(wsb_ctx* ctx, const uint8_t* q_codes, const uint8_t* q_packed, int32_t q_len,
                                   const uint8_t* s_codes, const uint8_t* s_packed, int32_t s_len, int64_t n_pairs,
                                   wsb_batch** out);
void wsb_batch_destroy(wsb_batch* b);

/* Score every pair on the device; results stay in HBM until wsb_batch_fetch_scores.  kernel_ms (optional) receives
 * the device time of the launched kernels measured with CUDA events on the ctx stream; n_launches (optional) the
 * number of kernels launched.  Plans are cached per (scheme, align_type, variant). */
int wsb_batch_score(wsb_batch* b, const wsb_scheme* scheme, int align_type, int variant, float* kernel_ms,
                    int32_t* n_launches);

/* out_i/out_j: end cell (query, subject), 1-based matrix coordinates = exclusive 0-based span ends; global -> (m, n).
 * status (optional): per-pair wsb_status (0 or WSB_E_LENGTH / WSB_E_RANGE). */
int wsb_batch_fetch_scores(wsb_batch* b, int32_t* out_score, int32_t* out_i, int32_t* out_j, int32_t* status);

/* wsb_batch_score + wsb_batch_fetch_scores in one call.  While the batch is still uploading piece by piece (the first score
 * after wsb_batch_create_*_async) the results of every finished piece are downloaded on their own stream under the upload
 * and the kernels of later pieces, so a step's download costs no time of its own.  Same outputs and status contract. */
int wsb_batch_score_fetch(wsb_batch* b, const wsb_scheme* scheme, int align_type, int variant, float* kernel_ms,
                          int32_t* n_launches, int32_t* out_score, int32_t* out_i, int32_t* out_j, int32_t* status);

/* Direction-code fill + on-device walk + run-length CIGAR emission.  cigar receives runs packed as
 * (length << 2) | op with op 0 = M, 1 = I, 2 = D in forward order; pair p owns cigar[cigar_off[p] .. cigar_off[p+1]).
 * cigar_off has n_pairs + 1 entries.  If cigar_cap is too small the call returns WSB_E_CAPACITY and
 * cigar_off[n_pairs] holds the required run count. */
int wsb_batch_traceback(wsb_batch* b, const wsb_scheme* scheme, int align_type, float* kernel_ms, int32_t* n_launches);
int wsb_batch_fetch_traceback(wsb_batch* b, int32_t* out_score, int32_t* q_start, int32_t* q_end, int32_t* s_start,
                              int32_t* s_end, uint32_t* cigar, int64_t cigar_cap, int64_t* cigar_off, int32_t* status);

/* Bounded-memory traceback (the reference's linear-space path: traceback.py:208-344 hirschberg, :312-344
 * locate_endpoints).  A pair whose direction codes (0.5 byte per cell) exceed the scratch budget is traced through
 * checkpointed tiles instead: same path as the full-matrix walk, 8/R + 8/512 bytes per cell.  wsb_batch_set_tb_scratch
 * overrides the budget of this batch (bytes; 0 = library default 16 GiB or WSB_TB_SCRATCH_MB); wsb_batch_tb_info
 * reports the last traceback call: out4 = {pairs that took the bounded path, cells they computed, tiles re-filled by
 * their walks, peak scratch bytes of one such pair}. */
int wsb_batch_set_tb_scratch(wsb_batch* b, int64_t bytes);
int wsb_batch_tb_info(const wsb_batch* b, int64_t* out4);

/* 1 when the last plan of the batch holds per-pair faults (then fetch the status array), else 0 */
int wsb_batch_has_faults(const wsb_batch* b);
/* Page-locked host memory for result buffers, recycled by the library (a fetch into such a block runs at PCIe speed;
 * pageable destinations are staged by the driver).  Blocks are process-wide, not tied to a context. */
int wsb_pinned_alloc(size_t bytes, void** out);
void wsb_pinned_free(void* block);

int64_t wsb_batch_h2d_bytes(const wsb_batch* b);   /* bytes uploaded at creation (arrays generated on the device excluded) */
int64_t wsb_batch_total_runs(const wsb_batch* b);  /* CIGAR runs of the last traceback (size the cigar buffer with it); -1 if none */
int64_t wsb_batch_total_cells(const wsb_batch* b); /* sum of m*n over pairs (BatchReport.total_cells, batch.py:243-247) */

/* ---- one-shot host API (host buffers in, host buffers out) ---- */
int wsb_score_batch(wsb_ctx* ctx, const wsb_scheme* scheme, int align_type, int variant, const uint8_t* q_codes,
                    const int64_t* q_off, const int32_t* q_len, int64_t n_q, const uint8_t* s_codes,
                    const int64_t* s_off, const int32_t* s_len, int64_t n_s, const int32_t* pair_q,
                    const int32_t* pair_s, int64_t n_pairs, int32_t* out_score, int32_t* out_i, int32_t* out_j,
                    int32_t* status);

int wsb_traceback_batch(wsb_ctx* ctx, const wsb_scheme* scheme, int align_type, const uint8_t* q_codes,
                        const int64_t* q_off, const int32_t* q_len, int64_t n_q, const uint8_t* s_codes,
                        const int64_t* s_off, const int32_t* s_len, int64_t n_s, const int32_t* pair_q,
                        const int32_t* pair_s, int64_t n_pairs, int32_t* out_score, int32_t* q_start, int32_t* q_end,
                        int32_t* s_start, int32_t* s_end, uint32_t* cigar, int64_t cigar_cap, int64_t* cigar_off,
                        int32_t* status);

/* ---- host-only helpers (no GPU needed) ---- */

/* engine.merged_state_exact (engine.py:71-94) */
int wsb_merged_state_exact(const wsb_scheme* scheme);
/* 1 when an m x n problem under the scheme is exact in the packed half2 kernel (all values integers, |v| <= 2048) */
int wsb_f16_range_ok(const wsb_scheme* scheme, int32_t m, int32_t n);
/* Cell-count balanced sharding of pairs over n_shards GPUs (longest-processing-time first).  shard_of[p] receives
 * the shard of pair p; shard_cells[k] (optional) the cells assigned to shard k. */
int wsb_plan_shards(const int32_t* q_len, const int32_t* s_len, const int32_t* pair_q, const int32_t* pair_s,
                    int64_t n_pairs, int32_t n_shards, int32_t* shard_of, int64_t* shard_cells);

/* Geometry counters of the batch's last plan -- the GPU counterpart of the reference's EngineStats (engine.py:109-146,
 * pinned by tests/test_engine.py:187-245): out8 = {stages, wavefront iterations, cell updates executed (padding included,
 * stages * m * stage width per alignment), max instructions, add / sub instructions, substitution lookups (thread-instruction
 * counts of the kernels' cell bodies: packed kernels advance two cells per instruction), launch groups, pairs launched}. */
int wsb_batch_plan_stats(const wsb_batch* b, int64_t* out8);

/* SM cycles the last packed int16 short-read launch of the batch took (largest per-block clock64 span; 0 if none ran):
 * the denominator of the cycle-based roofline fraction, independent of the clock the GPU happened to hold. */
int64_t wsb_batch_kernel_cycles(wsb_batch* batch);

/* Gather sequences ids[0 .. n_ids) of a pool into a compact pool: out_codes (sum of their lengths) receives them back to
 * back, out_off[k] the new offset of sequence ids[k].  Used by the multi-GPU runner so that every shard uploads only the
 * sequences its pairs reference (the reference's worker threads share one read-only copy, batch.py:213-240). */
int wsb_compact_pool(const uint8_t* codes, const int64_t* off, const int32_t* len, const int64_t* ids, int64_t n_ids,
                     uint8_t* out_codes, int64_t* out_off);

#ifdef __cplusplus
}
#endif
#endif /* WSB200_H */
