// score_long.cuh -- int32 score kernel for long reads (1 kbp .. 100 kbp+): column stages of one pair are pipelined
// over the warps of a block, only the stage borders leave the register file.
//
// A pair's matrix is cut into column stages of 32 lanes x 16 columns = 512 columns.  Warp w of a block of NW warps owns
// stages w, w + NW, w + 2 NW, ... and sweeps each of them top to bottom as a lane wavefront (lane t computes row it - t
// at iteration it, exactly like score_kernels.cuh).  A stage's right-most column {T - gamma, H} is the only state the
// next stage needs; lane 31 streams it row by row into a global scratch column (8 bytes per row, L2 resident), and
// the warp owning the next stage follows 64-96 rows behind: it polls a shared-memory progress counter once per 32 rows,
// pulls the next 32 border rows with one coalesced 256-byte load, parks them in shared memory and feeds lane 0 from
// there.  So a 100 kbp x 100 kbp pair keeps up to 16 warps busy instead of one, a 10 kbp pair four, and no lane ever
// waits on a per-row global load.  NW + 1 scratch columns per block make the reuse of a column race-free by
// construction: the warp that overwrites column (s mod (NW+1)) with stage s + NW + 1 is the warp that consumed it.
//
// Blocks take pairs from a work queue (atomic counter) over a work-descending list, i.e. longest-processing-time-first.
//
// Cell update (reference: _kernels.py:259-276 merged affine, :113-126 linear; same algebra as score_kernels.cuh, with
// TA = T - alpha and TG = T - gamma kept per column so that both maxima are single 3-input DPX instructions):
//     d     = H_diag + sigma = dp4a(profile[c], onehot(q), H_diag)   IDP.4A   profile bytes = sigma(a, s_c), a = 0..3
//     h     = max3(TA_up, TA_left, d [,0])                           VIMNMX3[.RELU]
//     tn    = max3(TG_up, TG_left, d [,0])                           VIMNMX3[.RELU]
//     TA    = tn - alpha ; TG = tn - gamma                           2 x IMAD
// = 5 instructions per cell (the reference counts 7, local 8: _kernels.py:277-279).  A flagged query symbol (one-hot
// word 0) takes a lane-divergent copy of the row with sigma = mismatch.
#pragma once
#include "score_kernels.cuh"

#include <cooperative_groups.h>
#include <type_traits>

namespace wsb {

constexpr int kLongK = 16;
constexpr int kLongW = 32 * kLongK;
constexpr int kLongMaxWarps = 16;

struct LongParams {
    const uint8_t* q_codes; const int64_t* q_off; const int32_t* q_len;
    const uint8_t* s_codes; const int64_t* s_off; const int32_t* s_len;
    const int32_t* pair_q; const int32_t* pair_s;
    const int32_t* units;  // pair indices, work-descending
    int64_t n_units;
    int32_t* out_score; int32_t* out_i; int32_t* out_j;
    int32_t match, mismatch, alpha, beta;  // beta == alpha for the linear model
    int2* bnd;             // per block: (NW + 1) border columns of bnd_rows entries {T - gamma, H}
    int64_t bnd_rows;
    unsigned int* queue;   // work queue head, zeroed before the launch
    int32_t* redo; int32_t* redo_count;   // packed int16 kernel (score_long16.cuh): pairs handed back to this kernel
    const int32_t* n_units_dev;           // re-score launch: number of units is read from the device
    int32_t* cflags;       // cluster launches: per cluster kLongCf ints (progress counters of its warps, unit slot, reduction slots)
    int32_t one;           // 1, opaque to the compiler: keeps selected adds on the FMA pipe as IMAD
};

__device__ __forceinline__ int prmt(unsigned a, unsigned b, unsigned sel) {
    unsigned d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return (int)d;
}
// a * one + b with one == 1 at run time: an add that issues on the FMA pipe
__device__ __forceinline__ int fma_add(int a, int one, int b) {
    int d;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(one), "r"(b));
    return d;
}

using LongFn = void (*)(const LongParams);

// flag block of a cluster launch (LongParams::cflags): progress counters of up to 16 x 16 warps + 1, stage counter, unit slot,
// one (value, row, column) reduction slot per block
constexpr int kLongCf = 320, kLongCfNext = 257, kLongCfUnit = 258, kLongCfRed = 260;
constexpr int kLongCfClusters = 256;   // flag blocks per cluster size (2, 4, 8, 16)

template <int ATYPE, int GAP, bool CLUSTER = false>
__global__ void __launch_bounds__(kLongMaxWarps * 32) score_long_kernel(const LongParams prm) {
    constexpr int K = kLongK, W = kLongW;
    constexpr bool LOCAL = ATYPE == AT_LOCAL;
    constexpr bool SEMI = ATYPE == AT_SEMI;
    constexpr bool GLOBAL_EDGES = ATYPE == AT_GLOBAL;
    constexpr bool MERGED = GAP == GAP_MERGED;
    static_assert(GAP == GAP_LINEAR || GAP == GAP_MERGED, "the exact three-state model stays in score_kernel");

    __shared__ int s_prog[kLongMaxWarps + 1];       // border rows published per stage slot: generation * (m + 1) + rows
    __shared__ int s_next;                          // next stage of the current pair to hand out
    __shared__ int s_unit;
    __shared__ int s_red[kLongMaxWarps][3];
    __shared__ int4 s_in[kLongMaxWarps][64];        // two chunks of 32 rows of lane-0 inputs per warp: {T - gamma, H, selector}

    // A pair is spread over the GW = CS * NW warps of a thread-block cluster (CS = 1 for ordinary launches).  With
    // CS > 1 the progress counters and the stage counter live in global memory (release / acquire at gpu scope); the
    // border columns are global anyway.
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = CLUSTER ? (int)cluster.num_blocks() : 1;      // CLUSTER = false: compile-time 1, no cluster code at all
    const int crank = CLUSTER ? (int)cluster.block_rank() : 0;
    const int NW = blockDim.x >> 5;
    const int GW = CS * NW;
    const int w = threadIdx.x >> 5;
    const int t = threadIdx.x & 31;
    const int alpha = prm.alpha, beta = prm.beta, mism = prm.mismatch, one = prm.one;
    const int gamma = MERGED ? min(alpha, beta) : alpha;
    const int nalpha = -alpha, ngamma = -gamma;
    const unsigned mism4 = (unsigned)(mism & 0xff) * 0x01010101u;
    const int64_t cluster_id = blockIdx.x / CS;
    int2* const bnd_block = prm.bnd + cluster_id * (GW + 1) * prm.bnd_rows;
    // per cluster kLongCf ints: [0..256] progress (up to 16 blocks x 16 warps + 1), [257] next stage, [258] unit, [260..307] reduction
    int32_t* const cf = CS > 1 ? prm.cflags + cluster_id * kLongCf : nullptr;
    volatile int* prog = CS > 1 ? cf : s_prog;
    int* const next_stage = CS > 1 ? cf + kLongCfNext : &s_next;

    for (;;) {
        // previous pair fully retired (progress counters, reduction slots), next unit fetched by one thread
        if (CS > 1) {
            cluster.sync();
            if (crank == 0 && threadIdx.x == 0) cf[kLongCfUnit] = (int)atomicAdd(prm.queue, 1u);
            if (crank == 0 && threadIdx.x < kLongCfUnit) cf[threadIdx.x] = 0;
            __threadfence();
            cluster.sync();
            if (threadIdx.x == 0) s_unit = *(volatile int*)(cf + kLongCfUnit);
            __syncthreads();
        } else {
            __syncthreads();
            if (threadIdx.x == 0) s_unit = (int)atomicAdd(prm.queue, 1u);
            if (threadIdx.x <= kLongMaxWarps) s_prog[threadIdx.x] = 0;
            if (threadIdx.x == 0) s_next = 0;
            __syncthreads();
        }
        const int64_t u = s_unit;
        if (u >= (prm.n_units_dev ? (int64_t)*prm.n_units_dev : prm.n_units)) break;
        const int p = prm.units[u];
        const int qa = prm.pair_q[p], sb = prm.pair_s[p];
        const int m = prm.q_len[qa], n = prm.s_len[sb];
        const uint8_t* qp = prm.q_codes + prm.q_off[qa];
        const uint8_t* sp = prm.s_codes + prm.s_off[sb];
        const int nstages = (n + W - 1) / W;

        int best_v = GLOBAL_EDGES ? kNeg32 : 0, best_i = 0, best_j = SEMI ? n : 0;

        // Stages are handed out in order to whichever warp is free (atomic counter): the GW warps stay busy until the
        // pair runs out of stages, whatever the stage count.  Stage st writes border column st mod (GW + 1); when it is
        // handed out, stages <= st - GW have finished, so that column's previous reader is done.
#ifdef WSB_LONG_STATIC
        for (int st = crank * NW + w; st < nstages; st += GW) {
#else
        for (;;) {
            int st = 0;
            if (t == 0) st = atomicAdd(next_stage, 1);
            st = __shfl_sync(0xffffffffu, st, 0);
            if (st >= nstages) break;
#endif
            const bool first = st == 0, last = st + 1 == nstages;
            const int col0 = st * W + t * K;  // this strip holds matrix columns col0+1 .. col0+K
            unsigned prof[K];
            int TA[K], H[K], TG[MERGED ? K : 1];
#pragma unroll
            for (int c = 0; c < K; ++c) {
                unsigned pw = mism4;  // pad / flagged subject: never matches
                if (col0 + c < n) {
                    const int x = sp[col0 + c];
                    if (x < 4) pw = (mism4 & ~(0xffu << (8 * x))) | ((unsigned)(prm.match & 0xff) << (8 * x));
                }
                prof[c] = pw;
                const int h0 = edge_h(GLOBAL_EDGES, col0 + c + 1, alpha, beta);
                H[c] = h0; TA[c] = h0 - alpha;
                if (MERGED) TG[c] = h0 - gamma;
            }
            const int h_top = edge_h(GLOBAL_EDGES, col0, alpha, beta);  // H(0, col0): diagonal of this strip's row 1
            int hdiag = h_top;
            int tg_l = kNeg32, h_l = kNeg32;        // left border {T - gamma, H} of the row this lane computes next
            unsigned sel = 0u;                      // that row's query symbol, one-hot in bytes (0 = flagged)
            int edge = edge_h(GLOBAL_EDGES, 1, alpha, beta);   // stage 0: H(r, 0) of lane 0's current row
            // incoming border column (stage st - 1) and its producer
            const int2* in_col = bnd_block + (int64_t)((st + GW) % (GW + 1)) * prm.bnd_rows;   // (st - 1) mod (GW + 1)
            int2* out_ptr = bnd_block + (int64_t)(st % (GW + 1)) * prm.bnd_rows - 31;  // lane 31 at iteration it: row it - 31 -> slot it - 32 (it starts at 1)
            const int pw_id = (st + GW) % (GW + 1);                    // progress slot of stage st - 1
            const int p_base = st > 0 ? (st - 1) / (GW + 1) * (m + 1) : 0;   // its generation offset
            const int out_slot = st % (GW + 1);
            const int out_base = st / (GW + 1) * (m + 1);
            const bool do_out = t == 31 && !last;
            const int cap_rel = n - 1 - col0;  // register index of matrix column n, if inside this strip
            const bool has_cap = last && cap_rel >= 0 && cap_rel < K;

            // Rows 32c+1 .. 32c+32 of lane 0's inputs (incoming border + query selector) are fetched one chunk ahead
            // with coalesced loads, parked in shared memory, and read back one row per iteration.
            int2 pre = make_int2(kNeg32, kNeg32);
            unsigned pre_sel = 0u;
            auto fetch_chunk = [&](int chunk) {
                const int row0 = 32 * chunk;
                if (row0 >= m) return;
                const int q = qp[min(row0 + t, m - 1)];
                pre_sel = q < 4 ? 1u << (8 * q) : 0u;
                if (!first) {
                    const int need = p_base + min(m, row0 + 32);
                    while (prog[pw_id] < need) __nanosleep(40);
                    if (CS > 1) __threadfence(); else __threadfence_block();
                    pre = __ldcg(in_col + row0 + t);
                }
            };
            fetch_chunk(0);

            // one row of the strip; CHECK = the row may lie outside 1..m (ramp-up / ramp-down chunks)
            auto iteration = [&](int it, auto check_tag) {
                constexpr bool CHECK = decltype(check_tag)::value;
                const int4 in = s_in[w][(it - 1) & 63];   // lane 0's inputs for row it (broadcast load)
                if (t == 0) {
                    sel = (unsigned)in.z;
                    if (first) { h_l = edge; tg_l = edge - gamma; }
                    else { tg_l = in.x; h_l = in.y; }
                }
                if (first && GLOBAL_EDGES) edge -= beta;
                const int r = it - t;
                int out_tg = tg_l, out_h = h_l;
                if (!CHECK || (unsigned)(r - 1) < (unsigned)m) {
                    int hd = hdiag;
                    int la = MERGED ? tg_l + (gamma - alpha) : h_l - alpha;   // T_left - alpha
                    int lg = tg_l;
                    int rm = 0;
                    auto cells = [&](auto flagged_tag) {
                        constexpr bool FLAGGED = decltype(flagged_tag)::value;  // flagged query symbol: sigma = mismatch
#pragma unroll
                        for (int c = 0; c < K; ++c) {
                            const int d = FLAGGED ? fma_add(hd, one, mism) : __dp4a((int)prof[c], (int)sel, hd);
                            hd = H[c];
                            const int h = LOCAL ? __vimax3_s32_relu(TA[c], la, d) : __vimax3_s32(TA[c], la, d);
                            if (MERGED) {
                                const int tn = LOCAL ? __vimax3_s32_relu(TG[c], lg, d) : __vimax3_s32(TG[c], lg, d);
                                la = fma_add(tn, one, nalpha);
                                lg = fma_add(tn, one, ngamma);
                                TG[c] = lg;
                            } else {
                                la = fma_add(h, one, nalpha);
                            }
                            TA[c] = la;
                            H[c] = h;
                            if (LOCAL) {
                                if (c & 1) rm = __vimax3_s32(rm, H[c - 1], h);
                            }
                        }
                    };
                    if (sel != 0u) cells(std::false_type{});
                    else cells(std::true_type{});
                    out_tg = lg; out_h = H[K - 1];
                    if (LOCAL) {
                        if (rm >= best_v && rm > 0 && (rm > best_v || r < best_i)) {  // rare: a new record row
                            int pos = K - 1;
#pragma unroll
                            for (int c = K - 2; c >= 0; --c) if (H[c] == rm) pos = c;
                            best_v = rm; best_i = r; best_j = col0 + pos + 1;
                        }
                    }
                    if (SEMI && has_cap && r < m) {  // last matrix column, rows above the last one
                        const int hv = select_reg<int, K>(H, cap_rel);
                        if (better_cell(hv, r, n, best_v, best_i, best_j)) { best_v = hv; best_i = r; best_j = n; }
                    }
                    if (do_out) *out_ptr = make_int2(out_tg, out_h);
                }
                // right-most column and the row's selector move to the next lane
                hdiag = h_l;
                tg_l = __shfl_up_sync(0xffffffffu, out_tg, 1);
                h_l = __shfl_up_sync(0xffffffffu, out_h, 1);
                sel = __shfl_up_sync(0xffffffffu, sel, 1);
                if (CHECK && r == 0) hdiag = h_top;
                ++out_ptr;
            };

            const int it_end = m + 31;
            const int nchunks = (it_end + 31) / 32;
#pragma unroll 1
            for (int c = 0; c < nchunks; ++c) {
                s_in[w][(c & 1) * 32 + t] = make_int4(pre.x, pre.y, (int)pre_sel, 0);
                __syncwarp();
                fetch_chunk(c + 1);
                const int it0 = 32 * c + 1, it1 = min(it0 + 31, it_end);
                if (c >= 1 && it1 <= m) {   // every lane's row is inside the matrix
#pragma unroll 1
                    for (int it = it0; it <= it1; ++it) iteration(it, std::false_type{});
                } else {
#pragma unroll 1
                    for (int it = it0; it <= it1; ++it) iteration(it, std::true_type{});
                }
                if (do_out) {  // publish the border rows lane 31 has completed
                    if (CS > 1) __threadfence(); else __threadfence_block();
                    prog[out_slot] = out_base + min(max(it1 - 31, 0), m);
                }
            }
            // rows are complete: every lane's registers hold row m of its strip
            if (SEMI) {
#pragma unroll
                for (int c = 0; c < K; ++c)
                    if (col0 + c < n && better_cell(H[c], m, col0 + c + 1, best_v, best_i, best_j)) {
                        best_v = H[c]; best_i = m; best_j = col0 + c + 1;
                    }
            }
            if (GLOBAL_EDGES && has_cap) { best_v = select_reg<int, K>(H, cap_rel); best_i = m; best_j = n; }
            __syncwarp();
        }

        // reduce over lanes, then over warps: larger value, then smaller row, then smaller column
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const int ov = __shfl_xor_sync(0xffffffffu, best_v, off);
            const int oi = __shfl_xor_sync(0xffffffffu, best_i, off);
            const int oj = __shfl_xor_sync(0xffffffffu, best_j, off);
            if (better_cell(ov, oi, oj, best_v, best_i, best_j)) { best_v = ov; best_i = oi; best_j = oj; }
        }
        if (t == 0) { s_red[w][0] = best_v; s_red[w][1] = best_i; s_red[w][2] = best_j; }
        __syncthreads();
        if (threadIdx.x == 0) {
            int bv = s_red[0][0], bi = s_red[0][1], bj = s_red[0][2];
            for (int x = 1; x < NW; ++x)
                if (better_cell(s_red[x][0], s_red[x][1], s_red[x][2], bv, bi, bj)) {
                    bv = s_red[x][0]; bi = s_red[x][1]; bj = s_red[x][2];
                }
            if (CS > 1) { cf[kLongCfRed + 3 * crank] = bv; cf[kLongCfRed + 1 + 3 * crank] = bi; cf[kLongCfRed + 2 + 3 * crank] = bj; __threadfence(); }
            else {
                if (LOCAL && bv <= 0) { bv = 0; bi = 0; bj = 0; }
                prm.out_score[p] = bv; prm.out_i[p] = bi; prm.out_j[p] = bj;
            }
        }
        if (CS > 1) {
            cluster.sync();
            if (crank == 0 && threadIdx.x == 0) {
                volatile int* r = cf + kLongCfRed;
                int bv = r[0], bi = r[1], bj = r[2];
                for (int x = 1; x < CS; ++x)
                    if (better_cell(r[3 * x], r[3 * x + 1], r[3 * x + 2], bv, bi, bj)) { bv = r[3 * x]; bi = r[3 * x + 1]; bj = r[3 * x + 2]; }
                if (LOCAL && bv <= 0) { bv = 0; bi = 0; bj = 0; }
                prm.out_score[p] = bv; prm.out_i[p] = bi; prm.out_j[p] = bj;
            }
        }
    }
}

}  // namespace wsb
