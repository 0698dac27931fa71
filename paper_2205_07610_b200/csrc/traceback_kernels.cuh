// traceback_kernels.cuh -- direction-code fill + on-device walk + run-length CIGAR emission (sm_100a).
//
// Fill: the same lane-group wavefront as the score kernels (lane t owns K columns, row r = it - t), int32, exact
// three-state Gotoh (H, E, F kept apart because the walk must tell "came from E" from "came from F" and "gap extended"
// from "gap opened").  Every cell emits four bits, stored as bit planes of eight cells per 32-bit word:
//     byte 0  diagonal >= E            byte 1  max(diagonal, E) >= F      (origin of H: diagonal, E = vertical/I, F = horizontal/D)
//     byte 2  E(i,j) == E(i-1,j) - beta (the vertical gap arriving here is an extension)
//     byte 3  F(i,j) == F(i,j-1) - beta
// (local: H == 0 is stored as byte-1 bit clear + byte-0 bit set, a pattern the other modes read as plain "F").
// Priorities are the reference walk's: diagonal, then E, then F; extension before open (refdp.py:162-165, 196-220).
// Per cell: one IDP.4A (H_diag + sigma from a byte profile, as in score_long.cuh), four DPX max-with-predicate
// instructions (__vibmax_s32 -> VIMNMX + predicate: value and "which side won" in one issue slot), four predicated
// adds that set the plane bits, three adds (E - beta, F - beta, H - alpha).  Codes leave the SM in wavefront order -- the lane group writes P*K/2 contiguous bytes per iteration --
// so the only HBM traffic of the fill is 0.5 byte per cell of coalesced 8/16-byte stores.
//
// Walk: one thread per pair starts at the end cell the score kernels found (same tie-break) and follows the codes as
// the reference's state machine does (refdp.py:178-230), first counting runs, then -- after a prefix sum -- writing them
// in forward order as (length << 2 | op) words, op 0 = M, 1 = I, 2 = D.
#pragma once
#include "score_kernels.cuh"

#include <cuda_runtime.h>

#include <type_traits>

namespace wsb {

struct TbParams {
    const uint8_t* q_codes; const int64_t* q_off; const int32_t* q_len;
    const uint8_t* s_codes; const int64_t* s_off; const int32_t* s_len;
    const int32_t* pair_q; const int32_t* pair_s;
    int64_t first_pair;        // this launch covers pairs [first_pair, first_pair + n_pairs)
    int64_t n_pairs;
    const int64_t* code_off;   // per pair of the launch: offset of its code block, in 32-bit words
    uint32_t* codes;
    int32_t match, mismatch, alpha, beta;  // beta == alpha for the linear model
    int2* bnd;                 // stage border scratch: per lane group bnd_rows x {H, F - beta}
    int64_t bnd_rows;
    // walk
    const int32_t* end_i; const int32_t* end_j;   // end cells (score pass, or this fill for global / semiglobal)
    int32_t* w_score; int32_t* w_i; int32_t* w_j; // global / semiglobal: the fill writes score and end cell itself
    int32_t* start_i; int32_t* start_j;           // out: alignment start (0-based span starts)
    int32_t* n_runs;                              // per pair of the launch
    const int64_t* run_off;                       // exclusive prefix of n_runs, relative to the launch
    uint32_t* runs;                               // out (pass 2): runs of the launch, forward order
    int32_t tb_p, tb_k;                           // lane-group shape the codes were written with
    int32_t one;                                  // 1, opaque to the compiler (keeps plane-bit adds on the FMA pipe)
    uint32_t* run_tmp;                            // pass 1 parks up to kTbTmpRuns runs per pair here (reverse order), so
                                                  // that pass 2 is a copy for all but the most fragmented alignments
    int32_t lane_major = 0;                       // code layout (tb_code_index): 1 = written by the packed int16 fill
};

// Code block geometry shared by fill and walk.  A pair's block holds, per stage, one K/8-word entry per (iteration, lane);
// iteration it = i + t computes row i in lane t.  Two orders:
//   wavefront-major (int32 fill, bounded-memory tiles): entry (it, t) at (it - 1) * P + t -- what a lane group writes per
//     iteration is contiguous;
//   lane-major (packed int16 fill): entry (it, t) at t * rows4 + (it - 1), rows4 = iterations rounded up to a multiple of 4
//     -- four consecutive iterations of a lane share one 32-byte sector, so a walk that moves up or diagonally stays in a
//     sector for four steps instead of touching a new one every step (the walk's first pass was 15 % of cfg3, bound by one
//     DRAM sector per step); the fill collects four iterations per lane in shared memory and stores whole granules.
__host__ __device__ inline int tb_rows4(int m, int P) { return (m + P - 1 + 3) & ~3; }
__host__ __device__ inline int64_t tb_code_words(int m, int n, int P, int K) {
    const int W = P * K;
    const int stages = (n + W - 1) / W;
    return (int64_t)stages * tb_rows4(m, P) * P * (K / 8);
}

// max(a, b) with "a wins ties", and the plane bit added to w when a wins: compare, select, predicated add
// (the add is written as bit * one + w with one == 1 at run time, so that it issues on the FMA pipe as IMAD: compare
// and select already fill the ALU pipe)
__device__ __forceinline__ int max_mark(int a, int b, uint32_t& w, uint32_t bit, int one) {
    int r;
    asm("{\n\t.reg .pred p;\n\t"
        "setp.ge.s32 p, %2, %3;\n\t"
        "selp.s32 %0, %2, %3, p;\n\t"
        "@p mad.lo.u32 %1, %5, %4, %1;\n\t"
        "}" : "=r"(r), "+r"(w) : "r"(a), "r"(b), "r"(bit), "r"(one));
    return r;
}

// WIDE: substitution scores whose sum with alpha does not fit the signed-byte profile (|match + alpha| or |mismatch + alpha|
// > 127): the strip keeps the subject symbols instead of profile words and a cell takes compare + select + add instead of
// the one IDP.4A (three instructions for one; such schemes are rare, so only the (32, 16) shape is instantiated).
template <int P, int K, int ATYPE, bool AFFINE, bool WIDE = false>
__global__ void __launch_bounds__(kThreads) tb_fill_kernel(const TbParams prm) {
    constexpr int GPB = kThreads / P;
    constexpr int W = P * K;
    constexpr int NW = K / 8;  // 32-bit code words per lane and row
    constexpr bool LOCAL = ATYPE == AT_LOCAL;
    constexpr bool GLOBAL_EDGES = ATYPE == AT_GLOBAL;
    static_assert(K % 8 == 0, "K must pack into whole code words");

    const int tid = threadIdx.x;
    const int t = tid & (P - 1);
    const int gib = tid / P;
    const int64_t group_global = (int64_t)blockIdx.x * GPB + gib;
    const int64_t n_groups = (int64_t)gridDim.x * GPB;
    int2* bnd = prm.bnd ? prm.bnd + group_global * prm.bnd_rows : nullptr;
    const int alpha = prm.alpha, beta = prm.beta, mism = prm.mismatch, one = prm.one;
    // profile bytes hold sigma + alpha, so that the diagonal candidate comes straight from the stored H - alpha
    const unsigned miss4 = (unsigned)((mism + alpha) & 0xff) * 0x01010101u;
    const unsigned hit = (unsigned)((prm.match + alpha) & 0xff);
    const int hit_w = prm.match + alpha, miss_w = mism + alpha;   // WIDE: the same two values, unpacked

    const int64_t rounds = (prm.n_pairs + n_groups - 1) / n_groups;
    for (int64_t rd = 0; rd < rounds; ++rd) {
        const int64_t u = rd * n_groups + group_global;
        int m = 0, n = 0;
        const uint8_t* qp = nullptr;
        const uint8_t* sp = nullptr;
        uint32_t* code = nullptr;
        if (u < prm.n_pairs) {
            const int64_t p = prm.first_pair + u;
            const int a = prm.pair_q[p], b = prm.pair_s[p];
            if (prm.code_off[u] >= 0) {  // negative offset: pair rejected by the length check, nothing to fill
                m = prm.q_len[a]; n = prm.s_len[b];
                qp = prm.q_codes + prm.q_off[a];
                sp = prm.s_codes + prm.s_off[b];
                code = prm.codes + prm.code_off[u];
            }
        }
        const int mm_w = __reduce_max_sync(0xffffffffu, m);
        const int nn_w = __reduce_max_sync(0xffffffffu, n);
        if (mm_w == 0 || nn_w == 0) continue;
        const int nstages_w = (nn_w + W - 1) / W;
        const int nstages = (n + W - 1) / W;
        const int iters = m + P - 1;  // rows of this pair's code block per stage
        // global / semiglobal: score and end cell come out of this fill (same rule as the score kernels: larger value,
        // then smaller row, then smaller column); local alignments take them from the packed score pass
        int best_v = GLOBAL_EDGES ? kNeg32 : 0, best_i = 0, best_j = ATYPE == AT_SEMI ? n : 0;

        for (int st = 0; st < nstages_w; ++st) {
            const int col0 = st * W + t * K;
            // per column: profile word (sigma + alpha for query symbols 0..3), AL = H - alpha, EP = E - beta
            unsigned prof[K];
            int AL[K], EP[AFFINE ? K : 1];
#pragma unroll
            for (int c = 0; c < K; ++c) {
                unsigned pw = miss4;
                if (col0 + c < n) {
                    const int x = sp[col0 + c];
                    if (x < 4) pw = (miss4 & ~(0xffu << (8 * x))) | (hit << (8 * x));
                    if (WIDE) pw = x < 4 ? (unsigned)x : 4u;
                } else if (WIDE) pw = 4u;
                prof[c] = pw;
                AL[c] = edge_h(GLOBAL_EDGES, col0 + c + 1, alpha, beta) - alpha;
                if (AFFINE) EP[c] = kNeg32;
            }
            const int al_top = edge_h(GLOBAL_EDGES, col0, alpha, beta) - alpha;   // H(0, col0) - alpha
            int al_diag = al_top, all = kNeg32, fpl = kNeg32;  // left border {H - alpha, F - beta} of the current row
            int edge = edge_h(GLOBAL_EDGES, 1, alpha, beta);
            if (t == 0) {
                if (st == 0) { all = edge - alpha; fpl = kNeg32; }
                else if (m >= 1 && st < nstages) { const int2 b = bnd[1]; all = b.x; fpl = b.y; }
            }
            const int cap_rel = n - 1 - col0;   // register index of matrix column n, if inside this strip
            const bool has_cap = !LOCAL && st + 1 == nstages && cap_rel >= 0 && cap_rel < K;
            auto q_at = [&](int it) { return m > 0 ? (int)qp[min(max(it - t - 1, 0), m - 1)] : 4; };
            int q_cur = q_at(1), q_nxt = q_at(2);
            const int it_end = mm_w + P - 1;
            for (int it = 1; it <= it_end; ++it) {
                const int q_nn = q_at(it + 2);
                const int r = it - t;
                int out_al = all, out_fp = fpl;
                if (r >= 1 && r <= m && st < nstages) {
                    const unsigned qsel = q_cur < 4 ? 1u << (8 * q_cur) : 0u;   // one-hot bytes; 0 = flagged
                    int ad = al_diag, fl = fpl, al = all;
                    uint32_t words[NW];
                    auto cells = [&](auto flagged_tag) {
                        constexpr bool FLAGGED = decltype(flagged_tag)::value;
#pragma unroll
                        for (int w8 = 0; w8 < NW; ++w8) {
                            // bit planes of eight cells: byte 0 "diagonal >= E", byte 1 "max(diagonal, E) >= F",
                            // byte 2 "E extends", byte 3 "F extends" (ties: diagonal, then E, then F; extension first)
                            uint32_t wd = 0u, wm = 0u, we = 0u, wf = 0u;
#pragma unroll
                            for (int c8 = 0; c8 < 8; ++c8) {
                                const int c = w8 * 8 + c8;
                                const int d = FLAGGED ? ad + (mism + alpha)
                                              : WIDE  ? ad + ((int)prof[c] == q_cur ? hit_w : miss_w)
                                                      : __dp4a((int)prof[c], (int)qsel, ad);
                                ad = AL[c];
                                int h;
                                if (LOCAL) {
                                    bool xe = false, xf = false, pd, pm;
                                    int e, f;
                                    if (AFFINE) {
                                        e = __vibmax_s32(EP[c], AL[c], &xe);
                                        f = __vibmax_s32(fl, al, &xf);
                                    } else {
                                        e = AL[c]; f = al;
                                    }
                                    const int m1 = __vibmax_s32(d, e, &pd);
                                    h = __vibmax_s32(m1, f, &pm);
                                    // H == 0 stops the walk: encoded as "F wins" with the diagonal bit set
                                    const bool stop = h <= 0;
                                    h = max(h, 0);
                                    pd = (pd && pm) || stop;
                                    pm = pm && !stop;
                                    if (pd) wd += 1u << c8;
                                    if (pm) wm += 1u << (8 + c8);
                                    if (AFFINE) {
                                        if (xe) we += 1u << (16 + c8);
                                        if (xf) wf += 1u << (24 + c8);
                                        EP[c] = e - beta; fl = f - beta;
                                    }
                                } else {
                                    int e, f;
                                    if (AFFINE) {
                                        e = max_mark(EP[c], AL[c], we, 1u << (16 + c8), one);
                                        f = max_mark(fl, al, wf, 1u << (24 + c8), one);
                                        EP[c] = e - beta; fl = f - beta;
                                    } else {
                                        e = AL[c]; f = al;
                                    }
                                    const int m1 = max_mark(d, e, wd, 1u << c8, one);
                                    h = max_mark(m1, f, wm, 1u << (8 + c8), one);
                                }
                                al = h - alpha;
                                AL[c] = al;
                            }
                            words[w8] = (wd | wm) | (we | wf);
                        }
                    };
                    if (qsel != 0u) cells(std::false_type{});
                    else cells(std::true_type{});
                    // wavefront-major: iteration it of stage st, lane t
                    uint32_t* dst = code + (((int64_t)st * iters + (it - 1)) * P + t) * NW;
                    if (NW == 2) *reinterpret_cast<uint2*>(dst) = make_uint2(words[0], words[1]);
                    else if (NW == 4) *reinterpret_cast<uint4*>(dst) = make_uint4(words[0], words[1], words[2], words[NW - 1]);
                    else {
#pragma unroll
                        for (int w8 = 0; w8 < NW; ++w8) dst[w8] = words[w8];
                    }
                    out_al = al;
                    out_fp = AFFINE ? fl : kNeg32;
                    if (ATYPE == AT_SEMI && has_cap && r < m) {   // last matrix column, rows above the last one
                        const int hv = select_reg<int, K>(AL, cap_rel) + alpha;
                        if (better_cell(hv, r, n, best_v, best_i, best_j)) { best_v = hv; best_i = r; best_j = n; }
                    }
                    if (t == P - 1 && st + 1 < nstages) bnd[r] = make_int2(out_al, out_fp);
                }
                int nal = __shfl_up_sync(0xffffffffu, out_al, 1, P);
                int nfp = __shfl_up_sync(0xffffffffu, out_fp, 1, P);
                al_diag = all;
                if (t == 0) {
                    if (st == 0) {
                        if (GLOBAL_EDGES) edge -= beta;
                        nal = edge - alpha; nfp = kNeg32;
                    } else if (r + 1 <= m && st < nstages) {
                        const int2 b = bnd[r + 1];
                        nal = b.x; nfp = b.y;
                    }
                }
                all = nal; fpl = nfp;
                if (r == 0) al_diag = al_top;
                q_cur = q_nxt; q_nxt = q_nn;
            }
            // every lane's registers now hold row m of its strip
            if (ATYPE == AT_SEMI && st < nstages) {
#pragma unroll
                for (int c = 0; c < K; ++c)
                    if (col0 + c < n && better_cell(AL[c] + alpha, m, col0 + c + 1, best_v, best_i, best_j)) {
                        best_v = AL[c] + alpha; best_i = m; best_j = col0 + c + 1;
                    }
            }
            if (GLOBAL_EDGES && has_cap) { best_v = select_reg<int, K>(AL, cap_rel) + alpha; best_i = m; best_j = n; }
            __syncwarp();
        }
        if (!LOCAL) {
            const unsigned gmask = group_mask<P>(tid & 31);
#pragma unroll
            for (int off = P / 2; off >= 1; off >>= 1) {
                const int ov = __shfl_xor_sync(gmask, best_v, off, P);
                const int oi = __shfl_xor_sync(gmask, best_i, off, P);
                const int oj = __shfl_xor_sync(gmask, best_j, off, P);
                if (better_cell(ov, oi, oj, best_v, best_i, best_j)) { best_v = ov; best_i = oi; best_j = oj; }
            }
            if (t == 0 && m > 0 && n > 0) {
                const int64_t p = prm.first_pair + u;
                prm.w_score[p] = best_v; prm.w_i[p] = best_i; prm.w_j[p] = best_j;
            }
        }
    }
}

// code of cell (i, j), 1 <= i <= m, 1 <= j <= n, translated from the fill's bit planes to
//   bits 1:0 origin of H (0 stop, 1 diagonal, 2 E, 3 F), bit 2 "E extends", bit 3 "F extends"
template <bool LOCAL>
__device__ __forceinline__ uint32_t tb_code_at(const uint32_t* code, int i, int j, int m, int P, int K, bool lane_major = false) {
    const int W = P * K;
    const int st = (j - 1) / W;
    const int col = (j - 1) - st * W;
    const int t = col / K, c = col - t * K;
    const int it = i + t;
    const int64_t entry = lane_major ? ((int64_t)st * P + t) * tb_rows4(m, P) + (it - 1)
                                     : ((int64_t)st * (m + P - 1) + (it - 1)) * P + t;
    const int64_t word = entry * (K / 8) + c / 8;
    const uint32_t bits = __ldcg(code + word) >> (c % 8);   // L2 only: random 4-byte reads
    const bool pd = bits & 1u, pm = bits & 0x100u;
    const uint32_t origin = pm ? (pd ? 1u : 2u) : ((LOCAL && pd) ? 0u : 3u);   // local: "F wins" + diagonal bit = stop
    return origin | ((bits >> 14) & 4u) | ((bits >> 21) & 8u);
}

constexpr int kTbTmpRuns = 128;   // unrelated 250 bp reads average 77 runs, 99th percentile 99

// Position of the walk inside a pair's code block, kept incrementally: a step changes the row by one and / or the column by
// one, so the lane (t), the column inside the lane's strip (c) and the stage are carried along instead of being re-derived
// from (i, j) with two integer divisions by run-time lane-group shapes per step.
template <bool LOCAL>
struct TbCursor {
    const uint32_t* code;
    int P, K, NW, m, rows4, st, t, c;
    bool lane_major;
    __device__ __forceinline__ void init(const uint32_t* code_, int m_, int P_, int K_, bool lane_major_, int j) {
        code = code_; m = m_; P = P_; K = K_; NW = K_ / 8; lane_major = lane_major_; rows4 = tb_rows4(m_, P_);
        const int W = P * K;
        st = (j - 1) / W;
        const int col = (j - 1) - st * W;
        t = col / K; c = col - t * K;
    }
    __device__ __forceinline__ void left() {   // j -> j - 1
        if (--c < 0) { c = K - 1; if (--t < 0) { t = P - 1; --st; } }
    }
    __device__ __forceinline__ uint32_t at(int i) const {   // code of cell (i, current column), as tb_code_at returns it
        const int it = i + t;
        const int64_t entry = lane_major ? ((int64_t)st * P + t) * rows4 + (it - 1) : ((int64_t)st * (m + P - 1) + (it - 1)) * P + t;
        // read-only path through L1: with the lane-major layout the next three steps up or diagonal hit the sector this load
        // brings in (the codes were written by an earlier kernel, so the non-coherent path is safe)
        const uint32_t bits = (lane_major ? __ldg(code + entry * NW + (c >> 3)) : __ldcg(code + entry * NW + (c >> 3))) >> (c & 7);
        const bool pd = bits & 1u, pm = bits & 0x100u;
        const uint32_t origin = pm ? (pd ? 1u : 2u) : ((LOCAL && pd) ? 0u : 3u);
        return origin | ((bits >> 14) & 4u) | ((bits >> 21) & 8u);
    }
};

// PASS 1 counts the runs, records the start cell and parks the first kTbTmpRuns runs (in walk order); PASS 2 writes the
// runs in forward order: a reversed copy of the parked runs, or a second walk for alignments with more runs than that.
template <int ATYPE, int PASS>
__device__ __forceinline__ void tb_walk_pair(const TbParams& prm, int64_t u, int64_t p, int m, int n, const uint32_t* code,
                                             int i, int j) {
    uint32_t* out = nullptr;
    int64_t w = 0;
    if (PASS == 2) { out = prm.runs + prm.run_off[u]; w = prm.n_runs[u]; }
    uint32_t* tmp = prm.run_tmp ? prm.run_tmp + u * kTbTmpRuns : nullptr;
    if (PASS == 2 && tmp && w <= kTbTmpRuns) {   // the walk of pass 1 already produced every run
        for (int k = 0; k < (int)w; ++k) out[k] = tmp[w - 1 - k];
        return;
    }
    int count = 0;
    int cur_op = -1, cur_len = 0;
    auto flush = [&]() {
        const uint32_t word = ((uint32_t)cur_len << 2) | (uint32_t)cur_op;
        if (PASS == 1 && tmp && count < kTbTmpRuns) tmp[count] = word;
        ++count;
        if (PASS == 2) out[--w] = word;
    };
    auto emit = [&](int op, int len) {
        if (len <= 0) return;
        if (op == cur_op) { cur_len += len; return; }
        if (cur_op >= 0) flush();
        cur_op = op; cur_len = len;
    };
    int state = 0;  // 0: at H, 1: inside a vertical run (E), 2: inside a horizontal run (F)
    if (m > 0 && n > 0) {
        TbCursor<ATYPE == AT_LOCAL> cur;
        cur.init(code, m, prm.tb_p, prm.tb_k, prm.lane_major != 0, max(j, 1));
        for (;;) {
            if (state == 0) {
                if (i == 0 && j == 0) break;
                if (ATYPE == AT_GLOBAL) {
                    if (i == 0) { emit(2, j); j = 0; break; }
                    if (j == 0) { emit(1, i); i = 0; break; }
                } else if (i == 0 || j == 0) break;  // local: H == 0 on the edges; semiglobal: free edges
                const uint32_t cd = cur.at(i);
                const uint32_t origin = cd & 3u;
                if (origin == 0u) break;                        // local stop: H(i, j) == 0
                if (origin == 1u) { emit(0, 1); --i; --j; cur.left(); continue; }
                state = origin == 2u ? 1 : 2;
                continue;
            }
            const uint32_t cd = cur.at(i);
            if (state == 1) { emit(1, 1); const bool ext = cd & 4u; --i; if (!ext) state = 0; }
            else { emit(2, 1); const bool ext = cd & 8u; --j; cur.left(); if (!ext) state = 0; }
        }
    } else if (ATYPE == AT_GLOBAL) {  // an empty side: one gap run (ref_traceback walks the edge)
        if (i == 0 && j > 0) { emit(2, j); j = 0; }
        else if (j == 0 && i > 0) { emit(1, i); i = 0; }
    }
    if (cur_op >= 0) flush();
    if (PASS == 1) {
        prm.n_runs[u] = count;
        prm.start_i[p] = i;
        prm.start_j[p] = j;
    }
}

template <int ATYPE, int PASS>
__global__ void tb_walk_kernel(const TbParams prm) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= prm.n_pairs) return;
    const int64_t p = prm.first_pair + u;
    const int m = prm.q_len[prm.pair_q[p]], n = prm.s_len[prm.pair_s[p]];
    if (prm.code_off[u] < 0) {  // rejected pair: no alignment
        if (PASS == 1) { prm.n_runs[u] = 0; prm.start_i[p] = 0; prm.start_j[p] = 0; }
        return;
    }
    tb_walk_pair<ATYPE, PASS>(prm, u, p, m, n, prm.codes + prm.code_off[u], prm.end_i[p], prm.end_j[p]);
}

__global__ void add_base_kernel(const int64_t* chunk_off, int64_t base, int64_t count, int64_t* out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < count) out[k] = chunk_off[k] + base;
}

// host-side state of the traceback path kept with a batch
struct TracebackState {
    int32_t *d_qs = nullptr, *d_ss = nullptr;  // alignment starts per pair
    int64_t* d_run_off = nullptr;              // n_pairs + 1, global exclusive prefix of run counts
    uint32_t* d_runs = nullptr;
    int64_t runs_cap = 0, total_runs = 0;
    bool valid = false;
    void release() {
        if (d_qs) cudaFree(d_qs);
        if (d_ss) cudaFree(d_ss);
        if (d_run_off) cudaFree(d_run_off);
        if (d_runs) cudaFree(d_runs);
        d_qs = d_ss = nullptr; d_run_off = nullptr; d_runs = nullptr; runs_cap = total_runs = 0; valid = false;
    }
};

}  // namespace wsb
