// score_long16.cuh -- packed int16x2 (DPX) variant of the long-read kernel: TWO pairs of identical shape per block.
//
// Same stage pipeline as score_long.cuh (512-column stages handed out in order to the warps of a block, borders streamed
// through an L2-resident scratch column, lane 0 fed from shared memory), but every register carries two alignments in
// its 16-bit halves, as the reference's packed mode does (stage_*16, _kernels.py:553-858: int16 halves).  The
// substitution scores of both alignments come from one byte permute: a row's two query symbols are "row words"
// (sigma(q, s) for s = 0..3 in the four bytes; a flagged query symbol is mismatch in all four), each column keeps a
// 16-bit PRMT selector built from its two subject symbols.  Per packed cell (two cells):
//     sigma = PRMT(rowA, rowB, sel[c])  ALU        d  = H_diag + sigma                 VIADD.16x2   FMA pipe
//     h  = max3(TA_up, TA_left, d[,0])  VIMNMX3.S16x2[.RELU]   tn = max3(TG_up, TG_left, d[,0])   VIMNMX3.S16x2[.RELU]
//     TA = tn - alpha ; TG = tn - gamma  2 x VIADD.16x2
// = 6 instructions per two cells, against 5 per cell in int32.
//
// Conditions (planner): both pairs of a unit have the same (m, n); every DP value fits 16 bits (scores rise by at most
// match per diagonal step and never fall below the all-gap path: match * min(m, n) and 3 alpha + beta (m + n) + |mismatch|
// both <= 32000, e.g. 10 kbp x 10 kbp global at 2/-1/2/1); |match|, |mismatch| <= 127; merged-exact or linear scheme; local: pads
// non-improving.  A flagged SUBJECT symbol has no selector encoding: the unit's pairs are listed in LongParams::redo and
// re-scored by the int32 long-read kernel right after this launch (its unit count is read from device memory).
#pragma once
#include "score_long.cuh"
#include "score_short16.cuh"

namespace wsb {

// AIMM / GIMM > 0: gap costs alpha / gamma as immediates (the host picks such an instantiation when the scheme matches):
// at ptxas -O1 the packed constants are otherwise re-materialised from the kernel parameters in every row.
template <int ATYPE, int GAP, int AIMM = 0, int GIMM = 0>
__global__ void __launch_bounds__(kLongMaxWarps * 32) score_long16_kernel(const LongParams prm) {
    constexpr int K = kLongK, W = kLongW;
    constexpr bool LOCAL = ATYPE == AT_LOCAL;
    constexpr bool SEMI = ATYPE == AT_SEMI;
    constexpr bool GLOBAL_EDGES = ATYPE == AT_GLOBAL;
    constexpr bool MERGED = GAP == GAP_MERGED;

    __shared__ int s_prog[kLongMaxWarps + 1];
    __shared__ int s_next;
    __shared__ int s_unit;
    __shared__ int s_red[kLongMaxWarps][6];
    __shared__ int4 s_in[kLongMaxWarps][64];        // lane-0 inputs per row: {T - gamma, H, row word A, row word B}

    const int NW = blockDim.x >> 5;
    const int w = threadIdx.x >> 5;
    const int t = threadIdx.x & 31;
    const int alpha = AIMM > 0 ? AIMM : prm.alpha, beta = prm.beta;
    const int gamma = GIMM > 0 ? GIMM : (MERGED ? min(prm.alpha, beta) : prm.alpha);
    const unsigned c_nalpha = AIMM > 0 ? ((unsigned)(-AIMM) & 0xffffu) * 0x10001u : pack16(-alpha);
    const unsigned c_ngamma = GIMM > 0 ? ((unsigned)(-GIMM) & 0xffffu) * 0x10001u : pack16(-gamma);
    const unsigned c_gma = (AIMM > 0 && GIMM > 0) ? ((unsigned)(GIMM - AIMM) & 0xffffu) * 0x10001u : pack16(gamma - alpha);
    const unsigned c_nbeta = pack16(-beta);
    const unsigned s_in_base = (unsigned)__cvta_generic_to_shared(&s_in[threadIdx.x >> 5][0]);
    const unsigned mism4 = (unsigned)(prm.mismatch & 0xff) * 0x01010101u;
    const unsigned match1 = (unsigned)(prm.match & 0xff);
    int2* const bnd_block = prm.bnd + (int64_t)blockIdx.x * (NW + 1) * prm.bnd_rows;
    volatile int* prog = s_prog;

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_unit = (int)atomicAdd(prm.queue, 1u);
        if (threadIdx.x <= kLongMaxWarps) s_prog[threadIdx.x] = 0;
        if (threadIdx.x == 0) s_next = 0;
        __syncthreads();
        const int64_t u = s_unit;
        if (u >= prm.n_units) break;
        int pidx[2] = {prm.units[2 * u], prm.units[2 * u + 1]};
        const bool single = pidx[1] < 0;         // odd tail: the second half shadows the first and is not written
        if (single) pidx[1] = pidx[0];
        const uint8_t* qp[2];
        const uint8_t* sp[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            qp[v] = prm.q_codes + prm.q_off[prm.pair_q[pidx[v]]];
            sp[v] = prm.s_codes + prm.s_off[prm.pair_s[pidx[v]]];
        }
        // global / semiglobal: both pairs have the same shape (planner); local: shapes may differ, the unit runs
        // max(m) x max(n) and the shorter alignment sees never-improving pad rows / columns beyond its own matrix
        int mv[2], nv[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) { mv[v] = prm.q_len[prm.pair_q[pidx[v]]]; nv[v] = prm.s_len[prm.pair_s[pidx[v]]]; }
        const int m = max(mv[0], mv[1]), n = max(nv[0], nv[1]);
        const int nstages = (n + W - 1) / W;

        int best_v[2], best_i[2], best_j[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) { best_v[v] = GLOBAL_EDGES ? kNeg32 : 0; best_i[v] = 0; best_j[v] = SEMI ? n : 0; }
        bool flagged_subject = false;

        for (;;) {
            int st = 0;
            if (t == 0) st = atomicAdd(&s_next, 1);
            st = __shfl_sync(0xffffffffu, st, 0);
            if (st >= nstages) break;
            const bool first = st == 0, last = st + 1 == nstages;
            const int col0 = st * W + t * K;
            unsigned sel[K], TA[K], H[K], TG[MERGED ? K : 1];
#pragma unroll
            for (int c = 0; c < K; ++c) {
                unsigned nib[2] = {0x88u, 0x88u};   // pad column: sign fill -> sigma in {0, -1}, never improving
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (col0 + c < nv[v]) {
                        const unsigned x = sp[v][col0 + c];
                        if (x < 4) nib[v] = (x + 4u * v) | ((x + 4u * v) | 8u) << 4;
                        else flagged_subject = true;
                    }
                sel[c] = nib[0] | (nib[1] << 8);
                const int h0 = edge_h(GLOBAL_EDGES, col0 + c + 1, alpha, beta);
                H[c] = pack16(h0); TA[c] = pack16(h0 - alpha);
                if (MERGED) TG[c] = pack16(h0 - gamma);
            }
            const unsigned h_top = pack16(edge_h(GLOBAL_EDGES, col0, alpha, beta));
            unsigned hdiag = h_top;
            unsigned tg_l = 0u, h_l = 0u, rwA = mism4, rwB = mism4;   // left border and row words of the lane's next row
            // stage 0: packed {H, T - gamma} of the matrix' left border at lane 0's current row
            unsigned edge_h16 = pack16(edge_h(GLOBAL_EDGES, 1, alpha, beta));
            unsigned edge_tg16 = pack16(edge_h(GLOBAL_EDGES, 1, alpha, beta) - gamma);
            const int2* in_col = bnd_block + (int64_t)((st + NW) % (NW + 1)) * prm.bnd_rows;
            int2* out_ptr = bnd_block + (int64_t)(st % (NW + 1)) * prm.bnd_rows - 31;
            const int pw_id = (st + NW) % (NW + 1);
            const int p_base = st > 0 ? (st - 1) / (NW + 1) * (m + 1) : 0;
            const int out_slot = st % (NW + 1);
            const int out_base = st / (NW + 1) * (m + 1);
            const bool do_out = t == 31 && !last;
            const int cap_rel = n - 1 - col0;
            const bool has_cap = last && cap_rel >= 0 && cap_rel < K;

            int2 pre = make_int2(0, 0);
            unsigned pre_a = mism4, pre_b = mism4;
            auto row_word = [&](int q) { return q < 4 ? (mism4 & ~(0xffu << (8 * q))) | (match1 << (8 * q)) : mism4; };
            auto fetch_chunk = [&](int chunk) {
                const int row0 = 32 * chunk;
                if (row0 >= m) return;
                const int idx = row0 + t;   // rows beyond an alignment's own query are pads: mismatch against everything
                pre_a = idx < mv[0] ? row_word(qp[0][idx]) : mism4;
                pre_b = idx < mv[1] ? row_word(qp[1][idx]) : mism4;
                if (!first) {
                    const int need = p_base + min(m, row0 + 32);
                    while (prog[pw_id] < need) __nanosleep(40);
                    __threadfence_block();
                    pre = __ldcg(in_col + row0 + t);
                }
            };
            fetch_chunk(0);

            auto iteration = [&](int it, auto check_tag) {
                constexpr bool CHECK = decltype(check_tag)::value;
                int4 in;   // lane 0's inputs for this row (broadcast load from a precomputed shared-memory address)
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(in.x), "=r"(in.y), "=r"(in.z), "=r"(in.w)
                             : "r"(s_in_base + 16u * (unsigned)((it - 1) & 63)) : "memory");
                if (t == 0) {
                    rwA = (unsigned)in.z; rwB = (unsigned)in.w;
                    if (first) { h_l = edge_h16; tg_l = edge_tg16; }
                    else { tg_l = (unsigned)in.x; h_l = (unsigned)in.y; }
                }
                if (first && GLOBAL_EDGES) { edge_h16 = __vadd2(edge_h16, c_nbeta); edge_tg16 = __vadd2(edge_tg16, c_nbeta); }
                const int r = it - t;
                unsigned out_tg = tg_l, out_h = h_l;
                if (!CHECK || (unsigned)(r - 1) < (unsigned)m) {
                    unsigned la = MERGED ? __vadd2(tg_l, c_gma) : __vadd2(h_l, c_nalpha);
                    unsigned lg = tg_l;
                    unsigned rm = 0u, hprev = 0u;
                    // the diagonal candidate runs one column ahead of the cell: it reads H(r - 1, c) BEFORE the cell of column c
                    // overwrites that register with H(r, c), so H[] is updated in place (no register rotation at the loop end)
                    unsigned dn;
                    {
                        unsigned sg;
                        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(sg) : "r"(rwA), "r"(rwB), "r"(sel[0]));
                        dn = __vadd2(hdiag, sg);
                    }
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        const unsigned d = dn;
                        if (c + 1 < K) {
                            unsigned sg;
                            asm("prmt.b32 %0, %1, %2, %3;" : "=r"(sg) : "r"(rwA), "r"(rwB), "r"(sel[c + 1]));
                            dn = __vadd2(H[c], sg);
                        }
                        const unsigned h = LOCAL ? __vimax3_s16x2_relu(TA[c], la, d) : __vimax3_s16x2(TA[c], la, d);
                        if (MERGED) {
                            const unsigned tn = LOCAL ? __vimax3_s16x2_relu(TG[c], lg, d) : __vimax3_s16x2(TG[c], lg, d);
                            la = __vadd2(tn, c_nalpha);
                            lg = __vadd2(tn, c_ngamma);
                            TG[c] = lg;
                        } else {
                            la = __vadd2(h, c_nalpha);
                        }
                        TA[c] = la;
                        H[c] = h;
                        if (LOCAL) {
                            if (c & 1) rm = __vimax3_s16x2(rm, hprev, h);
                            hprev = h;
                        }
                    }
                    out_tg = lg; out_h = H[K - 1];
                    if (LOCAL) {
#pragma unroll
                        for (int v = 0; v < 2; ++v) {
                            const int rv = half16(rm, v);
                            if (rv >= best_v[v] && rv > 0 && (rv > best_v[v] || r < best_i[v])) {  // rare: a new record row
                                int pos = K - 1;
#pragma unroll
                                for (int c = K - 2; c >= 0; --c) if (half16(H[c], v) == rv) pos = c;
                                best_v[v] = rv; best_i[v] = r; best_j[v] = col0 + pos + 1;
                            }
                        }
                    }
                    if (SEMI && has_cap && r < m) {
                        const unsigned hw = select_reg<unsigned, K>(H, cap_rel);
#pragma unroll
                        for (int v = 0; v < 2; ++v) {
                            const int hv = half16(hw, v);
                            if (better_cell(hv, r, n, best_v[v], best_i[v], best_j[v])) { best_v[v] = hv; best_i[v] = r; best_j[v] = n; }
                        }
                    }
                    if (do_out) *out_ptr = make_int2((int)out_tg, (int)out_h);
                }
                hdiag = h_l;
                tg_l = __shfl_up_sync(0xffffffffu, out_tg, 1);
                h_l = __shfl_up_sync(0xffffffffu, out_h, 1);
                rwA = __shfl_up_sync(0xffffffffu, rwA, 1);
                rwB = __shfl_up_sync(0xffffffffu, rwB, 1);
                if (CHECK && r == 0) hdiag = h_top;
                ++out_ptr;
            };

            const int it_end = m + 31;
            const int nchunks = (it_end + 31) / 32;
#pragma unroll 1
            for (int c = 0; c < nchunks; ++c) {
                s_in[w][(c & 1) * 32 + t] = make_int4(pre.x, pre.y, (int)pre_a, (int)pre_b);
                __syncwarp();
                fetch_chunk(c + 1);
                const int it0 = 32 * c + 1, it1 = min(it0 + 31, it_end);
                if (c >= 1 && it1 <= m) {
#pragma unroll 1
                    for (int it = it0; it <= it1; ++it) iteration(it, std::false_type{});
                } else {
#pragma unroll 1
                    for (int it = it0; it <= it1; ++it) iteration(it, std::true_type{});
                }
                if (do_out) {
                    __threadfence_block();
                    prog[out_slot] = out_base + min(max(it1 - 31, 0), m);
                }
            }
            // rows are complete: every lane's registers hold row m of its strip
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                if (SEMI) {
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        const int hv = half16(H[c], v);
                        if (col0 + c < n && better_cell(hv, m, col0 + c + 1, best_v[v], best_i[v], best_j[v])) {
                            best_v[v] = hv; best_i[v] = m; best_j[v] = col0 + c + 1;
                        }
                    }
                }
                if (GLOBAL_EDGES && has_cap) { best_v[v] = half16(select_reg<unsigned, K>(H, cap_rel), v); best_i[v] = m; best_j[v] = n; }
            }
            __syncwarp();
        }

        // a flagged subject symbol cannot be encoded: the pairs of this unit go to the int32 kernel
        const bool any_flag = __syncthreads_or(flagged_subject ? 1 : 0) != 0;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                const int ov = __shfl_xor_sync(0xffffffffu, best_v[v], off);
                const int oi = __shfl_xor_sync(0xffffffffu, best_i[v], off);
                const int oj = __shfl_xor_sync(0xffffffffu, best_j[v], off);
                if (better_cell(ov, oi, oj, best_v[v], best_i[v], best_j[v])) { best_v[v] = ov; best_i[v] = oi; best_j[v] = oj; }
            }
            if (t == 0) { s_red[w][3 * v] = best_v[v]; s_red[w][3 * v + 1] = best_i[v]; s_red[w][3 * v + 2] = best_j[v]; }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int v = 0; v < (single ? 1 : 2); ++v) {
                if (any_flag) { const int at = atomicAdd(prm.redo_count, 1); prm.redo[at] = pidx[v]; continue; }
                int bv = s_red[0][3 * v], bi = s_red[0][3 * v + 1], bj = s_red[0][3 * v + 2];
                for (int x = 1; x < NW; ++x)
                    if (better_cell(s_red[x][3 * v], s_red[x][3 * v + 1], s_red[x][3 * v + 2], bv, bi, bj)) {
                        bv = s_red[x][3 * v]; bi = s_red[x][3 * v + 1]; bj = s_red[x][3 * v + 2];
                    }
                if (LOCAL && bv <= 0) { bv = 0; bi = 0; bj = 0; }
                prm.out_score[pidx[v]] = bv; prm.out_i[pidx[v]] = bi; prm.out_j[pidx[v]] = bj;
            }
        }
    }
}

}  // namespace wsb
