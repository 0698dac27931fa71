// score_short16g.cuh -- packed int16x2 (DPX) GLOBAL scoring of short reads that fit one stage (cfg1's shape).
//
// The lane-group wavefront, in-place strip state and unit pipeline of score_short16.cuh (one row per trip, D[c] = diagonal
// candidate of the next row, TA = T - alpha, TG = T - gamma, substitution scores from one PRMT of the row words), minus
// everything local alignment needs (zero floor, row maximum, row snapshots) and plus what the Needleman-Wunsch edges need:
//   * matrix edges H(0, j) = H(i, 0) = -(alpha + beta (k - 1)) (refdp.py:53-58): the strip starts from the row-0 values,
//     lane 0's left border walks down by beta per row (one packed add per trip; the hand-over multiply becomes a
//     multiply-add: IMAD, same instruction count as the local kernel's);
//   * no fixed point above row 1: a lane is MASKED until its first row (the P - 1 ramp trips run as a separate copy of
//     the loop body under a branch); rows below m are junk that nobody reads, because
//   * the score H(m, n) is taken when it is produced: the trips in which some lane finishes row m (the last P trips of
//     a uniform batch, every trip of a ragged one) park that row's H values in shared memory, and the lane that owns
//     column n reads its word afterwards.
// Cell (merged affine, _kernels.py:259-276): PRMT, VIADD, 2 x VIMNMX3.S16x2, 2 x VIADD = 3 ALU + 3 FMA-pipe instructions
// per two cells; linear gaps (_kernels.py:113-126): PRMT, VIADD, VIMNMX3, VIADD = 2 + 2.
// Limits (planner): |match|, |mismatch| <= 127, merged-exact scheme, values within 16 bits, no flagged SUBJECT symbol
// (such pairs are listed in ScoreParams::redo and re-scored by the int32 kernel in the same call).
#pragma once
#include "score_short16.cuh"

namespace wsb {

template <int P, int K> constexpr size_t short16g_smem_bytes() {
    return (size_t)2 * (K / 4 + 1) * (kThreads / P) * 16    // row m of both halves: the strip of the lane that owns column n
           + (size_t)(kThreads / P) * short16_qrows<P>() * 8
           + (size_t)(kThreads / P) * 4 * kShort16Raw
           + (size_t)(kThreads / P) * 16 * 4;
}


// One row of a strip (global, no floor).  CAP: also hand the row's H values out (the row-m capture).
template <int K, int NW, bool MERGED, bool CAP>
__device__ __forceinline__ void g16_row(const unsigned (&sel)[K], unsigned (&TA)[K], unsigned (&TG)[MERGED ? K : 1], unsigned (&D)[K],
                                        unsigned c_nalpha, unsigned c_ngamma, unsigned rw0, unsigned rw1, unsigned nw0, unsigned nw1,
                                        unsigned h_diag, unsigned& la, unsigned& lg, unsigned& h_last, unsigned& t_last,
                                        unsigned (&hrow)[NW]) {
    unsigned hprev = 0u;
#pragma unroll
    for (int c = 0; c < K; ++c) {
        unsigned d;
        if (c == 0) {
            unsigned sg;
            asm("prmt.b32 %0, %1, %2, %3;" : "=r"(sg) : "r"(rw0), "r"(rw1), "r"(sel[0]));
            d = __vadd2(h_diag, sg);
        } else d = D[c];
        const unsigned h = __vimax3_s16x2(TA[c], la, d);
        if (MERGED) {
            const unsigned tn = __vimax3_s16x2(TG[c], lg, d);
            if (c == K - 1) t_last = tn;
            la = __vadd2(tn, c_nalpha);
            lg = __vadd2(tn, c_ngamma);
            TG[c] = lg;
        } else {
            la = __vadd2(h, c_nalpha);
            if (c == K - 1) t_last = h;
        }
        TA[c] = la;
        if (c >= 1) {
            unsigned sg;
            asm("prmt.b32 %0, %1, %2, %3;" : "=r"(sg) : "r"(nw0), "r"(nw1), "r"(sel[c]));
            D[c] = __vadd2(hprev, sg);
        }
        if (CAP) hrow[c] = h;
        hprev = h;
    }
    h_last = hprev;
}

#ifndef WSB_S16G_MINB
#define WSB_S16G_MINB 4
#endif
template <int P, int K, int GAP, bool RAGGED, int AIMM = 0, int GIMM = 0, int MINB = WSB_S16G_MINB>
__global__ void __launch_bounds__(kThreads, MINB) s16_global_short_kernel(const ScoreParams prm) {
    constexpr int GPB = kThreads / P;
    constexpr int NCH = K / 4 + 1;
    constexpr int NW = NCH * 4;
    constexpr bool MERGED = GAP == GAP_MERGED;
    static_assert(P >= 4, "lanes 0..3 of a group carry the metadata of the four sequences of a unit");
    extern __shared__ uint4 smem_dyn[];
    uint4 (*snap)[NCH][GPB] = reinterpret_cast<uint4 (*)[NCH][GPB]>(smem_dyn);   // [half][quad][lane group]
    constexpr int QROWS = short16_qrows<P>();
    uint2 (*qbuf)[QROWS] = reinterpret_cast<uint2 (*)[QROWS]>(smem_dyn + 2 * NCH * GPB);
    uint8_t (*raw)[4][kShort16Raw] = reinterpret_cast<uint8_t (*)[4][kShort16Raw]>(&qbuf[GPB][0]);
    int (*meta)[16] = reinterpret_cast<int (*)[16]>(&raw[GPB][0][0]);

    const long long cycles_at_start = prm.block_cycles ? clock64() : 0;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int t = tid & (P - 1);
    const int gib = tid / P;
    const unsigned gmask = group_mask<P>(lane);
    const int64_t group_global = (int64_t)blockIdx.x * GPB + gib;
    const int64_t n_groups = (int64_t)gridDim.x * GPB;

    const int alpha = AIMM > 0 ? AIMM : prm.alpha;
    const int beta = prm.beta;
    const int gamma = GIMM > 0 ? GIMM : (MERGED ? min(prm.alpha, prm.beta) : prm.alpha);
    const unsigned c_nalpha = AIMM > 0 ? ((unsigned)(-AIMM) & 0xffffu) * 0x10001u : pack16(-prm.alpha);
    const unsigned c_ngamma = GIMM > 0 ? ((unsigned)(-GIMM) & 0xffffu) * 0x10001u : pack16(-gamma);
    const unsigned mism4 = (unsigned)(prm.mismatch & 0xff) * 0x01010101u;
    const unsigned dm1 = (unsigned)((prm.match ^ prm.mismatch) & 0xff);
    const unsigned keep = t == 0 ? 0u : (unsigned)prm.one;
    const unsigned estep = t == 0 ? pack16(-beta) : 0u;   // lane 0: the matrix' left border walks down by beta per row
    const int col0 = t * K;

    const int64_t rounds = (prm.n_units + n_groups - 1) / n_groups;
    const int sv = t & 3, pv = sv >> 1;
    const bool is_subject = (sv & 1) != 0;
    int mt_p = -1, mt_seq = 0, mt_len = 0;
    const uint8_t* mt_ptr = nullptr;
    auto meta_step = [&](int step, int64_t u) {   // as in score_short16.cuh: one dependent load per step
        if (step == 0) {
            mt_p = -1;
            if (u < prm.n_units) {
                if (prm.units) mt_p = prm.units[u * 2 + pv];
                else { const int64_t pp = prm.pair_base + u * 2 + pv; mt_p = pp < prm.n_pairs ? (int)pp : -1; }
            }
        } else if (step == 1) {
            mt_seq = mt_p >= 0 ? (is_subject ? prm.pair_s[mt_p] : prm.pair_q[mt_p]) : 0;
        } else if (step == 2) {
            mt_len = 0; mt_ptr = is_subject ? prm.s_codes : prm.q_codes;
            if (mt_p >= 0) {
                mt_len = is_subject ? prm.s_len[mt_seq] : prm.q_len[mt_seq];
                mt_ptr += is_subject ? prm.s_off[mt_seq] : prm.q_off[mt_seq];
            }
        } else {
            const unsigned shift = (unsigned)(reinterpret_cast<uintptr_t>(mt_ptr) & 15u);
            if (t < 4) {
                meta[gib][2 + sv] = mt_len;
                meta[gib][6 + sv] = (int)shift;
                if (!is_subject) meta[gib][pv] = mt_p;
            }
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint8_t* base = reinterpret_cast<const uint8_t*>(
                    __shfl_sync(gmask, (unsigned long long)(reinterpret_cast<uintptr_t>(mt_ptr) & ~(uintptr_t)15), s, P));
                const int bytes = __shfl_sync(gmask, mt_len > 0 ? mt_len + (int)shift : 0, s, P);
                const unsigned dst = (unsigned)__cvta_generic_to_shared(&raw[gib][s][0]);
                for (int x = t * 16; x < bytes; x += P * 16) cp_async16(dst + x, base + x);
            }
        }
    };
    if (rounds > 0) {
#pragma unroll
        for (int step = 0; step < 4; ++step) meta_step(step, group_global);
    }

    for (int64_t rd = 0; rd < rounds; ++rd) {
        cp_async_wait_all();
        __syncwarp();
        int pidx[2], m[2], n[2], qsh[2], ssh[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            pidx[v] = meta[gib][v];
            m[v] = meta[gib][2 + 2 * v]; n[v] = meta[gib][3 + 2 * v];
            qsh[v] = meta[gib][6 + 2 * v]; ssh[v] = meta[gib][7 + 2 * v];
        }
        const int mm_w = __reduce_max_sync(0xffffffffu, max(m[0], m[1]));
        const int64_t u_next = (rd + 1) * n_groups + group_global;
        if (mm_w == 0) {
            __syncwarp();
            if (rd + 1 < rounds) {
#pragma unroll
                for (int step = 0; step < 4; ++step) meta_step(step, u_next);
            }
            continue;
        }
        {   // query buffer: P pad rows, the rows of both queries as row words, pad rows for the ramp-down
            constexpr int UNR = 4;
            const int total = mm_w + 2 * P + 2;
            for (int x0 = t; x0 < total; x0 += P * UNR) {
                unsigned c0[UNR], c1[UNR];
#pragma unroll
                for (int k = 0; k < UNR; ++k) {
                    const int row = x0 + P * k - P;
                    c0[k] = (row >= 0 && row < m[0]) ? raw[gib][0][qsh[0] + row] : 4u;
                    c1[k] = (row >= 0 && row < m[1]) ? raw[gib][2][qsh[1] + row] : 4u;
                }
#pragma unroll
                for (int k = 0; k < UNR; ++k) {
                    uint2 rw;
                    rw.x = c0[k] < 4 ? mism4 ^ (dm1 << (8 * c0[k])) : mism4;
                    rw.y = c1[k] < 4 ? mism4 ^ (dm1 << (8 * c1[k])) : mism4;
                    if (x0 + P * k < total) qbuf[gib][x0 + P * k] = rw;
                }
            }
        }
        // strip state at row 0: T(0, j) = H(0, j) = edge; D[c] = H(0, c - 1) + sigma(row 1, c)
        unsigned sel[K], TA[K], TG[MERGED ? K : 1], D[K];
        D[0] = 0u;
        const bool flagged_subject = build_selectors16<K>(raw[gib][1], raw[gib][3], ssh[0] + col0, ssh[1] + col0, n[0] - col0,
                                                          n[1] - col0, sel);
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const int e = edge_h(true, col0 + c + 1, prm.alpha, beta);
            TA[c] = pack16(e - alpha);
            if (MERGED) TG[c] = pack16(e - gamma);
        }
        if (__any_sync(gmask, flagged_subject)) {
            if (t == 0) {
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (pidx[v] >= 0) { const int at = atomicAdd(prm.redo_count, 1); prm.redo[at] = pidx[v]; }
            }
        }
        __syncwarp();
        {
            const uint2 rw = qbuf[gib][P];   // row 1 (every lane starts at row 1: masked until then)
#pragma unroll
            for (int c = 1; c < K; ++c) {
                unsigned sg;
                asm("prmt.b32 %0, %1, %2, %3;" : "=r"(sg) : "r"(rw.x), "r"(rw.y), "r"(sel[c]));
                D[c] = __vadd2(pack16(edge_h(true, col0 + c, prm.alpha, beta)), sg);
            }
        }
        unsigned ta_l = 0u, tg_l = 0u;
        unsigned h_l = pack16(edge_h(true, col0, prm.alpha, beta)), h_d = 0u;   // H(0, col0): diagonal of the strip's row 1
        unsigned eg = t == 0 ? pack16(edge_h(true, 1, prm.alpha, beta)) : 0u;   // lane 0: H(row, 0) = T(row, 0)
        const unsigned qbase = (unsigned)__cvta_generic_to_shared(&qbuf[gib][0]);
        unsigned qaddr = qbase + 8u * (unsigned)P;    // row r lives at index r - 1 + P; a lane advances only while active

        unsigned s_t = 0u, s_h = 0u;
        unsigned qc0, qc1, qn0, qn1;   // row words of the lane's coming row and the one after it (fetched one trip ahead)
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(qc0), "=r"(qc1) : "r"(qaddr) : "memory");
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2+8];" : "=r"(qn0), "=r"(qn1) : "r"(qaddr) : "memory");
        int rowi = 0;   // row this lane finished last
        const int own0 = (n[0] - 1) / K, own1 = (n[1] - 1) / K;   // lanes that own column n of either half
        // one trip: CAP = park the row in shared memory when it is row m of a half
        auto trip = [&](auto cap_tag) {
            constexpr bool CAP = decltype(cap_tag)::value;
            // hand-over from the previous trip: lane 0 takes the matrix edge (keep = 0) through the multiply-add
            h_d = h_l;
            const unsigned t_in = s_t * keep + eg;
            ta_l = __vadd2(t_in, c_nalpha);
            if (MERGED) tg_l = __vadd2(t_in, c_ngamma);
            h_l = s_h * keep + eg;
            eg = __vadd2(eg, estep);
            unsigned la = ta_l, lg = tg_l, h_last, t_last;
            unsigned hrow[NW];
            g16_row<K, NW, MERGED, CAP>(sel, TA, TG, D, c_nalpha, c_ngamma, qc0, qc1, qn0, qn1, h_d, la, lg, h_last, t_last, hrow);
            asm volatile("ld.shared.v2.b32 {%0, %1}, [%2+8];" : "=r"(qc0), "=r"(qc1) : "r"(qaddr) : "memory");
            asm volatile("ld.shared.v2.b32 {%0, %1}, [%2+16];" : "=r"(qn0), "=r"(qn1) : "r"(qaddr) : "memory");
            qaddr += 8;
            if constexpr (CAP) {
                ++rowi;
#pragma unroll
                for (int c = K; c < NW; ++c) hrow[c] = 0u;
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (rowi == m[v] && t == (v ? own1 : own0)) {   // only the lane that owns column n parks its strip
#pragma unroll
                        for (int ch = 0; ch < NCH; ++ch)
                            snap[v][ch][gib] = make_uint4(hrow[4 * ch], hrow[4 * ch + 1], hrow[4 * ch + 2], hrow[4 * ch + 3]);
                    }
            }
            s_t = t_last; s_h = h_last;   // sent by the caller, outside the mask
        };
        auto send = [&]() {
            s_t = __shfl_up_sync(0xffffffffu, s_t, 1, P);
            s_h = __shfl_up_sync(0xffffffffu, s_h, 1, P);
        };

        // ---- ramp-up: lane t joins at trip t + 1
        int done = 0, tau = 1;
#pragma unroll 1
        for (; tau < P; ++tau) {
            if (tau > t) {
                if constexpr (RAGGED) trip(std::true_type{}); else trip(std::false_type{});
            }
            send();
            ++done;
        }
        // ---- steady trips (every lane inside the matrix), interleaved with the next unit's metadata chain
        const int steps = mm_w + P - 1;
        const int body = RAGGED ? steps - done : max(0, mm_w - 1 - done);   // uniform: the last P trips capture
        const int quarter1 = (body + 3) / 4;
        int left = body;
#pragma unroll 1
        for (int part = 0; part < 4; ++part) {
            if (rd + 1 < rounds) meta_step(part, u_next);
            const int cnt = min(quarter1, left);
            left -= cnt;
#pragma unroll 1
            for (int k = 0; k < cnt; ++k, ++tau) {
                if (tau > t) {   // always true here; the branch keeps ptxas from rotating the strip registers (one MOV per column otherwise)
                    if constexpr (RAGGED) trip(std::true_type{}); else trip(std::false_type{});
                }
                send();
            }
        }
        done += body;
        if constexpr (!RAGGED) rowi = done - t;   // rows finished so far (the planner keeps m >= 2 P here: every lane is inside)
        // ---- the trips in which row m is finished (uniform batches)
#pragma unroll 1
        for (; done < steps; ++done) {
            trip(std::true_type{});
            send();
        }
        __syncwarp();

        // the lane that owns column n reads H(m, n) from its parked row
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            if (pidx[v] < 0 || m[v] <= 0 || n[v] <= 0) continue;
            const int owner = (n[v] - 1) / K, idx = (n[v] - 1) - owner * K;
            if (t == owner) {
                const unsigned* words = reinterpret_cast<const unsigned*>(&snap[v][idx >> 2][gib]);
                const int sc = half16(words[idx & 3], v);
                prm.out_score[pidx[v]] = sc;
                prm.out_i[pidx[v]] = m[v];
                prm.out_j[pidx[v]] = n[v];
            }
        }
        __syncwarp();
    }
    if (prm.block_cycles && tid == 0) prm.block_cycles[blockIdx.x] = (unsigned long long)(clock64() - cycles_at_start);
}

}  // namespace wsb
