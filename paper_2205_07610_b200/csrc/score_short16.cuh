// score_short16.cuh -- packed int16x2 (DPX) LOCAL scoring of short reads that fit one stage.
//
// Same lane-group wavefront, two alignments per register and two rows per trip as score_short.cuh, but in 16-bit
// integers with the DPX packed instructions instead of half2 arithmetic.  What that buys (measured with
// tools/ubench: 8.5 cycles per packed cell against 10.7 for the half2 mix):
//   * the substitution scores of BOTH alignments come from ONE byte permute: the two query symbols of a row are kept as
//     two "row words" (sigma(q, s) for s = 0..3 in the four bytes), each column keeps a 16-bit PRMT selector built from
//     its two subject symbols, and PRMT(rowA, rowB, sel[c]) is the packed pair {sigma_B, sigma_A}, sign-extended;
//   * no "+ mismatch" carry: the diagonal candidate is H_diag + sigma directly, so a cell is
//         sigma = PRMT(rowA, rowB, sel[c])                 ALU
//         d     = H_diag + sigma                           VIADD.16x2       FMA pipe
//         h     = max3(TA_up, TA_left, d, 0)               VIMNMX3.S16x2.RELU  ALU
//         tn    = max3(TG_up, TG_left, d, 0)               VIMNMX3.S16x2.RELU  ALU
//         TA    = tn - alpha ; TG = tn - gamma             2 x VIADD.16x2   FMA pipe
//     = 3 ALU + 3 FMA-pipe instructions per two cells (+ half a VIMNMX3 for the row maximum), against 3.5 + 4 in half2;
//   * a 16-bit value range: max_step * (m + n) up to 32 000 instead of 2 048.
// Reference semantics: merged affine update _kernels.py:259-276, linear :113-126, end-cell rule :130-145.
//
// Limits (the planner checks them, otherwise the half2 / int32 kernels run): |match|, |mismatch| <= 127, mismatch <= 0 <=
// match, merged-exact scheme, and no flagged (non-ACGT) SUBJECT symbol -- a selector can only pick one of the four
// row-word bytes, so a flagged subject symbol has no exact encoding.  The kernel detects such a symbol while loading
// the strip and reports the pair through ScoreParams::redo (it is then re-scored by the half2 / int32 path); pad columns
// use a sign-fill selector (sigma in {0, -1}: never improving, which is all a pad needs).  Flagged QUERY symbols are
// exact (row word = mismatch in all four bytes).
#pragma once
#include "score_kernels.cuh"

namespace wsb {

constexpr int kShort16QRows = 200;  // query rows per lane group (150 bp reads + 4P + 2 pad rows at P = 8)

template <int P, int K> constexpr size_t short16_smem_bytes() {
    return (size_t)2 * (K / 4 + 1) * kThreads * 16 + (size_t)(kThreads / P) * kShort16QRows * 8;
}

__device__ __forceinline__ unsigned pack16(int x) { return ((unsigned)x & 0xffffu) * 0x10001u; }
__device__ __forceinline__ int half16(unsigned w, int v) { return (int)(short)(v ? (w >> 16) : (w & 0xffffu)); }

// Record test + snapshot for both halves: a half records when the row maximum raised its running best
// (nb = max(best, rm) differs from best in that half).  The strip's H row goes to that half's snapshot area in 16-byte
// chunks (one chunk every kThreads * 16 = 2048 bytes); stores are predicated, a row without a record costs issue slots only.
#define WSB_S16_PRED                                   \
    "{\n\t.reg .pred p, q;\n\t.reg .b32 c, l;\n\t"     \
    "xor.b32 c, %0, %1;\n\t"                           \
    "and.b32 l, c, 0xffff;\n\t"                        \
    "setp.ne.u32 p, l, 0;\n\t"                         \
    "setp.gt.u32 q, c, 0xffff;\n\t"
#define WSB_S16_ST(off, a, b, c_, d)                                                  \
    "@p st.shared.v4.b32 [%2+" #off "], {%" #a ", %" #b ", %" #c_ ", %" #d "};\n\t"   \
    "@q st.shared.v4.b32 [%3+" #off "], {%" #a ", %" #b ", %" #c_ ", %" #d "};\n\t"

template <int NC>
__device__ __forceinline__ void record16_chunks(const unsigned* w, unsigned nb, unsigned best, unsigned addr_p, unsigned addr_q) {
    static_assert(NC >= 1 && NC <= 5, "chunk group size");
    if constexpr (NC == 4) {
        asm volatile(WSB_S16_PRED WSB_S16_ST(0, 4, 5, 6, 7) WSB_S16_ST(2048, 8, 9, 10, 11) WSB_S16_ST(4096, 12, 13, 14, 15)
                     WSB_S16_ST(6144, 16, 17, 18, 19) "}\n"
                     :
                     : "r"(nb), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]),
                       "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]),
                       "r"(w[14]), "r"(w[15])
                     : "memory");
    }
    if constexpr (NC == 5) {
        asm volatile(WSB_S16_PRED WSB_S16_ST(0, 4, 5, 6, 7) WSB_S16_ST(2048, 8, 9, 10, 11) WSB_S16_ST(4096, 12, 13, 14, 15)
                     WSB_S16_ST(6144, 16, 17, 18, 19) WSB_S16_ST(8192, 20, 21, 22, 23) "}\n"
                     :
                     : "r"(nb), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]),
                       "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]),
                       "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19])
                     : "memory");
    }
    static_assert(NC == 4 || NC == 5, "instantiated strip widths: K = 12..19");
}

// H[] row plus the iteration tag in the first spare word after the K columns (the snapshot then also records WHEN)
template <int K> __device__ __forceinline__ void record16_rows(const unsigned (&h)[K], unsigned nb, unsigned best,
                                                               unsigned snap_addr, unsigned tag) {
    constexpr int NCH = K / 4 + 1;
    unsigned w[NCH * 4];
#pragma unroll
    for (int c = 0; c < NCH * 4; ++c) w[c] = c < K ? h[c] : tag;
    constexpr unsigned HS = NCH * kThreads * 16;  // byte distance between the two halves' snapshot areas
    record16_chunks<NCH>(w, nb, best, snap_addr, snap_addr + HS);
}

template <int NCH> __device__ __forceinline__ void record16_quads(const uint4 (&hq)[NCH], unsigned nb, unsigned best,
                                                                  unsigned snap_addr) {
    unsigned w[NCH * 4];
#pragma unroll
    for (int k = 0; k < NCH; ++k) { w[4 * k] = hq[k].x; w[4 * k + 1] = hq[k].y; w[4 * k + 2] = hq[k].z; w[4 * k + 3] = hq[k].w; }
    constexpr unsigned HS = NCH * kThreads * 16;
    record16_chunks<NCH>(w, nb, best, snap_addr, snap_addr + HS);
}

template <int P, int K, int GAP>
__global__ void __launch_bounds__(kThreads, 4) s16_local_short_kernel(const ScoreParams prm) {
    constexpr int GPB = kThreads / P;
    constexpr int NCH = K / 4 + 1;
    extern __shared__ uint4 smem_dyn[];
    uint4 (*snap)[NCH][kThreads] = reinterpret_cast<uint4 (*)[NCH][kThreads]>(smem_dyn);
    uint2 (*qbuf)[kShort16QRows] = reinterpret_cast<uint2 (*)[kShort16QRows]>(smem_dyn + 2 * NCH * kThreads);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int t = tid & (P - 1);
    const int gib = tid / P;
    const unsigned gmask = group_mask<P>(lane);
    const int64_t group_global = (int64_t)blockIdx.x * GPB + gib;
    const int64_t n_groups = (int64_t)gridDim.x * GPB;
    const unsigned snap_addr = (unsigned)__cvta_generic_to_shared(&snap[0][0][tid]);

    const int gamma = GAP == GAP_MERGED ? min(prm.alpha, prm.beta) : prm.alpha;
    const unsigned c_nalpha = pack16(-prm.alpha);
    const unsigned c_ngamma = pack16(-gamma);
    const unsigned mism4 = (unsigned)(prm.mismatch & 0xff) * 0x01010101u;
    const unsigned match1 = (unsigned)(prm.match & 0xff);
    // lane 0 sees the matrix' zero left border instead of a neighbour: x * keep + edge (IMAD, FMA pipe)
    const unsigned keep = t == 0 ? 0u : 1u;
    const unsigned edge_ta = t == 0 ? c_nalpha : 0u;
    const unsigned edge_tg = t == 0 ? c_ngamma : 0u;
    const int col0 = t * K;

    const int64_t rounds = (prm.n_units + n_groups - 1) / n_groups;
    for (int64_t rd = 0; rd < rounds; ++rd) {
        const int64_t u = rd * n_groups + group_global;
        int pidx[2], m[2], n[2];
        const uint8_t* qp[2];
        const uint8_t* sp[2];
        int mm = 0;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            int p = -1;
            if (u < prm.n_units) {
                if (prm.units) p = prm.units[u * 2 + v];
                else { const int64_t pp = prm.pair_base + u * 2 + v; p = pp < prm.n_pairs ? (int)pp : -1; }
            }
            pidx[v] = p; m[v] = 0; n[v] = 0; qp[v] = nullptr; sp[v] = nullptr;
            if (p >= 0) {
                const int a = prm.pair_q[p], b = prm.pair_s[p];
                m[v] = prm.q_len[a]; n[v] = prm.s_len[b];
                qp[v] = prm.q_codes + prm.q_off[a];
                sp[v] = prm.s_codes + prm.s_off[b];
            }
            mm = max(mm, m[v]);
        }
        const int mm_w = __reduce_max_sync(0xffffffffu, mm);
        if (mm_w == 0) continue;

        // query buffer: 2P pad rows, the rows of both queries as row words, then pad rows for the ramp-down.  Loads are
        // issued in batches of 8 per lane before any is consumed.
        __syncwarp();
        {
            constexpr int UNR = 8;
            const int total = mm_w + 4 * P + 2;
            for (int x0 = t; x0 < total; x0 += P * UNR) {
                int raw[UNR][2];
#pragma unroll
                for (int k = 0; k < UNR; ++k) {
                    const int row = x0 + P * k - 2 * P;
#pragma unroll
                    for (int v = 0; v < 2; ++v) raw[k][v] = (row >= 0 && row < m[v]) ? (int)qp[v][row] : 4;
                }
#pragma unroll
                for (int k = 0; k < UNR; ++k) {
                    const int x = x0 + P * k;
                    uint2 rw;   // sigma(q, s) for s = 0..3: match in the byte of the query symbol, mismatch elsewhere
                    rw.x = raw[k][0] < 4 ? (mism4 & ~(0xffu << (8 * raw[k][0]))) | (match1 << (8 * raw[k][0])) : mism4;
                    rw.y = raw[k][1] < 4 ? (mism4 & ~(0xffu << (8 * raw[k][1]))) | (match1 << (8 * raw[k][1])) : mism4;
                    if (x < total) qbuf[gib][x] = rw;
                }
            }
        }
        // per column: PRMT selector of the two subject symbols, TA = T - alpha, TG = T - gamma, H
        // H lives in uint4 quads (the snapshot stores are 16-byte stores; the spare word after column K-1 takes the tag)
        unsigned sel[K], TA[K], TG[GAP == GAP_MERGED ? K : 1];
        uint4 Hq[NCH];
        auto Hc = [&](int c) -> unsigned& {
            uint4& q4 = Hq[c >> 2];
            return (c & 3) == 0 ? q4.x : (c & 3) == 1 ? q4.y : (c & 3) == 2 ? q4.z : q4.w;
        };
        bool flagged_subject = false;
#pragma unroll
        for (int c = 0; c < K; ++c) {
            unsigned nib[2] = {0x88u, 0x88u};   // pad column: sign fill of byte 0 in both bytes -> sigma in {0, -1}
#pragma unroll
            for (int v = 0; v < 2; ++v)
                if (col0 + c < n[v]) {
                    const unsigned x = sp[v][col0 + c];
                    if (x < 4) nib[v] = (x + 4u * v) | ((x + 4u * v) | 8u) << 4;   // value byte, then its sign byte
                    else flagged_subject = true;
                }
            sel[c] = nib[0] | (nib[1] << 8);
            TA[c] = c_nalpha;
            if (GAP == GAP_MERGED) TG[c] = c_ngamma;
            Hc(c) = 0u;
        }
#pragma unroll
        for (int c = K; c < 4 * NCH; ++c) Hc(c) = 0u;
        // a flagged subject symbol cannot be encoded: hand the pair(s) of this unit to the fallback list
        if (__any_sync(gmask, flagged_subject)) {
            if (t == 0) {
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (pidx[v] >= 0) { const int at = atomicAdd(prm.redo_count, 1); prm.redo[at] = pidx[v]; }
            }
        }
        __syncwarp();

        unsigned ta_lA = c_nalpha, tg_lA = c_ngamma, h_lA = 0u;   // left border of row A: T - alpha, T - gamma, H
        unsigned ta_lB = c_nalpha, tg_lB = c_ngamma, h_lB = 0u;   // ... of row B
        unsigned h_dA = 0u;                                       // H(rA - 1, left column): diagonal of row A, cell 0
        unsigned bestvec = 0u;
        const unsigned qbase = (unsigned)__cvta_generic_to_shared(&qbuf[gib][0]);
        unsigned qaddr = qbase + 8u * (unsigned)(2 * P - 2 * t);    // row r lives at qbuf index r - 1 + 2P
        const unsigned qend = qaddr + 16u * (unsigned)((mm_w + 1) / 2 + P - 1);

        // one row of the strip, in place: H[] holds the previous row on entry and this row on exit
        auto row = [&](unsigned rwA, unsigned rwB, unsigned h_diag, unsigned& la, unsigned& lg, unsigned& rm) {
            rm = 0u;
            unsigned hd = h_diag, hprev = 0u;
#pragma unroll
            for (int c = 0; c < K; ++c) {
                unsigned sg;
                asm("prmt.b32 %0, %1, %2, %3;" : "=r"(sg) : "r"(rwA), "r"(rwB), "r"(sel[c]));
                const unsigned d = __vadd2(hd, sg);
                hd = Hc(c);
                const unsigned h = __vimax3_s16x2_relu(TA[c], la, d);
                if (GAP == GAP_MERGED) {
                    const unsigned tn = __vimax3_s16x2_relu(TG[c], lg, d);
                    la = __vadd2(tn, c_nalpha);
                    lg = __vadd2(tn, c_ngamma);
                    TG[c] = lg;
                } else {
                    la = __vadd2(h, c_nalpha);
                }
                TA[c] = la;
                Hc(c) = h;
                if (c & 1) rm = __vimax3_s16x2(rm, hprev, h);
                else if (c == K - 1) rm = __vmaxs2(rm, h);
                hprev = h;
            }
        };
        unsigned qa0, qa1, qb0, qb1;  // row words of rows A and B, fetched one trip ahead of their use
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(qa0), "=r"(qa1), "=r"(qb0), "=r"(qb1) : "r"(qaddr) : "memory");
#pragma unroll 1
        while (qaddr != qend) {
            const unsigned a0 = qa0, a1 = qa1, b0 = qb0, b1 = qb1;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4+16];" : "=r"(qa0), "=r"(qa1), "=r"(qb0), "=r"(qb1) : "r"(qaddr) : "memory");
            unsigned laA = ta_lA, lgA = tg_lA, laB = ta_lB, lgB = tg_lB, rmA, rmB;
            row(a0, a1, h_dA, laA, lgA, rmA);
            unsigned nb = __vmaxs2(bestvec, rmA);
            Hc(K) = qaddr;
            record16_quads<NCH>(Hq, nb, bestvec, snap_addr);
            bestvec = nb;
            const unsigned hA_last = Hc(K - 1);
            row(b0, b1, h_lA, laB, lgB, rmB);
            h_dA = h_lB;
            const unsigned s0 = __shfl_up_sync(0xffffffffu, laA, 1, P);
            const unsigned s1 = __shfl_up_sync(0xffffffffu, hA_last, 1, P);
            const unsigned s2 = __shfl_up_sync(0xffffffffu, laB, 1, P);
            const unsigned s3 = __shfl_up_sync(0xffffffffu, Hc(K - 1), 1, P);
            unsigned s4 = 0u, s5 = 0u;
            if (GAP == GAP_MERGED) {
                s4 = __shfl_up_sync(0xffffffffu, lgA, 1, P);
                s5 = __shfl_up_sync(0xffffffffu, lgB, 1, P);
            }
            nb = __vmaxs2(bestvec, rmB);
            Hc(K) = qaddr + 8;
            record16_quads<NCH>(Hq, nb, bestvec, snap_addr);
            bestvec = nb;
            qaddr += 16;
            ta_lA = s0 * keep + edge_ta;
            h_lA = s1 * keep;
            ta_lB = s2 * keep + edge_ta;
            h_lB = s3 * keep;
            if (GAP == GAP_MERGED) {
                tg_lA = s4 * keep + edge_tg;
                tg_lB = s5 * keep + edge_tg;
            }
        }

        // reduce over the group: max value, then smallest row, then smallest strip; the winner resolves its column
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            int bv = half16(bestvec, v);
            int bi = 0, bj = col0, who = t;
            if (bv > 0) {  // the tag word after the K columns holds the query-buffer address of the record row
                const uint4 w = snap[v][K / 4][tid];
                const unsigned tag = (K % 4 == 0) ? w.x : (K % 4 == 1) ? w.y : (K % 4 == 2) ? w.z : w.w;
                bi = (int)((tag - qbase) >> 3) - 2 * P + 1;  // buffer index -> matrix row
                if (bi > m[v] || bi < 1) bv = 0;       // cannot happen for a real record; keeps pads out defensively
            }
#pragma unroll
            for (int off = P / 2; off >= 1; off >>= 1) {
                const int ov = __shfl_xor_sync(gmask, bv, off, P);
                const int oi = __shfl_xor_sync(gmask, bi, off, P);
                const int oj = __shfl_xor_sync(gmask, bj, off, P);
                const int ow = __shfl_xor_sync(gmask, who, off, P);
                if (better_cell(ov, oi, oj, bv, bi, bj)) { bv = ov; bi = oi; bj = oj; who = ow; }
            }
            if (t == who && pidx[v] >= 0) {
                int j = 0;
                if (bv > 0) {
                    int pos = K;
#pragma unroll
                    for (int ch = (K - 1) / 4; ch >= 0; --ch) {
                        const uint4 w = snap[v][ch][tid];
                        if (4 * ch + 3 < K && half16(w.w, v) == bv) pos = 4 * ch + 3;
                        if (4 * ch + 2 < K && half16(w.z, v) == bv) pos = 4 * ch + 2;
                        if (4 * ch + 1 < K && half16(w.y, v) == bv) pos = 4 * ch + 1;
                        if (half16(w.x, v) == bv) pos = 4 * ch;
                    }
                    j = bj + pos + 1;
                } else { bi = 0; }
                prm.out_score[pidx[v]] = bv;
                prm.out_i[pidx[v]] = bi;
                prm.out_j[pidx[v]] = j;
            }
        }
    }
}

}  // namespace wsb
