// traceback_fill16.cuh -- packed int16 direction-code fill: two alignments of a uniform batch per thread (sm_100a).
//
// Same wavefront, same bit planes and the same code-block layout as tb_fill_kernel (traceback_kernels.cuh), so the walk
// kernels read either fill's output.  The two alignments of a unit live in the 16-bit halves of every value, and the
// four "max with who-won" steps of the Gotoh cell become one VIMNMX.S16x2 each: the instruction returns the packed
// maximum AND one predicate per half ("the first operand won"), which the int32 form needs ISETP + SEL for.  Per packed
// cell (two matrix cells): 4 VIMNMX.S16x2, 8 predicated plane-bit adds (ptxas splits them between IMAD and LEA, i.e.
// between the FMA and the ALU pipe), 5 VIADD.16x2, and HSET2.EQ + LOP3 for the substitution score -- 19 instructions
// for two cells where the int32 fill issues 16 for one.
//
// Substitution: symbols travel as the half-precision bit patterns 0x4000 | code (normal numbers, so the comparison is
// exact whatever the denormal mode); flagged query symbols are 0x4004, flagged or padded subject symbols 0x4005, which
// never compare equal (core.py:147-151: flagged symbols never match, even N-N).
//
// Scope (the host checks it, traceback_host.inl): every subject of the launch within one stage (n <= P*K, no border
// scratch) and the int16 range rule below; affine or linear gaps (AFFINE = false drops E / F and their planes: two
// packed maxes per cell).  Longer reads and wider schemes stay on the int32 fill.  Local alignments add a fifth max per packed cell (0 against H: the "H == 0" stop plane, folded into the two
// origin planes once per eight cells).
#pragma once
#include "traceback_kernels.cuh"

#include <cuda_fp16.h>

namespace wsb {

#ifndef WSB_TB16_ALU_E
#define WSB_TB16_ALU_E 0
#endif
constexpr bool kMarkE = WSB_TB16_ALU_E != 0;   // 1: set the "E extends" plane bits on the ALU pipe (measured 9 % slower: the packed adds already live there)
#ifndef WSB_TB16_FMA_ADDS
#define WSB_TB16_FMA_ADDS 0
#endif
// Values are stored biased by kBias16 per half, so that every half is a non-negative number: subtracting a packed
// non-negative constant with ONE 32-bit operation then never borrows across the halves, and the three "minus gap cost"
// steps of the cell can issue as IMAD on the FMA pipe instead of VIADD.16x2 on the ALU pipe (bit mask: 1 = E - beta,
// 2 = F - beta, 4 = H - alpha).
constexpr int kFmaAdds = WSB_TB16_FMA_ADDS;
constexpr int kBias16 = 16384;
constexpr int kNeg16 = -16000;   // "minus infinity" of the packed fill: below every reachable value, never extended twice

// the packed fill is exact while every reachable value stays inside int16 with room for one more step below kNeg16
__host__ __device__ inline bool tb_fill16_range_ok(int m, int n, int match, int mismatch, int alpha, int beta) {
    const int64_t lo = 3ll * alpha + (int64_t)beta * (m + n) + (mismatch < 0 ? -mismatch : mismatch) + (match < 0 ? -match : match);
    const int64_t hi = (int64_t)(match > 0 ? match : 0) * (m < n ? m : n) + alpha + beta;
    return lo <= 8000 && hi <= 16000 && alpha <= 300 && beta <= 300;
}

__device__ __forceinline__ unsigned pk16(int v) { return ((unsigned)v & 0xffffu) * 0x00010001u; }          // plain, both halves
__device__ __forceinline__ unsigned pk16b(int v) { return (unsigned)(v + kBias16) * 0x00010001u; }           // biased value
__device__ __forceinline__ int lo16(unsigned v) { return (int)(v & 0xffffu) - kBias16; }
__device__ __forceinline__ int hi16(unsigned v) { return (int)(v >> 16) - kBias16; }
// x - cost in both halves (cost = c * 0x10001, 0 <= c <= every half of x): one IMAD, or VIADD.16x2 with the negated halves
template <bool ON_FMA>
__device__ __forceinline__ unsigned sub_cost(unsigned x, unsigned cost32, unsigned neg2, int one) {
    if (ON_FMA) {
        unsigned r;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(one), "r"(0u - cost32), "r"(x));
        return r;
    }
    return __vadd2(x, neg2);
}

// packed max(a, b), "a wins ties"; the plane bit goes to wlo / whi where a won in the low / high half.  The bit is
// set on the FMA pipe (IMAD with the opaque multiplier one == 1) or, ON_ALU, on the ALU pipe (predicated LOP3): the cell
// mixes both so that neither pipe carries the whole load.
// a[idx] for a register array: a binary tree of selects under log2 predicates (the array is padded to a power of two with
// copies of its last element), where the linear compare-and-select chain of select_reg costs 2K instructions -- it runs
// on every row of a semiglobal fill
template <int K>
__device__ __forceinline__ unsigned pick_reg(const unsigned (&a)[K], int idx) {
    constexpr int N = K <= 8 ? 8 : K <= 16 ? 16 : K <= 32 ? 32 : 64;
    static_assert(K <= N, "strip too wide");
    unsigned v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = a[i < K ? i : K - 1];
#pragma unroll
    for (int width = N / 2, bit = 1; width >= 1; width /= 2, bit *= 2) {
        const bool odd = (idx & bit) != 0;
#pragma unroll
        for (int i = 0; i < width; ++i) v[i] = odd ? v[2 * i + 1] : v[2 * i];
    }
    return v[0];
}

// a[idx] with an index that is the same in every lane of the warp (uniform batches: column n sits in the same register of
// every lane group): a jump table instead of a select tree
template <int K>
__device__ __forceinline__ unsigned pick_reg_uniform(const unsigned (&a)[K], int idx) {
    unsigned v = a[K - 1];
    switch (idx) {
#define WSB_PICK(i) case i: if (i < K) v = a[i < K ? i : 0]; break;
        WSB_PICK(0) WSB_PICK(1) WSB_PICK(2) WSB_PICK(3) WSB_PICK(4) WSB_PICK(5) WSB_PICK(6) WSB_PICK(7)
        WSB_PICK(8) WSB_PICK(9) WSB_PICK(10) WSB_PICK(11) WSB_PICK(12) WSB_PICK(13) WSB_PICK(14) WSB_PICK(15)
        WSB_PICK(16) WSB_PICK(17) WSB_PICK(18) WSB_PICK(19) WSB_PICK(20) WSB_PICK(21) WSB_PICK(22) WSB_PICK(23)
        WSB_PICK(24) WSB_PICK(25) WSB_PICK(26) WSB_PICK(27) WSB_PICK(28) WSB_PICK(29) WSB_PICK(30) WSB_PICK(31)
#undef WSB_PICK
        default: break;
    }
    return v;
}

template <bool ON_ALU>
__device__ __forceinline__ unsigned max_mark2(unsigned a, unsigned b, uint32_t& wlo, uint32_t& whi, uint32_t bit, int one) {
    unsigned r;
    if (ON_ALU) {
        asm("{\n\t.reg .pred pl, ph;\n\t.reg .s16 r0, r1, a0, a1;\n\t"
            "max.s16x2 %0, %3, %4;\n\t"
            "mov.b32 {r0, r1}, %0;\n\t"
            "mov.b32 {a0, a1}, %3;\n\t"
            "setp.eq.s16 pl, r0, a0;\n\t"
            "setp.eq.s16 ph, r1, a1;\n\t"
            "@pl or.b32 %1, %1, %5;\n\t"
            "@ph or.b32 %2, %2, %5;\n\t"
            "}" : "=r"(r), "+r"(wlo), "+r"(whi) : "r"(a), "r"(b), "r"(bit));
    } else {
        asm("{\n\t.reg .pred pl, ph;\n\t.reg .s16 r0, r1, a0, a1;\n\t"
            "max.s16x2 %0, %3, %4;\n\t"
            "mov.b32 {r0, r1}, %0;\n\t"
            "mov.b32 {a0, a1}, %3;\n\t"
            "setp.eq.s16 pl, r0, a0;\n\t"
            "setp.eq.s16 ph, r1, a1;\n\t"
            "@pl mad.lo.u32 %1, %6, %5, %1;\n\t"
            "@ph mad.lo.u32 %2, %6, %5, %2;\n\t"
            "}" : "=r"(r), "+r"(wlo), "+r"(whi) : "r"(a), "r"(b), "r"(bit), "r"(one));
    }
    return r;
}

// RAGGED = false: every pair of the launch has the same (m, n) (checked on the host), so the two alignments of a unit
// share every bound.  RAGGED = true: the halves carry pairs of different sizes; the unit runs max(m) rows, every half
// stores and tracks only inside its own rectangle (junk outside it flows right / down only, never back in -- the
// argument of the reference's packed mode, _kernels.py:557-562), and rejected or empty pairs ride along masked out.
template <int P, int K, int ATYPE, bool RAGGED, bool AFFINE = true>
__global__ void __launch_bounds__(kThreads, K <= 16 ? 4 : 1) tb_fill16_kernel(const TbParams prm) {
    constexpr int GPB = kThreads / P;
    constexpr int NW = K / 8;
    constexpr bool GLOBAL_EDGES = ATYPE == AT_GLOBAL;
    constexpr bool LOCAL = ATYPE == AT_LOCAL;   // end cells come from the score pass; H == 0 is stored as a stop code
    static_assert(K % 8 == 0, "K must pack into whole code words");

    // code words of four iterations per lane and half, read back by the thread that wrote them (no synchronisation); one
    // vector per (half, iteration, thread) keeps the 8- / 16-byte accesses of a warp contiguous
    using StageVec = typename std::conditional<NW == 2, uint2, typename std::conditional<NW == 4, uint4, uint3>::type>::type;
    static_assert(NW >= 2 && NW <= 4, "strip widths 16, 24, 32");
    __shared__ StageVec stage[2][4][kThreads];
    const int tid = threadIdx.x;
    const int t = tid & (P - 1);
    const int gib = tid / P;
    const int64_t group_global = (int64_t)blockIdx.x * GPB + gib;
    const int64_t n_groups = (int64_t)gridDim.x * GPB;
    const int alpha = prm.alpha, beta = prm.beta, one = prm.one;
    const unsigned nb2 = pk16(-beta), na2 = pk16(-alpha);
    const unsigned cb32 = (unsigned)beta * 0x00010001u, ca32 = (unsigned)alpha * 0x00010001u;
    const unsigned miss2 = pk16(prm.mismatch + alpha), hit2 = pk16(prm.match + alpha);   // sigma + alpha, both halves
    const unsigned neg2 = pk16b(kNeg16);
    // biased zero for the local stop test, kept opaque (times one == 1): as an immediate ptxas 12.9 moves it to the second
    // operand of VIMNMX.S16x2 and keeps using the "first operand won" predicates unchanged, which marks the wrong side
    const unsigned zero2 = pk16b(0) * (unsigned)one;
    const int64_t n_units = (prm.n_pairs + 1) / 2;

    // all lane groups of a warp run the same number of rounds (the shuffles below are warp-wide); a group without a unit
    // recomputes the last one and keeps its results to itself
    const int64_t rounds = (n_units + n_groups - 1) / n_groups;
    for (int64_t rd = 0; rd < rounds; ++rd) {
        const int64_t u_raw = rd * n_groups + group_global;
        const bool live = u_raw < n_units;
        const int64_t u = live ? u_raw : n_units - 1;
        const bool twin = 2 * u + 1 < prm.n_pairs;   // an odd tail computes its only alignment in both halves
        const int64_t ua = 2 * u, ub = twin ? ua + 1 : ua;
        const int64_t pa = prm.first_pair + ua, pb = prm.first_pair + ub;
        const int qa_i = prm.pair_q[pa], sa_i = prm.pair_s[pa], qb_i = prm.pair_q[pb], sb_i = prm.pair_s[pb];
        int m_a = prm.q_len[qa_i], n_a = prm.s_len[sa_i];
        int m_b = RAGGED ? prm.q_len[qb_i] : m_a, n_b = RAGGED ? prm.s_len[sb_i] : n_a;
        bool keep_a = live, keep_b = live && twin;   // this half stores codes and reports a result
        if (RAGGED) {   // rejected (negative code offset) or empty pairs: masked out, nothing read through their pointers
            if (prm.code_off[ua] < 0 || m_a == 0 || n_a == 0) { m_a = 0; n_a = 0; keep_a = false; }
            if (prm.code_off[ub] < 0 || m_b == 0 || n_b == 0) { m_b = 0; n_b = 0; keep_b = false; }
        }
        const int mm = max(m_a, m_b);
        const int mm_w = RAGGED ? __reduce_max_sync(0xffffffffu, mm) : mm;
        if (mm_w == 0) continue;
        const uint8_t* qa = prm.q_codes + prm.q_off[qa_i];
        const uint8_t* qb = prm.q_codes + prm.q_off[qb_i];
        const uint8_t* sa = prm.s_codes + prm.s_off[sa_i];
        const uint8_t* sb = prm.s_codes + prm.s_off[sb_i];
        uint32_t* code_a = prm.codes + ((!RAGGED || keep_a) ? prm.code_off[ua] : 0);
        uint32_t* code_b = prm.codes + ((!RAGGED || keep_b) ? prm.code_off[ub] : 0);
        const int col0 = t * K;
        const int rows4_a = tb_rows4(m_a, P), rows4_b = tb_rows4(m_b, P);

        unsigned ss[K], AL[K], EP[AFFINE ? K : 1];
#pragma unroll
        for (int c = 0; c < K; ++c) {
            unsigned x = 5u, y = 5u;
            if (col0 + c < n_a) { x = sa[col0 + c]; x = x < 4u ? x : 5u; }
            if (col0 + c < n_b) { y = sb[col0 + c]; y = y < 4u ? y : 5u; }
            ss[c] = (0x4000u | x) | ((0x4000u | y) << 16);
            AL[c] = pk16b(edge_h(GLOBAL_EDGES, col0 + c + 1, alpha, beta) - alpha);
            if (AFFINE) EP[c] = neg2;
        }
        const unsigned al_top = pk16b(edge_h(GLOBAL_EDGES, col0, alpha, beta) - alpha);
        unsigned al_diag = al_top, all = neg2, fpl = neg2;
        int edge = edge_h(GLOBAL_EDGES, 1, alpha, beta);
        if (t == 0) all = pk16b(edge - alpha);
        const int cap_a = n_a - 1 - col0, cap_b = n_b - 1 - col0;   // register index of matrix column n, if in this strip
        const bool has_cap_a = cap_a >= 0 && cap_a < K, has_cap_b = cap_b >= 0 && cap_b < K;
        int bv_a = GLOBAL_EDGES ? kNeg32 : 0, bi_a = 0, bj_a = ATYPE == AT_SEMI ? n_a : 0;
        int bv_b = bv_a, bi_b = 0, bj_b = ATYPE == AT_SEMI ? n_b : 0;
        // uniform semiglobal batches: the last matrix column is followed in packed form (both halves at once, biased
        // H - alpha values; the earliest row keeps ties), one VIMNMX.S16x2 + two selects per row
        const int cap_u = (n_a - 1) % K;
        unsigned col_best = pk16b(0 - alpha);   // H(0, n) = 0
        int col_i_a = 0, col_i_b = 0;

        // row m of a half: semiglobal scans it, global reads H(m, n)
        auto last_row = [&](bool second, int m, int n, bool has_cap, int cap_rel, int& bv, int& bi, int& bj) {
            if (ATYPE == AT_SEMI) {
#pragma unroll
                for (int c = 0; c < K; ++c)
                    if (col0 + c < n) {
                        const int v = (second ? hi16(AL[c]) : lo16(AL[c])) + alpha;
                        if (better_cell(v, m, col0 + c + 1, bv, bi, bj)) { bv = v; bi = m; bj = col0 + c + 1; }
                    }
            } else if (has_cap) {
                const unsigned hv = select_reg<unsigned, K>(AL, cap_rel);
                bv = (second ? hi16(hv) : lo16(hv)) + alpha; bi = m; bj = n;
            }
        };

        auto q_at = [&](int it) {
            unsigned a = 4u, b = 4u;
            if (!RAGGED || m_a > 0) { a = qa[min(max(it - t - 1, 0), m_a - 1)]; a = a < 4u ? a : 4u; }
            if (!RAGGED || m_b > 0) { b = qb[min(max(it - t - 1, 0), m_b - 1)]; b = b < 4u ? b : 4u; }
            return (0x4000u | a) | ((0x4000u | b) << 16);
        };
        unsigned q_cur = q_at(1), q_nxt = q_at(2);
        const int it_end = mm_w + P - 1;
        for (int it = 1; it <= it_end; ++it) {
            const unsigned q_nn = q_at(it + 2);
            const int r = it - t;
            unsigned out_al = all, out_fp = fpl;
            if (r >= 1 && r <= mm) {
                const __half2 qh = *reinterpret_cast<const __half2*>(&q_cur);
                unsigned ad = al_diag, fl = fpl, al = all;
                uint32_t wa[NW], wb[NW];
#pragma unroll
                for (int w8 = 0; w8 < NW; ++w8) {
                    uint32_t wd_a = 0u, wm_a = 0u, we_a = 0u, wf_a = 0u, wd_b = 0u, wm_b = 0u, we_b = 0u, wf_b = 0u;
                    uint32_t ws_a = 0u, ws_b = 0u;   // local: "H == 0" plane, folded into the two origin planes below
#pragma unroll
                    for (int c8 = 0; c8 < 8; ++c8) {
                        const int c = w8 * 8 + c8;
                        const unsigned eq = __heq2_mask(qh, *reinterpret_cast<const __half2*>(&ss[c]));
                        const unsigned d = __vadd2(ad, (eq & hit2) | (~eq & miss2));   // one LOP3 selects per half
                        ad = AL[c];
                        unsigned e = AL[c], f = al;   // linear gaps: E = H(up) - alpha, F = H(left) - alpha, no extension planes
                        if (AFFINE) {
                            e = max_mark2<kMarkE>(EP[c], AL[c], we_a, we_b, 1u << (16 + c8), one);
                            f = max_mark2<false>(fl, al, wf_a, wf_b, 1u << (24 + c8), one);
                            EP[c] = sub_cost<(kFmaAdds & 1) != 0>(e, cb32, nb2, one);
                            fl = sub_cost<(kFmaAdds & 2) != 0>(f, cb32, nb2, one);
                        }
                        const unsigned m1 = max_mark2<false>(d, e, wd_a, wd_b, 1u << c8, one);
                        unsigned h = max_mark2<false>(m1, f, wm_a, wm_b, 1u << (8 + c8), one);
                        if (LOCAL) h = max_mark2<false>(zero2, h, ws_a, ws_b, 1u << c8, one);   // 0 wins ties: stop iff H <= 0
                        al = sub_cost<(kFmaAdds & 4) != 0>(h, ca32, na2, one);
                        AL[c] = al;
                    }
                    if (LOCAL) {   // stop = "F wins" with the diagonal bit set (tb_code_at): pd = (pd && pm) || stop, pm = pm && !stop
                        wd_a = (wd_a & (wm_a >> 8)) | ws_a; wm_a &= ~(ws_a << 8);
                        wd_b = (wd_b & (wm_b >> 8)) | ws_b; wm_b &= ~(ws_b << 8);
                    }
                    wa[w8] = (wd_a | wm_a) | (we_a | wf_a);
                    wb[w8] = (wd_b | wm_b) | (we_b | wf_b);
                }
                // lane-major layout (tb_code_index): the words of four consecutive iterations are parked in shared memory and
                // leave as one granule (see the flush at the loop bottom)
                if constexpr (NW == 2) {
                    stage[0][(it - 1) & 3][tid] = make_uint2(wa[0], wa[1]);
                    stage[1][(it - 1) & 3][tid] = make_uint2(wb[0], wb[1]);
                } else if constexpr (NW == 4) {
                    stage[0][(it - 1) & 3][tid] = make_uint4(wa[0], wa[1], wa[2], wa[NW - 1]);
                    stage[1][(it - 1) & 3][tid] = make_uint4(wb[0], wb[1], wb[2], wb[NW - 1]);
                } else {
                    stage[0][(it - 1) & 3][tid] = make_uint3(wa[0], wa[1], wa[NW - 1]);
                    stage[1][(it - 1) & 3][tid] = make_uint3(wb[0], wb[1], wb[NW - 1]);
                }
                out_al = al;
                out_fp = fl;
                if (ATYPE == AT_SEMI && !RAGGED) {   // last matrix column, rows above the last one (only the owner lane's result counts)
                    const unsigned hv = r < mm ? pick_reg<K>(AL, cap_u) : col_best;
                    unsigned nb;
                    asm("{\n\t.reg .pred pl, ph;\n\t.reg .s16 r0, r1, a0, a1;\n\t"
                        "max.s16x2 %0, %3, %4;\n\t"
                        "mov.b32 {r0, r1}, %0;\n\t"
                        "mov.b32 {a0, a1}, %3;\n\t"
                        "setp.eq.s16 pl, r0, a0;\n\t"
                        "setp.eq.s16 ph, r1, a1;\n\t"
                        "@!pl mov.b32 %1, %5;\n\t"
                        "@!ph mov.b32 %2, %5;\n\t"
                        "}" : "=&r"(nb), "+r"(col_i_a), "+r"(col_i_b) : "r"(col_best), "r"(hv), "r"(r));
                    col_best = nb;
                } else if (ATYPE == AT_SEMI) {
                    if (has_cap_a && r < m_a) {
                        const int v = lo16(pick_reg<K>(AL, cap_a)) + alpha;
                        if (better_cell(v, r, n_a, bv_a, bi_a, bj_a)) { bv_a = v; bi_a = r; bj_a = n_a; }
                    }
                    if (has_cap_b && r < m_b) {
                        const int v = hi16(pick_reg<K>(AL, cap_b)) + alpha;
                        if (better_cell(v, r, n_b, bv_b, bi_b, bj_b)) { bv_b = v; bi_b = r; bj_b = n_b; }
                    }
                }
                if (RAGGED && !LOCAL) {   // the shorter half of a unit finishes before the registers reach row max(m)
                    if (r == m_a && m_a < mm) last_row(false, m_a, n_a, has_cap_a, cap_a, bv_a, bi_a, bj_a);
                    if (r == m_b && m_b < mm) last_row(true, m_b, n_b, has_cap_b, cap_b, bv_b, bi_b, bj_b);
                }
            }
            unsigned nal = __shfl_up_sync(0xffffffffu, out_al, 1, P);
            unsigned nfp = __shfl_up_sync(0xffffffffu, out_fp, 1, P);
            al_diag = all;
            if (t == 0) {
                if (GLOBAL_EDGES) edge -= beta;
                nal = pk16b(edge - alpha); nfp = neg2;
            }
            all = nal; fpl = nfp;
            if (r == 0) al_diag = al_top;
            q_cur = q_nxt; q_nxt = q_nn;
            if (((it - 1) & 3) == 3 || it == it_end) {   // a granule of four iterations is complete (or the sweep ends)
                const int g4 = (it - 1) & ~3;
                // equal-sized pairs: no guards -- an odd tail's second half and a group without a unit of its own recompute an
                // existing alignment and store the same words to the same place; rows outside the matrix leave stale words
                // that no walk reads
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const bool keep = v ? keep_b : keep_a;
                    const int rows4 = v ? rows4_b : rows4_a;
                    if (RAGGED && (!keep || g4 >= rows4)) continue;
                    uint32_t* dst = (v ? code_b : code_a) + ((int64_t)t * rows4 + g4) * NW;
                    uint32_t g[4 * NW];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const StageVec sv = stage[v][k][tid];
                        g[k * NW] = sv.x; g[k * NW + 1] = sv.y;
                        if constexpr (NW >= 3) g[k * NW + 2] = sv.z;
                        if constexpr (NW == 4) g[k * NW + 3] = reinterpret_cast<const uint4&>(sv).w;
                    }
#pragma unroll
                    for (int x = 0; x < NW; ++x)
                        reinterpret_cast<uint4*>(dst)[x] = make_uint4(g[4 * x], g[4 * x + 1], g[4 * x + 2], g[4 * x + 3]);
                }
            }
        }
        // every lane's registers now hold row max(m) of its strip
        if (LOCAL) { __syncwarp(); continue; }
        if (ATYPE == AT_SEMI && !RAGGED) {
            if (has_cap_a) { const int v = lo16(col_best) + alpha; if (better_cell(v, col_i_a, n_a, bv_a, bi_a, bj_a)) { bv_a = v; bi_a = col_i_a; bj_a = n_a; } }
            if (has_cap_b) { const int v = hi16(col_best) + alpha; if (better_cell(v, col_i_b, n_b, bv_b, bi_b, bj_b)) { bv_b = v; bi_b = col_i_b; bj_b = n_b; } }
        }
        if (m_a == mm && m_a > 0) last_row(false, m_a, n_a, has_cap_a, cap_a, bv_a, bi_a, bj_a);
        if (m_b == mm && m_b > 0) last_row(true, m_b, n_b, has_cap_b, cap_b, bv_b, bi_b, bj_b);
        const unsigned gmask = group_mask<P>(tid & 31);
#pragma unroll
        for (int off = P / 2; off >= 1; off >>= 1) {
            int ov = __shfl_xor_sync(gmask, bv_a, off, P), oi = __shfl_xor_sync(gmask, bi_a, off, P), oj = __shfl_xor_sync(gmask, bj_a, off, P);
            if (better_cell(ov, oi, oj, bv_a, bi_a, bj_a)) { bv_a = ov; bi_a = oi; bj_a = oj; }
            ov = __shfl_xor_sync(gmask, bv_b, off, P); oi = __shfl_xor_sync(gmask, bi_b, off, P); oj = __shfl_xor_sync(gmask, bj_b, off, P);
            if (better_cell(ov, oi, oj, bv_b, bi_b, bj_b)) { bv_b = ov; bi_b = oi; bj_b = oj; }
        }
        if (t == 0) {
            if (keep_a) { prm.w_score[pa] = bv_a; prm.w_i[pa] = bi_a; prm.w_j[pa] = bj_a; }
            if (keep_b) { prm.w_score[pb] = bv_b; prm.w_i[pb] = bi_b; prm.w_j[pb] = bj_b; }
        }
        __syncwarp();
    }
}

}  // namespace wsb
