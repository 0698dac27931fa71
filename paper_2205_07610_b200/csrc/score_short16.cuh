// score_short16.cuh -- packed int16x2 (DPX) LOCAL scoring of short reads that fit one stage: the headline kernel.
//
// Same lane-group wavefront, two alignments per register and two rows per trip as score_short.cuh, but in 16-bit
// integers with the DPX packed instructions instead of half2 arithmetic (the reference's own packed mode is int16
// halves, _kernels.py:553-858).  What that buys:
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
// Loop shape: ONE row per loop trip, lane t one row behind lane t - 1 (half the wavefront ramp of the two-rows-per-trip
// half2 kernel: 157 instead of 164 row steps for 150 bp).  All per-column state is updated in place by the instruction
// that produces it, so the trip carries no register copies: TA = T - alpha and TG = T - gamma are written by their
// VIADD, and instead of an H row the strip keeps D[c] = H(row, c - 1) + sigma(next row's symbol, c), the diagonal
// candidate of the NEXT row, written by the VIADD that follows the cell's VIMNMX3 (the PRMT takes the next row's row
// words, which are fetched one trip ahead anyway).  Per trip of K = 19 columns: 19 PRMT + 58 VIADD + 46 VIMNMX3 + the
// row hand-over (3 SHFL, 3 SEL) + the record (1 VIMNMX.S16x2 with predicates + 10 predicated STS.128) = 155 SASS
// instructions = 8.2 per packed cell pair (the half2 kernel: 336 per two rows = 8.8, on a ramp twice as long).
// End-cell snapshot: the record test is the packed maximum itself (VIMNMX.S16x2 returns max(best, rowmax) AND one
// predicate per half, "best won"); a half whose maximum rose parks the strip's T - gamma row -- whole 16-byte quads that never
// move -- in shared memory.  T == S <=> H == S for the global maximum S as long as gamma >= 1 (T is max(H, a gap state
// that lost at least gamma against an earlier T <= S)), so after the sweep the winner finds the first column with
// T - gamma == S - gamma; schemes with a zero-cost gap step take the half2 kernel.
//
// Unit pipeline: while a lane group sweeps unit u, the sequences of unit u + 1 travel from global to shared memory with
// cp.async (16-byte chunks of the aligned windows around the four sequences); their metadata chain (unit list -> pair
// -> offsets / lengths) advances one dependent load per quarter of the sweep, so no warp ever waits for global memory
// between two units.
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

template <int P> __host__ __device__ constexpr int short16_qrows() { return (kShort16MaxM + 2 * P + 2 + 1) / 2 * 2; }   // + P pad rows above, P + 2 below
constexpr int kShort16Raw = 192;     // bytes of one staged sequence window (16-byte aligned start, up to 177 symbols)
constexpr int kShort16MaxLen = kShort16Raw - 15;

template <int P, int K> constexpr size_t short16_smem_bytes() {
    return (size_t)2 * (K / 4 + 1) * kThreads * 16          // row snapshots, one area per packed half
           + (size_t)(kThreads / P) * short16_qrows<P>() * 8     // row words of the current unit
           + (size_t)(kThreads / P) * 4 * kShort16Raw       // staged sequences of the next unit
           + (size_t)(kThreads / P) * 16 * 4;               // metadata of the next unit
}

__device__ __forceinline__ unsigned pack16(int x) { return ((unsigned)x & 0xffffu) * 0x10001u; }
__device__ __forceinline__ int half16(unsigned w, int v) { return (int)(short)(v ? (w >> 16) : (w & 0xffffu)); }

// nb = max(best, rm) per half; a half whose maximum rose (best lost) parks the strip's H row: 16-byte chunks, one chunk
// every kThreads * 16 = 2048 bytes, in that half's snapshot area.  Stores are predicated, a row without a record costs
// issue slots only.  ptxas folds max + unpack + setp into ONE VIMNMX.S16x2 with two predicate results.
#define WSB_S16_HEAD                                                    \
    "{\n\t.reg .pred p, q;\n\t.reg .s16 r0, r1, a0, a1;\n\t"            \
    "max.s16x2 %0, %1, %2;\n\t"                                         \
    "mov.b32 {r0, r1}, %0;\n\t"                                         \
    "mov.b32 {a0, a1}, %1;\n\t"                                         \
    "setp.eq.s16 p, r0, a0;\n\t"                                        \
    "setp.eq.s16 q, r1, a1;\n\t"
#define WSB_S16_ST(off, a, b, c_, d)                                                   \
    "@!p st.shared.v4.b32 [%3+" #off "], {%" #a ", %" #b ", %" #c_ ", %" #d "};\n\t"   \
    "@!q st.shared.v4.b32 [%4+" #off "], {%" #a ", %" #b ", %" #c_ ", %" #d "};\n\t"

template <int NCH>
__device__ __forceinline__ unsigned record16(const unsigned (&w)[NCH * 4], unsigned best, unsigned rm, unsigned addr_p,
                                             unsigned addr_q) {
    static_assert(NCH >= 3 && NCH <= 5, "instantiated strip widths: K = 8..19");
    unsigned nb;
    if constexpr (NCH == 3) {
        asm volatile(WSB_S16_HEAD WSB_S16_ST(0, 5, 6, 7, 8) WSB_S16_ST(2048, 9, 10, 11, 12) WSB_S16_ST(4096, 13, 14, 15, 16) "}\n"
                     : "=&r"(nb)
                     : "r"(best), "r"(rm), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]),
                       "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11])
                     : "memory");
    }
    if constexpr (NCH == 4) {
        asm volatile(WSB_S16_HEAD WSB_S16_ST(0, 5, 6, 7, 8) WSB_S16_ST(2048, 9, 10, 11, 12) WSB_S16_ST(4096, 13, 14, 15, 16)
                     WSB_S16_ST(6144, 17, 18, 19, 20) "}\n"
                     : "=&r"(nb)
                     : "r"(best), "r"(rm), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]),
                       "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]),
                       "r"(w[14]), "r"(w[15])
                     : "memory");
    }
    if constexpr (NCH == 5) {
        asm volatile(WSB_S16_HEAD WSB_S16_ST(0, 5, 6, 7, 8) WSB_S16_ST(2048, 9, 10, 11, 12) WSB_S16_ST(4096, 13, 14, 15, 16)
                     WSB_S16_ST(6144, 17, 18, 19, 20) WSB_S16_ST(8192, 21, 22, 23, 24) "}\n"
                     : "=&r"(nb)
                     : "r"(best), "r"(rm), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]),
                       "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]),
                       "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19])
                     : "memory");
    }
    return nb;
}

__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// PRMT selectors of a strip of K columns for the two alignments of a unit, four columns at a time: the subject bytes come
// in as aligned 32-bit words of the staged windows (funnel-shifted to the strip's first column), every byte x < 4 becomes
// the selector byte x' * 0x11 + 0x80 (low nibble: value byte x' of the row words, high nibble: its sign fill; x' = x for
// the first alignment, x + 4 for the second) with ONE multiply-add per word; columns beyond the subject get 0x88 (sign
// fill of byte 0 in both nibbles: sigma in {0, -1}, never improving).  Returns true when a column inside a subject holds a
// flagged symbol (no selector encoding).  ~150 instructions per strip where the byte-by-byte form took ~520, most of them
// waiting for one-byte shared-memory loads.
template <int K>
__device__ __forceinline__ bool build_selectors16(const uint8_t* win_a, const uint8_t* win_b, int pos_a, int pos_b, int left_a,
                                                  int left_b, unsigned (&sel)[K]) {
    constexpr int NWD = (K + 3) / 4;
    unsigned nibs[2][NWD];
    unsigned fl = 0u;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
        const uint8_t* win = v ? win_b : win_a;
        const int pos = v ? pos_b : pos_a, left = v ? left_b : left_a;   // window byte of the strip's first column; columns left in the subject
        const unsigned* words = reinterpret_cast<const unsigned*>(win) + (pos >> 2);
        const unsigned sh = 8u * (unsigned)(pos & 3);
        unsigned w[NWD + 1];
#pragma unroll
        for (int k = 0; k <= NWD; ++k) w[k] = words[k];
#pragma unroll
        for (int k = 0; k < NWD; ++k) {
            const unsigned x = __funnelshift_r(w[k], w[k + 1], sh);
            const int valid = min(max(left - 4 * k, 0), 4);
            const unsigned mask = valid >= 4 ? 0xffffffffu : ((1u << (8 * valid)) - 1u);
            fl |= x & mask;
            const unsigned xm = x & mask & 0x03030303u;
            const unsigned base = 0x80808080u | (~mask & 0x08080808u) | (v ? (mask & 0x04040404u) * 0x11u : 0u);
            nibs[v][k] = xm * 0x11u + base;
        }
    }
#pragma unroll
    for (int c = 0; c < K; ++c)   // byte c of either word; the consumer PRMT reads the low 16 bits only
        sel[c] = __byte_perm(nibs[0][c >> 2], nibs[1][c >> 2], (unsigned)(c & 3) | ((4u + (unsigned)(c & 3)) << 4));
    return (fl & 0xfcfcfcfcu) != 0u;
}

// AIMM / GIMM > 0: gap costs alpha / gamma baked into the instruction stream as immediates (the host picks such an
// instantiation when the scheme matches): a VIADD.16x2 with an immediate reads one register instead of two, which the
// cell-stream microbenchmark (tools/ubench/cell_bench.cu) shows is worth ~6 % of issue rate at four warps per scheduler.
template <int P, int K, int GAP, int MINB = 4, int AIMM = 0, int GIMM = 0>
__global__ void __launch_bounds__(kThreads, MINB) s16_local_short_kernel(const ScoreParams prm) {
    constexpr int GPB = kThreads / P;
    constexpr int NCH = K / 4 + 1;   // always at least one spare word after the K columns: it takes the row tag
    constexpr int NW = NCH * 4;
    static_assert(P >= 4, "lanes 0..3 of a group carry the metadata of the four sequences of a unit");
    extern __shared__ uint4 smem_dyn[];
    uint4 (*snap)[NCH][kThreads] = reinterpret_cast<uint4 (*)[NCH][kThreads]>(smem_dyn);
    constexpr int QROWS = short16_qrows<P>();
    uint2 (*qbuf)[QROWS] = reinterpret_cast<uint2 (*)[QROWS]>(smem_dyn + 2 * NCH * kThreads);
    uint8_t (*raw)[4][kShort16Raw] = reinterpret_cast<uint8_t (*)[4][kShort16Raw]>(&qbuf[GPB][0]);
    int (*meta)[16] = reinterpret_cast<int (*)[16]>(&raw[GPB][0][0]);   // per group: pidx[2], len[4], shift[4]

    const long long cycles_at_start = prm.block_cycles ? clock64() : 0;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int t = tid & (P - 1);
    const int gib = tid / P;
    const unsigned gmask = group_mask<P>(lane);
    const int64_t group_global = (int64_t)blockIdx.x * GPB + gib;
    const int64_t n_groups = (int64_t)gridDim.x * GPB;
    const unsigned snap_addr = (unsigned)__cvta_generic_to_shared(&snap[0][0][tid]);
    constexpr unsigned HS = NCH * kThreads * 16;  // byte distance between the two halves' snapshot areas

    const int gamma = GIMM > 0 ? GIMM : (GAP == GAP_MERGED ? min(prm.alpha, prm.beta) : prm.alpha);
    const unsigned c_nalpha = AIMM > 0 ? ((unsigned)(-AIMM) & 0xffffu) * 0x10001u : pack16(-prm.alpha);
    const unsigned c_ngamma = GIMM > 0 ? ((unsigned)(-GIMM) & 0xffffu) * 0x10001u : pack16(-gamma);
    const unsigned mism4 = (unsigned)(prm.mismatch & 0xff) * 0x01010101u;
    const unsigned dm1 = (unsigned)((prm.match ^ prm.mismatch) & 0xff);
    // lane 0 sees the matrix' zero left border instead of a neighbour: x * keep (IMAD, FMA pipe).  0 stands for every
    // border value: H = 0 exactly, and T = 0 gives T - alpha, T - gamma <= 0, which never win against the local floor.
    const unsigned keep = t == 0 ? 0u : (unsigned)prm.one;   // prm.one == 1, opaque: keeps the selects multiplies (FMA pipe)
    const int col0 = t * K;

    // ---- metadata chain of a unit, one dependent load per step; lane v (< 4) follows sequence v: 0 = query of pair 0,
    // 1 = subject of pair 0, 2 = query of pair 1, 3 = subject of pair 1
    const int64_t rounds = (prm.n_units + n_groups - 1) / n_groups;
    const int sv = t & 3, pv = sv >> 1;
    const bool is_subject = (sv & 1) != 0;
    int mt_p = -1, mt_seq = 0, mt_len = 0;
    const uint8_t* mt_ptr = nullptr;
    auto meta_step = [&](int step, int64_t u) {
        if (step == 0) {          // unit -> pair
            mt_p = -1;
            if (u < prm.n_units) {
                if (prm.units) mt_p = prm.units[u * 2 + pv];
                else { const int64_t pp = prm.pair_base + u * 2 + pv; mt_p = pp < prm.n_pairs ? (int)pp : -1; }
            }
        } else if (step == 1) {   // pair -> sequence
            mt_seq = mt_p >= 0 ? (is_subject ? prm.pair_s[mt_p] : prm.pair_q[mt_p]) : 0;
        } else if (step == 2) {   // sequence -> window
            mt_len = 0; mt_ptr = is_subject ? prm.s_codes : prm.q_codes;
            if (mt_p >= 0) {
                mt_len = is_subject ? prm.s_len[mt_seq] : prm.q_len[mt_seq];
                mt_ptr += is_subject ? prm.s_off[mt_seq] : prm.q_off[mt_seq];
            }
        } else {                  // window -> shared memory; the metadata the sweep needs goes to the group's slot
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

    // prologue: the first unit of this group goes through the whole chain at once
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
        if (mm_w == 0) {   // nothing to sweep in this warp: still keep the pipeline of the next unit going
            __syncwarp();
            if (rd + 1 < rounds) {
#pragma unroll
                for (int step = 0; step < 4; ++step) meta_step(step, u_next);
            }
            continue;
        }

        // query buffer: P pad rows, the rows of both queries as row words, then pad rows for the ramp-down.  The byte
        // loads of four rows are in flight before the first is used.
#ifndef WSB_ABL_NOQBUF     // timing experiment only
        {
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
                    uint2 rw;   // sigma(q, s) for s = 0..3: match in the byte of the query symbol, mismatch elsewhere
                    rw.x = c0[k] < 4 ? mism4 ^ (dm1 << (8 * c0[k])) : mism4;
                    rw.y = c1[k] < 4 ? mism4 ^ (dm1 << (8 * c1[k])) : mism4;
                    if (x0 + P * k < total) qbuf[gib][x0 + P * k] = rw;
                }
            }
        }
#endif
        // per column: PRMT selector of the two subject symbols, TA = T - alpha (whole quads: the snapshot source), TG = T - gamma,
        // D = diagonal candidate of the NEXT row (H of the column to the left + sigma of the next row's symbol)
        unsigned sel[K], TA[GAP == GAP_MERGED ? K : NW], TG[GAP == GAP_MERGED ? NW : 1], D[K];   // the snapshot source holds whole quads
        D[0] = 0u;
#ifdef WSB_ABL_NOSEL       // timing experiment only
        bool flagged_subject = false;
#pragma unroll
        for (int c = 0; c < K; ++c) sel[c] = 0x9180u + (unsigned)(ssh[0] + c);
#else
        const bool flagged_subject = build_selectors16<K>(raw[gib][1], raw[gib][3], ssh[0] + col0, ssh[1] + col0, n[0] - col0,
                                                          n[1] - col0, sel);
#endif
#pragma unroll
        for (int c = 0; c < K; ++c) {
            TA[c] = c_nalpha;
            if (GAP == GAP_MERGED) TG[c] = c_ngamma;
        }
#pragma unroll
        for (int c = K; c < NW; ++c) { if (GAP == GAP_MERGED) TG[c] = 0u; else TA[c] = 0u; }
        // a flagged subject symbol cannot be encoded: hand the pair(s) of this unit to the fallback list
        if (__any_sync(gmask, flagged_subject)) {
            if (t == 0) {
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (pidx[v] >= 0) { const int at = atomicAdd(prm.redo_count, 1); prm.redo[at] = pidx[v]; }
            }
        }
        __syncwarp();   // raw[] and meta[] of this unit are consumed, qbuf is complete
        {   // candidates of the first row this lane sweeps: H of the row above it is zero
            const uint2 rw = qbuf[gib][P - t];
#pragma unroll
            for (int c = 1; c < K; ++c) asm("prmt.b32 %0, %1, %2, %3;" : "=r"(D[c]) : "r"(rw.x), "r"(rw.y), "r"(sel[c]));
        }

        unsigned ta_l = 0u, tg_l = 0u;     // left border of the coming row: T - alpha, T - gamma
        unsigned h_l = 0u, h_d = 0u;       // H of the left column in the coming row's row / in the row above it (diagonal)
        unsigned bestvec = 0u;
        const unsigned qbase = (unsigned)__cvta_generic_to_shared(&qbuf[gib][0]);
        unsigned qaddr = qbase + 8u * (unsigned)(P - t);    // row r lives at qbuf index r - 1 + P; lane t runs t rows behind lane 0

        // one row of the strip.  rw0/rw1: row words of this row (cell 0's candidate), nw0/nw1: of the next row
        auto row = [&](unsigned rw0, unsigned rw1, unsigned nw0, unsigned nw1, unsigned h_diag, unsigned& la, unsigned& lg,
                       unsigned& rm, unsigned& h_last, unsigned& t_last) {
            rm = 0u;
            unsigned hprev = 0u;
#pragma unroll
            for (int c = 0; c < K; ++c) {
                unsigned d;
                if (c == 0) {
                    unsigned sg;
                    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(sg) : "r"(rw0), "r"(rw1), "r"(sel[0]));
                    d = __vadd2(h_diag, sg);
                } else d = D[c];
                const unsigned h = __vimax3_s16x2_relu(TA[c], la, d);
                if (GAP == GAP_MERGED) {
                    const unsigned tn = __vimax3_s16x2_relu(TG[c], lg, d);
                    if (c == K - 1) t_last = tn;
                    la = __vadd2(tn, c_nalpha);
                    lg = __vadd2(tn, c_ngamma);
                    TG[c] = lg;
                } else {
                    la = __vadd2(h, c_nalpha);
                    if (c == K - 1) t_last = h;
                }
                TA[c] = la;
                if (c >= 1) {   // this column's candidate for the NEXT row, in place: its old value was consumed just above
                    unsigned sg;
                    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(sg) : "r"(nw0), "r"(nw1), "r"(sel[c]));
                    D[c] = __vadd2(hprev, sg);
                }
                if (c & 1) rm = __vimax3_s16x2(rm, hprev, h);
                else if (c == K - 1) rm = __vmaxs2(rm, h);
                hprev = h;
            }
            h_last = hprev;
        };
        // The right border leaves for the next lane right after the row's last cell (send) and is taken over at the top
        // of the NEXT trip (receive): the loop branch keeps the two apart, so the record stores, the row-word loads and the
        // loop bookkeeping run under the shuffle latency instead of behind it.
        unsigned s_t = 0u, s_h = 0u;
        auto send = [&](unsigned t_last, unsigned h_last) {
#ifdef WSB_ABLATE_SHFL     // timing experiment only (wrong results): the lane feeds itself
            s_t = t_last; s_h = h_last;
#else
            s_t = __shfl_up_sync(0xffffffffu, t_last, 1, P);
            s_h = __shfl_up_sync(0xffffffffu, h_last, 1, P);
#endif
        };
        auto receive = [&]() {   // two multiplies and two packed adds on the FMA pipe; the ALU pipe is the busy one
            h_d = h_l;
            const unsigned t_in = s_t * keep;
            ta_l = __vadd2(t_in, c_nalpha);
            if (GAP == GAP_MERGED) tg_l = __vadd2(t_in, c_ngamma);
            h_l = s_h * keep;
        };

        unsigned qn0, qn1, qc0, qc1;  // row words of the coming row and the one after it
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(qc0), "=r"(qc1) : "r"(qaddr) : "memory");
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2+8];" : "=r"(qn0), "=r"(qn1) : "r"(qaddr) : "memory");
        int done = 0;
        const int steps = mm_w + P - 1;
        const int quarter1 = (steps + 3) / 4;
#pragma unroll 1
        for (int part = 0; part < 4; ++part) {
            if (rd + 1 < rounds) meta_step(part, u_next);
            const unsigned qstop = qaddr + 8u * (unsigned)max(0, min(quarter1, steps - done));
            done += quarter1;
#ifdef WSB_S16_UNROLL2
#pragma unroll 2
#else
#pragma unroll 1
#endif
            while (qaddr != qstop) {
                receive();
                unsigned la = ta_l, lg = tg_l, rm, h_last, t_last;
                row(qc0, qc1, qn0, qn1, h_d, la, lg, rm, h_last, t_last);
                // The address register is bumped BEFORE the loads that read it: bumped behind them (at the loop end) the add
                // has to wait until the loads, queued in the memory pipe behind other warps' stores, have read the register
                // -- 14 % of all stall samples of the kernel sat on that add (profiles/r02_ncu_s16_local_short_before.md).
                qaddr += 8;
                asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(qc0), "=r"(qc1) : "r"(qaddr) : "memory");
                asm volatile("ld.shared.v2.b32 {%0, %1}, [%2+8];" : "=r"(qn0), "=r"(qn1) : "r"(qaddr) : "memory");
#ifdef WSB_S16_SEND_FIRST
                send(t_last, h_last);
#endif
                // the row that just finished: T - gamma of the strip (linear gaps: h - alpha, the same thing) plus the row tag
#ifdef WSB_S16_NOREC      // timing experiment only (end cells wrong)
                bestvec = __vmaxs2(bestvec, rm);
#else
                if constexpr (GAP == GAP_MERGED) {
                    TG[K] = qaddr;
                    bestvec = record16<NCH>(TG, bestvec, rm, snap_addr, snap_addr + HS);
                } else {
                    TA[K] = qaddr;
                    bestvec = record16<NCH>(TA, bestvec, rm, snap_addr, snap_addr + HS);
                }
#endif
#ifndef WSB_S16_SEND_FIRST
                send(t_last, h_last);
#endif
            }
        }

        // reduce over the group: max value, then smallest row, then smallest strip; the winner resolves its column
#ifdef WSB_ABL_NOFIN       // timing experiment only
        if (t == 0 && pidx[0] >= 0) prm.out_score[pidx[0]] = (int)bestvec;
#else
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            int bv = half16(bestvec, v);
            int bi = 0, bj = col0, who = t;
            if (bv > 0) {  // the tag word after the K columns holds the query-buffer address of the record row
                const uint4 w = snap[v][K / 4][tid];
                const unsigned tag = (K % 4 == 0) ? w.x : (K % 4 == 1) ? w.y : (K % 4 == 2) ? w.z : w.w;
                bi = (int)((tag - qbase) >> 3) - P;      // the tag is the buffer address of the row AFTER the recorded one
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
                        if (4 * ch + 3 < K && half16(w.w, v) == bv - gamma) pos = 4 * ch + 3;
                        if (4 * ch + 2 < K && half16(w.z, v) == bv - gamma) pos = 4 * ch + 2;
                        if (4 * ch + 1 < K && half16(w.y, v) == bv - gamma) pos = 4 * ch + 1;
                        if (half16(w.x, v) == bv - gamma) pos = 4 * ch;
                    }
                    j = bj + pos + 1;
                } else { bi = 0; }
                prm.out_score[pidx[v]] = bv;
                prm.out_i[pidx[v]] = bi;
                prm.out_j[pidx[v]] = j;
            }
        }
#endif
    }
    // cycle-based roofline fraction: a resident block lives as long as the launch, so the largest value is the
    // launch's duration in cycles of the SM it ran on
    if (prm.block_cycles && tid == 0) prm.block_cycles[blockIdx.x] = (unsigned long long)(clock64() - cycles_at_start);
}

}  // namespace wsb
