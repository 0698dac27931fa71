// score_short.cuh -- the hot kernel: packed half2 LOCAL scoring of short reads that fit one stage.
//
// Same lane-group wavefront as score_kernels.cuh (lane t owns K columns, row r = it - t at iteration it, two
// independent alignments in the halves of every register) but specialised for the case that carries the headline
// benchmark (150 bp / 250 bp reads, local alignment): the whole subject fits P*K columns, the whole query fits the
// shared-memory query buffer, and the 0 floor of local alignment makes the edge state a fixed point, so
//   * there is no stage loop, no border scratch, no ring refill;
//   * no lane ever idles or branches on "is my row inside the matrix": rows above row 1 and below row m are computed
//     with a never-matching pad symbol, which keeps the all-zero edge state unchanged above the matrix and cannot
//     produce a record below it (pads only lose score: mismatch <= 0, gaps cost >= 0 -- checked by the planner);
//   * the per-row work beside the K cell updates is: one shared-memory load (query symbols), two shuffles, the
//     record test and its predicated snapshot stores.
//
// Cell update, per packed pair of cells (reference semantics: _kernels.py:259-276 merged affine, :113-126 linear):
//     eq = (q == s)                      HSET2.BF.EQ      ALU
//     d  = max(hm_diag + delta*eq, 0)    HFMA2.RELU       FMA      hm = h + mismatch, so this is H_diag + sigma
//     g  = max(T_up, T_left)             HMNMX2           ALU
//     h  = max(g - alpha, d)             HADD2 + HMNMX2   FMA+ALU
//     T  = max(g - gamma, d)             HADD2 + HMNMX2   FMA+ALU  gamma = min(alpha, beta)   (linear: T = h)
//     hm = h + mismatch                  HADD2            FMA
//     rm = max(rm, h)                    VHMNMX per 2     ALU
#pragma once
#include "score_kernels.cuh"

namespace wsb {

constexpr int kShortQRows = 324;  // query rows the short kernel can hold per lane group (>= 250 bp reads + P pads)

template <int P, int K> constexpr size_t short_smem_bytes() {
    return (size_t)2 * (K / 4 + 1) * kThreads * 16 + (size_t)(kThreads / P) * kShortQRows * 4;
}

__device__ __forceinline__ unsigned h2u(__half2 v) { return *reinterpret_cast<unsigned*>(&v); }
__device__ __forceinline__ __half2 u2h(unsigned v) { return *reinterpret_cast<__half2*>(&v); }

// Record test + snapshot for both halves: if rm.half > best.half, park the strip's hm row (16-byte chunks, one chunk
// every kThreads*16 = 2048 bytes) in that half's snapshot area and remember the iteration.  One SETP yields both
// predicates; the stores and the two moves are predicated, so a row without a record costs issue slots only.
static_assert(kThreads * 16 == 2048, "chunk stride is baked into the store offsets below");
template <int NC, bool REC>
__device__ __forceinline__ void record_chunks(const unsigned* w, unsigned rm, unsigned best, unsigned addr_p,
                                              unsigned addr_q, int it, int& rec0, int& rec1) {
    static_assert(NC >= 1 && NC <= 5, "chunk group size");
    if constexpr (NC == 1 && REC) {
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.gt.f16x2 p|q, %2, %3;\n\t"
            "@p st.shared.v4.b32 [%4+0], {%6, %7, %8, %9};\n\t"
            "@q st.shared.v4.b32 [%5+0], {%6, %7, %8, %9};\n\t"
            "@p mov.b32 %0, %10;\n\t"
            "@q mov.b32 %1, %10;\n\t"
            "}\n"
            : "+r"(rec0), "+r"(rec1)
            : "r"(rm), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(it)
            : "memory");
    }
    if constexpr (NC == 1 && !REC) {
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.gt.f16x2 p|q, %0, %1;\n\t"
            "@p st.shared.v4.b32 [%2+0], {%4, %5, %6, %7};\n\t"
            "@q st.shared.v4.b32 [%3+0], {%4, %5, %6, %7};\n\t"
            "}\n"
            : 
            : "r"(rm), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
            : "memory");
    }
    if constexpr (NC == 2 && REC) {
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.gt.f16x2 p|q, %2, %3;\n\t"
            "@p st.shared.v4.b32 [%4+0], {%6, %7, %8, %9};\n\t"
            "@q st.shared.v4.b32 [%5+0], {%6, %7, %8, %9};\n\t"
            "@p st.shared.v4.b32 [%4+2048], {%10, %11, %12, %13};\n\t"
            "@q st.shared.v4.b32 [%5+2048], {%10, %11, %12, %13};\n\t"
            "@p mov.b32 %0, %14;\n\t"
            "@q mov.b32 %1, %14;\n\t"
            "}\n"
            : "+r"(rec0), "+r"(rec1)
            : "r"(rm), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(it)
            : "memory");
    }
    if constexpr (NC == 2 && !REC) {
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.gt.f16x2 p|q, %0, %1;\n\t"
            "@p st.shared.v4.b32 [%2+0], {%4, %5, %6, %7};\n\t"
            "@q st.shared.v4.b32 [%3+0], {%4, %5, %6, %7};\n\t"
            "@p st.shared.v4.b32 [%2+2048], {%8, %9, %10, %11};\n\t"
            "@q st.shared.v4.b32 [%3+2048], {%8, %9, %10, %11};\n\t"
            "}\n"
            : 
            : "r"(rm), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
            : "memory");
    }
    if constexpr (NC == 3 && REC) {
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.gt.f16x2 p|q, %2, %3;\n\t"
            "@p st.shared.v4.b32 [%4+0], {%6, %7, %8, %9};\n\t"
            "@q st.shared.v4.b32 [%5+0], {%6, %7, %8, %9};\n\t"
            "@p st.shared.v4.b32 [%4+2048], {%10, %11, %12, %13};\n\t"
            "@q st.shared.v4.b32 [%5+2048], {%10, %11, %12, %13};\n\t"
            "@p st.shared.v4.b32 [%4+4096], {%14, %15, %16, %17};\n\t"
            "@q st.shared.v4.b32 [%5+4096], {%14, %15, %16, %17};\n\t"
            "@p mov.b32 %0, %18;\n\t"
            "@q mov.b32 %1, %18;\n\t"
            "}\n"
            : "+r"(rec0), "+r"(rec1)
            : "r"(rm), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(it)
            : "memory");
    }
    if constexpr (NC == 3 && !REC) {
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.gt.f16x2 p|q, %0, %1;\n\t"
            "@p st.shared.v4.b32 [%2+0], {%4, %5, %6, %7};\n\t"
            "@q st.shared.v4.b32 [%3+0], {%4, %5, %6, %7};\n\t"
            "@p st.shared.v4.b32 [%2+2048], {%8, %9, %10, %11};\n\t"
            "@q st.shared.v4.b32 [%3+2048], {%8, %9, %10, %11};\n\t"
            "@p st.shared.v4.b32 [%2+4096], {%12, %13, %14, %15};\n\t"
            "@q st.shared.v4.b32 [%3+4096], {%12, %13, %14, %15};\n\t"
            "}\n"
            : 
            : "r"(rm), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11])
            : "memory");
    }
    if constexpr (NC == 4 && REC) {
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.gt.f16x2 p|q, %2, %3;\n\t"
            "@p st.shared.v4.b32 [%4+0], {%6, %7, %8, %9};\n\t"
            "@q st.shared.v4.b32 [%5+0], {%6, %7, %8, %9};\n\t"
            "@p st.shared.v4.b32 [%4+2048], {%10, %11, %12, %13};\n\t"
            "@q st.shared.v4.b32 [%5+2048], {%10, %11, %12, %13};\n\t"
            "@p st.shared.v4.b32 [%4+4096], {%14, %15, %16, %17};\n\t"
            "@q st.shared.v4.b32 [%5+4096], {%14, %15, %16, %17};\n\t"
            "@p st.shared.v4.b32 [%4+6144], {%18, %19, %20, %21};\n\t"
            "@q st.shared.v4.b32 [%5+6144], {%18, %19, %20, %21};\n\t"
            "@p mov.b32 %0, %22;\n\t"
            "@q mov.b32 %1, %22;\n\t"
            "}\n"
            : "+r"(rec0), "+r"(rec1)
            : "r"(rm), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(it)
            : "memory");
    }
    if constexpr (NC == 4 && !REC) {
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.gt.f16x2 p|q, %0, %1;\n\t"
            "@p st.shared.v4.b32 [%2+0], {%4, %5, %6, %7};\n\t"
            "@q st.shared.v4.b32 [%3+0], {%4, %5, %6, %7};\n\t"
            "@p st.shared.v4.b32 [%2+2048], {%8, %9, %10, %11};\n\t"
            "@q st.shared.v4.b32 [%3+2048], {%8, %9, %10, %11};\n\t"
            "@p st.shared.v4.b32 [%2+4096], {%12, %13, %14, %15};\n\t"
            "@q st.shared.v4.b32 [%3+4096], {%12, %13, %14, %15};\n\t"
            "@p st.shared.v4.b32 [%2+6144], {%16, %17, %18, %19};\n\t"
            "@q st.shared.v4.b32 [%3+6144], {%16, %17, %18, %19};\n\t"
            "}\n"
            : 
            : "r"(rm), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
            : "memory");
    }
    if constexpr (NC == 5 && REC) {
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.gt.f16x2 p|q, %2, %3;\n\t"
            "@p st.shared.v4.b32 [%4+0], {%6, %7, %8, %9};\n\t"
            "@q st.shared.v4.b32 [%5+0], {%6, %7, %8, %9};\n\t"
            "@p st.shared.v4.b32 [%4+2048], {%10, %11, %12, %13};\n\t"
            "@q st.shared.v4.b32 [%5+2048], {%10, %11, %12, %13};\n\t"
            "@p st.shared.v4.b32 [%4+4096], {%14, %15, %16, %17};\n\t"
            "@q st.shared.v4.b32 [%5+4096], {%14, %15, %16, %17};\n\t"
            "@p st.shared.v4.b32 [%4+6144], {%18, %19, %20, %21};\n\t"
            "@q st.shared.v4.b32 [%5+6144], {%18, %19, %20, %21};\n\t"
            "@p st.shared.v4.b32 [%4+8192], {%22, %23, %24, %25};\n\t"
            "@q st.shared.v4.b32 [%5+8192], {%22, %23, %24, %25};\n\t"
            "@p mov.b32 %0, %26;\n\t"
            "@q mov.b32 %1, %26;\n\t"
            "}\n"
            : "+r"(rec0), "+r"(rec1)
            : "r"(rm), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(it)
            : "memory");
    }
    if constexpr (NC == 5 && !REC) {
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.gt.f16x2 p|q, %0, %1;\n\t"
            "@p st.shared.v4.b32 [%2+0], {%4, %5, %6, %7};\n\t"
            "@q st.shared.v4.b32 [%3+0], {%4, %5, %6, %7};\n\t"
            "@p st.shared.v4.b32 [%2+2048], {%8, %9, %10, %11};\n\t"
            "@q st.shared.v4.b32 [%3+2048], {%8, %9, %10, %11};\n\t"
            "@p st.shared.v4.b32 [%2+4096], {%12, %13, %14, %15};\n\t"
            "@q st.shared.v4.b32 [%3+4096], {%12, %13, %14, %15};\n\t"
            "@p st.shared.v4.b32 [%2+6144], {%16, %17, %18, %19};\n\t"
            "@q st.shared.v4.b32 [%3+6144], {%16, %17, %18, %19};\n\t"
            "@p st.shared.v4.b32 [%2+8192], {%20, %21, %22, %23};\n\t"
            "@q st.shared.v4.b32 [%3+8192], {%20, %21, %22, %23};\n\t"
            "}\n"
            : 
            : "r"(rm), "r"(best), "r"(addr_p), "r"(addr_q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19])
            : "memory");
    }
}

// hm[] row plus the iteration tag in the first spare word after the K columns (the snapshot then also records WHEN).
template <int K> __device__ __forceinline__ void record_rows(const __half2 (&hm)[K], __half2 rm, __half2 best,
                                                             unsigned snap_addr, unsigned tag) {
    constexpr int NCH = K / 4 + 1;  // always at least one spare word for the tag
    unsigned w[NCH * 4];
#pragma unroll
    for (int c = 0; c < NCH * 4; ++c) w[c] = c < K ? h2u(hm[c]) : tag;
    constexpr int FIRST = NCH < 5 ? NCH : 5;
    constexpr unsigned HS = NCH * kThreads * 16;  // byte distance between the two halves' snapshot areas
    int dummy0 = 0, dummy1 = 0;
    record_chunks<FIRST, false>(w, h2u(rm), h2u(best), snap_addr, snap_addr + HS, 0, dummy0, dummy1);
    if constexpr (NCH > 5) {
        constexpr int SECOND = NCH - 5 < 5 ? NCH - 5 : 5;
        record_chunks<SECOND, false>(w + 20, h2u(rm), h2u(best), snap_addr + 5 * 2048, snap_addr + HS + 5 * 2048, 0, dummy0, dummy1);
        static_assert(NCH <= 10, "strip too wide for the snapshot helper");
    }
}

// LISTED = true: re-score launch behind the packed int16 kernel (unit list and its length live on the device); kept
// out of the main instantiation so that the headline kernel's code is untouched by it
template <int P, int K, int GAP, bool LISTED = false>
#ifdef WSB_SHORT_MINB
__global__ void __launch_bounds__(kThreads, (K <= 20 ? WSB_SHORT_MINB : 1)) f16_local_short_kernel(const ScoreParams prm) {
#else
__global__ void __launch_bounds__(kThreads) f16_local_short_kernel(const ScoreParams prm) {
#endif
    using AR = ArF16;
    constexpr int GPB = kThreads / P;
    constexpr int NCH = K / 4 + 1;
    extern __shared__ uint4 smem_dyn[];
    uint4 (*snap)[NCH][kThreads] = reinterpret_cast<uint4 (*)[NCH][kThreads]>(smem_dyn);
    __half2 (*qbuf)[kShortQRows] = reinterpret_cast<__half2 (*)[kShortQRows]>(smem_dyn + 2 * NCH * kThreads);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int t = tid & (P - 1);
    const int gib = tid / P;
    const unsigned gmask = group_mask<P>(lane);
    const int64_t group_global = (int64_t)blockIdx.x * GPB + gib;
    const int64_t n_groups = (int64_t)gridDim.x * GPB;
    const unsigned snap_addr = (unsigned)__cvta_generic_to_shared(&snap[0][0][tid]);

    const int mism = prm.mismatch;
    const int gamma = min(prm.alpha, prm.beta);
    const __half2 c_delta = AR::splat(prm.match - prm.mismatch);
    const __half2 c_mism = AR::splat(mism);
    const __half2 c_nalpha = AR::splat(-prm.alpha);
    const __half2 c_ngamma = AR::splat(-gamma);
    const __half2 c_ndelta = AR::splat(gamma - prm.alpha);  // -(alpha - gamma)
    const __half2 c_zero = AR::splat(0);
    (void)c_ndelta;
    // lane 0 sees the matrix' zero left border instead of a neighbour: x * keep + edge on the FMA pipe
    const __half2 keep = AR::splat(t == 0 ? 0 : 1);
    (void)keep;
    const __half2 edge_ta = t == 0 ? c_nalpha : c_zero;  // (T - alpha) of the border, T = 0
    const __half2 edge_tg = t == 0 ? c_ngamma : c_zero;
    const __half2 edge_hm = t == 0 ? c_mism : c_zero;
    (void)edge_ta; (void)edge_tg; (void)edge_hm;
    const int col0 = t * K;

    // re-score launch behind the packed int16 kernel: the unit list and its length live on the device
    const int64_t listed = LISTED ? (int64_t)*prm.n_pairs_dev : 0;
    const int64_t n_units = LISTED ? (listed + 1) / 2 : prm.n_units;
    const int64_t rounds = (n_units + n_groups - 1) / n_groups;
    for (int64_t rd = 0; rd < rounds; ++rd) {
        const int64_t u = rd * n_groups + group_global;
        int pidx[2], m[2], n[2];
        const uint8_t* qp[2];
        const uint8_t* sp[2];
        int mm = 0;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            int p = -1;
            if (u < n_units) {
                if (LISTED) p = u * 2 + v < listed ? prm.units[u * 2 + v] : -1;
                else if (prm.units) p = prm.units[u * 2 + v];
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

        // query buffer: 2P pad rows, the rows of both queries, then pad rows for the ramp-down.  Loads are issued in
        // batches of 8 per lane before any is consumed, so a unit pays ~3 memory round trips here instead of ~23.
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
                    for (int v = 0; v < 2; ++v) raw[k][v] = (row >= 0 && row < m[v]) ? (int)qp[v][row] : kPadQuery;
                }
#pragma unroll
                for (int k = 0; k < UNR; ++k) {
                    const int x = x0 + P * k;
                    const int c0 = raw[k][0] < 4 || raw[k][0] == kPadQuery ? raw[k][0] : kFlagQuery;
                    const int c1 = raw[k][1] < 4 || raw[k][1] == kPadQuery ? raw[k][1] : kFlagQuery;
                    if (x < total) qbuf[gib][x] = AR::codes(c0, c1);
                }
            }
        }
        // per column: TA = T - alpha, TG = T - gamma (merged model; linear: both are h - alpha), HM = h + mismatch
        __half2 sc[K], TA[K], TG[GAP == GAP_MERGED ? K : 1], HM[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
            int code[2] = {kPadSubject, kPadSubject};
#pragma unroll
            for (int v = 0; v < 2; ++v)
                if (col0 + c < n[v]) { const int x = sp[v][col0 + c]; code[v] = x < 4 ? x : kFlagSubject; }
            sc[c] = AR::codes(code[0], code[1]);
            TA[c] = c_nalpha;
            if (GAP == GAP_MERGED) TG[c] = c_ngamma;
            HM[c] = c_mism;
        }
        __syncwarp();

        // Two rows per trip: lane t handles rows rA = 2*(trip - t) - 1 and rB = rA + 1, one trip behind lane t-1.  Both
        // rows take their left border from the previous trip's shuffles, so their cell chains are independent of each
        // other except cell by cell (row B's cell c needs row A's cell c) and the scheduler can interleave them.
        __half2 ta_lA = c_nalpha, tg_lA = c_ngamma, hm_lA = c_mism;   // left border of row A: T - alpha, T - gamma, HM
        __half2 ta_lB = c_nalpha, tg_lB = c_ngamma, hm_lB = c_mism;   // ... of row B
        __half2 hm_dA = c_mism;                                      // HM(rA - 1, left column): diagonal of row A, cell 0
        __half2 bestvec = c_zero;
        // row r lives at qbuf index r - 1 + 2P; the running address doubles as loop counter and record tag
        const unsigned qbase = (unsigned)__cvta_generic_to_shared(&qbuf[gib][0]);
        unsigned qaddr = qbase + 4u * (unsigned)(2 * P - 2 * t);
        const unsigned qend = qaddr + 8u * (unsigned)((mm_w + 1) / 2 + P - 1);
        __half2 HM2[K];

        auto row = [&](__half2 q, const __half2 (&hin)[K], __half2 (&hout)[K], __half2 hm_diag, __half2& la, __half2& lg,
                       __half2& rm) {
            rm = c_zero;
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const __half2 d = __hfma2_relu(__heq2(q, sc[c]), c_delta, c == 0 ? hm_diag : hin[c - 1]);
                // h = max(d, T_up - alpha, T_left - alpha); T = max(d, T_up - gamma, T_left - gamma)
#ifdef WSB_TG_ONLY
                __half2 h;
                if (GAP == GAP_MERGED) {   // one gap array: M = max(T_up, T_left) - gamma; T = max(M, d); h = max(M - (alpha-gamma), d)
                    const __half2 mx = __hmax2(TG[c], lg);
                    const __half2 tn = __hmax2(mx, d);
                    h = __hmax2(__hadd2(mx, c_ndelta), d);
                    lg = __hadd2(tn, c_ngamma);
                    TG[c] = lg;
                } else {
                    h = __hmax2(__hmax2(TA[c], la), d);
                    la = __hadd2(h, c_nalpha);
                    TA[c] = la;
                }
#else
                const __half2 h = __hmax2(__hmax2(TA[c], la), d);
                if (GAP == GAP_MERGED) {
                    const __half2 tn = __hmax2(__hmax2(TG[c], lg), d);
                    la = __hadd2(tn, c_nalpha);
                    lg = __hadd2(tn, c_ngamma);
                    TG[c] = lg;
                } else {
                    la = __hadd2(h, c_nalpha);
                }
                TA[c] = la;
#endif
                hout[c] = __hadd2(h, c_mism);
                rm = __hmax2(rm, h);
            }
        };
        unsigned qa_next, qb_next;  // query symbols are fetched one trip ahead of their use
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(qa_next), "=r"(qb_next) : "r"(qaddr) : "memory");
#ifdef WSB_UNROLL2
#pragma unroll 2
#else
#pragma unroll 1
#endif
        while (qaddr != qend) {
            const unsigned qa = qa_next, qb = qb_next;
            asm volatile("ld.shared.v2.b32 {%0, %1}, [%2+8];" : "=r"(qa_next), "=r"(qb_next) : "r"(qaddr) : "memory");
            __half2 laA = ta_lA, lgA = tg_lA, laB = ta_lB, lgB = tg_lB, rmA, rmB;
            row(u2h(qa), HM, HM2, hm_dA, laA, lgA, rmA);
            // row A's right-most column leaves for the next lane as soon as it exists: the next trip's row A needs it
            // first, and the shuffle latency then hides behind row B.
#ifdef WSB_EARLY_SHFL
            __half2 s0 = __shfl_up_sync(0xffffffffu, laA, 1, P);
            __half2 s1 = __shfl_up_sync(0xffffffffu, HM2[K - 1], 1, P);
            __half2 s4 = c_zero;
            if (GAP == GAP_MERGED) s4 = __shfl_up_sync(0xffffffffu, lgA, 1, P);
#endif
            record_rows<K>(HM2, rmA, bestvec, snap_addr, qaddr);
            bestvec = __hmax2(bestvec, rmA);
            row(u2h(qb), HM2, HM, hm_lA, laB, lgB, rmB);
            hm_dA = hm_lB;
#ifndef WSB_EARLY_SHFL
            __half2 s0 = __shfl_up_sync(0xffffffffu, laA, 1, P);
            __half2 s1 = __shfl_up_sync(0xffffffffu, HM2[K - 1], 1, P);
            __half2 s4 = c_zero;
            if (GAP == GAP_MERGED) s4 = __shfl_up_sync(0xffffffffu, lgA, 1, P);
#endif
            __half2 s2 = __shfl_up_sync(0xffffffffu, laB, 1, P);
            __half2 s3 = __shfl_up_sync(0xffffffffu, HM[K - 1], 1, P);
            __half2 s5 = c_zero;
            if (GAP == GAP_MERGED) s5 = __shfl_up_sync(0xffffffffu, lgB, 1, P);
            record_rows<K>(HM, rmB, bestvec, snap_addr, qaddr + 4);
            bestvec = __hmax2(bestvec, rmB);
            qaddr += 8;
#ifndef WSB_BORDER_SEL
            // lane 0 sees the matrix' zero left border instead of a neighbour: x * keep + edge.  (Integer selects and
            // earlier shuffles were measured slower: ptxas then rotates the strip registers with ~40 moves per trip.)
            ta_lA = __hfma2(s0, keep, edge_ta);
            hm_lA = __hfma2(s1, keep, edge_hm);
            ta_lB = __hfma2(s2, keep, edge_ta);
            hm_lB = __hfma2(s3, keep, edge_hm);
            if (GAP == GAP_MERGED) {
                tg_lA = __hfma2(s4, keep, edge_tg);
                tg_lB = __hfma2(s5, keep, edge_tg);
            }
#else
            ta_lA = t == 0 ? c_nalpha : s0;
            hm_lA = t == 0 ? c_mism : s1;
            ta_lB = t == 0 ? c_nalpha : s2;
            hm_lB = t == 0 ? c_mism : s3;
            if (GAP == GAP_MERGED) {
                tg_lA = t == 0 ? c_ngamma : s4;
                tg_lB = t == 0 ? c_ngamma : s5;
            }
#endif
        }

        // reduce over the group: max value, then smallest row, then smallest strip; the winner resolves its column
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            int bv = AR::get(bestvec, v);
            int bi = 0, bj = col0, who = t;
            if (bv > 0) {  // the tag word after the K columns holds the query-buffer address of the record row
                const uint4 w = snap[v][K / 4][tid];
                const unsigned tag = (K % 4 == 0) ? w.x : (K % 4 == 1) ? w.y : (K % 4 == 2) ? w.z : w.w;
                bi = (int)((tag - qbase) >> 2) - 2 * P + 1;  // buffer index -> matrix row
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
                    const int target = bv + mism;
                    int pos = K;
#pragma unroll
                    for (int ch = (K - 1) / 4; ch >= 0; --ch) {
                        const uint4 w = snap[v][ch][tid];
                        if (4 * ch + 3 < K && AR::get_bits(w.w, v) == target) pos = 4 * ch + 3;
                        if (4 * ch + 2 < K && AR::get_bits(w.z, v) == target) pos = 4 * ch + 2;
                        if (4 * ch + 1 < K && AR::get_bits(w.y, v) == target) pos = 4 * ch + 1;
                        if (AR::get_bits(w.x, v) == target) pos = 4 * ch;
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
