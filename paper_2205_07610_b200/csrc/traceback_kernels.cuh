// traceback_kernels.cuh -- direction-code fill + on-device walk + run-length CIGAR emission (sm_100a).
//
// Fill: the same lane-group wavefront as the score kernels (lane t owns K columns, row r = it - t), int32, exact
// three-state Gotoh (H, E, F kept apart because the walk must tell "came from E" from "came from F" and "gap extended"
// from "gap opened").  Every cell emits one 4-bit code:
//     bits 1:0  origin of H   0 = stop (local, H == 0)   1 = diagonal (M)   2 = E, vertical (I)   3 = F, horizontal (D)
//     bit  2    E(i,j) == E(i-1,j) - beta   (the vertical gap arriving here is an extension)
//     bit  3    F(i,j) == F(i,j-1) - beta
// Priorities are the reference walk's: diagonal, then E, then F; extension before open (refdp.py:162-165, 196-220).
// The DPX max-with-predicate instructions (__vibmax_s32 -> VIMNMX + predicate) give value and "which side won" in one
// issue slot.  Codes leave the SM in wavefront order -- the lane group writes P*K/2 contiguous bytes per iteration --
// so the only HBM traffic of the fill is 0.5 byte per cell of coalesced 8/16-byte stores.
//
// Walk: one thread per pair starts at the end cell the score kernels found (same tie-break) and follows the codes as
// the reference's state machine does (refdp.py:178-230), first counting runs, then -- after a prefix sum -- writing them
// in forward order as (length << 2 | op) words, op 0 = M, 1 = I, 2 = D.
#pragma once
#include "score_kernels.cuh"

#include <cuda_runtime.h>

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
    const int32_t* end_i; const int32_t* end_j;   // end cells from the score pass
    int32_t* start_i; int32_t* start_j;           // out: alignment start (0-based span starts)
    int32_t* n_runs;                              // per pair of the launch
    const int64_t* run_off;                       // exclusive prefix of n_runs, relative to the launch
    uint32_t* runs;                               // out (pass 2): runs of the launch, forward order
    int32_t tb_p, tb_k;                           // lane-group shape the codes were written with
};

// code block geometry shared by fill and walk
__host__ __device__ inline int64_t tb_code_words(int m, int n, int P, int K) {
    const int W = P * K;
    const int stages = (n + W - 1) / W;
    return (int64_t)stages * (m + P - 1) * P * (K / 8);
}

template <int P, int K, int ATYPE, bool AFFINE>
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
    const int alpha = prm.alpha, beta = prm.beta, match = prm.match, mism = prm.mismatch;

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

        for (int st = 0; st < nstages_w; ++st) {
            const int col0 = st * W + t * K;
            int sc[K], H[K], EP[AFFINE ? K : 1];
#pragma unroll
            for (int c = 0; c < K; ++c) {
                int x = kPadSubject;
                if (col0 + c < n) { x = sp[col0 + c]; x = x < 4 ? x : kFlagSubject; }
                sc[c] = x;
                H[c] = edge_h(GLOBAL_EDGES, col0 + c + 1, alpha, beta);
                if (AFFINE) EP[c] = kNeg32;
            }
            const int h0 = edge_h(GLOBAL_EDGES, col0, alpha, beta);
            int hdiag = h0, hl = kNeg32, fpl = kNeg32;  // left border of the strip at the current row
            int edge = edge_h(GLOBAL_EDGES, 1, alpha, beta);
            if (t == 0) {
                if (st == 0) { hl = edge; fpl = kNeg32; }
                else if (m >= 1 && st < nstages) { const int2 b = bnd[1]; hl = b.x; fpl = b.y; }
            }
            const int it_end = mm_w + P - 1;
            for (int it = 1; it <= it_end; ++it) {
                const int r = it - t;
                int out_h = hl, out_fp = fpl;
                if (r >= 1 && r <= m && st < nstages) {
                    int q = qp[r - 1];
                    q = q < 4 ? q : kFlagQuery;
                    int hd = hdiag, left_h = hl, fl = fpl;
                    int al = left_h - alpha;
                    uint32_t words[NW];
#pragma unroll
                    for (int w = 0; w < NW; ++w) words[w] = 0u;
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        const int d = hd + ((q == sc[c]) ? match : mism);
                        hd = H[c];
                        const int au = H[c] - alpha;
                        bool xe = false, xf = false, pd, pm;
                        int e, f;
                        if (AFFINE) {
                            e = __vibmax_s32(EP[c], au, &xe);   // xe: extension wins ties (refdp.py:207)
                            f = __vibmax_s32(fl, al, &xf);
                        } else {
                            e = au; f = al;
                        }
                        const int m1 = __vibmax_s32(d, e, &pd);  // pd: diagonal wins ties over E
                        int h = __vibmax_s32(m1, f, &pm);        // pm: (diag | E) wins ties over F
                        uint32_t cd = pm ? (pd ? 1u : 2u) : 3u;
                        if (LOCAL && h <= 0) { h = 0; cd = 0u; }
                        if (AFFINE) cd |= (xe ? 4u : 0u) | (xf ? 8u : 0u);
                        words[c / 8] |= cd << (4 * (c % 8));
                        H[c] = h;
                        if (AFFINE) { EP[c] = e - beta; fl = f - beta; }
                        al = h - alpha;
                    }
                    // wavefront-major: iteration it of stage st, lane t
                    uint32_t* dst = code + (((int64_t)st * iters + (it - 1)) * P + t) * NW;
                    if (NW == 2) *reinterpret_cast<uint2*>(dst) = make_uint2(words[0], words[1]);
                    else if (NW == 4) *reinterpret_cast<uint4*>(dst) = make_uint4(words[0], words[1], words[2], words[NW - 1]);
                    else {
#pragma unroll
                        for (int w = 0; w < NW; ++w) dst[w] = words[w];
                    }
                    out_h = H[K - 1];
                    out_fp = AFFINE ? fl : kNeg32;
                    if (t == P - 1 && st + 1 < nstages) bnd[r] = make_int2(out_h, out_fp);
                }
                int nh = __shfl_up_sync(0xffffffffu, out_h, 1, P);
                int nfp = __shfl_up_sync(0xffffffffu, out_fp, 1, P);
                hdiag = hl;
                if (t == 0) {
                    if (st == 0) {
                        if (GLOBAL_EDGES) edge -= beta;
                        nh = edge; nfp = kNeg32;
                    } else if (r + 1 <= m && st < nstages) {
                        const int2 b = bnd[r + 1];
                        nh = b.x; nfp = b.y;
                    }
                }
                hl = nh; fpl = nfp;
                if (r == 0) hdiag = h0;
            }
            __syncwarp();
        }
    }
}

// 4-bit code of cell (i, j), 1 <= i <= m, 1 <= j <= n
__device__ __forceinline__ uint32_t tb_code_at(const uint32_t* code, int i, int j, int m, int P, int K) {
    const int W = P * K;
    const int st = (j - 1) / W;
    const int col = (j - 1) - st * W;
    const int t = col / K, c = col - t * K;
    const int it = i + t;
    const int64_t word = (((int64_t)st * (m + P - 1) + (it - 1)) * P + t) * (K / 8) + c / 8;
    return (code[word] >> (4 * (c % 8))) & 15u;
}

// PASS 1 counts the runs and records the start cell; PASS 2 writes the runs in forward order.
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
    const uint32_t* code = prm.codes + prm.code_off[u];
    const int P = prm.tb_p, K = prm.tb_k;
    int i = prm.end_i[p], j = prm.end_j[p];
    uint32_t* out = nullptr;
    int64_t w = 0;
    if (PASS == 2) { out = prm.runs + prm.run_off[u]; w = prm.n_runs[u]; }
    int count = 0;
    int cur_op = -1, cur_len = 0;
    auto emit = [&](int op, int len) {
        if (len <= 0) return;
        if (op == cur_op) { cur_len += len; return; }
        if (cur_op >= 0) { ++count; if (PASS == 2) out[--w] = ((uint32_t)cur_len << 2) | (uint32_t)cur_op; }
        cur_op = op; cur_len = len;
    };
    int state = 0;  // 0: at H, 1: inside a vertical run (E), 2: inside a horizontal run (F)
    if (m > 0 && n > 0) {
        for (;;) {
            if (state == 0) {
                if (i == 0 && j == 0) break;
                if (ATYPE == AT_GLOBAL) {
                    if (i == 0) { emit(2, j); j = 0; break; }
                    if (j == 0) { emit(1, i); i = 0; break; }
                } else if (i == 0 || j == 0) break;  // local: H == 0 on the edges; semiglobal: free edges
                const uint32_t cd = tb_code_at(code, i, j, m, P, K);
                const uint32_t origin = cd & 3u;
                if (origin == 0u) break;                        // local stop: H(i, j) == 0
                if (origin == 1u) { emit(0, 1); --i; --j; continue; }
                state = origin == 2u ? 1 : 2;
                continue;
            }
            const uint32_t cd = tb_code_at(code, i, j, m, P, K);
            if (state == 1) { emit(1, 1); const bool ext = cd & 4u; --i; if (!ext) state = 0; }
            else { emit(2, 1); const bool ext = cd & 8u; --j; if (!ext) state = 0; }
        }
    } else if (ATYPE == AT_GLOBAL) {  // an empty side: one gap run (ref_traceback walks the edge)
        if (i == 0 && j > 0) { emit(2, j); j = 0; }
        else if (j == 0 && i > 0) { emit(1, i); i = 0; }
    }
    if (cur_op >= 0) { ++count; if (PASS == 2) out[--w] = ((uint32_t)cur_len << 2) | (uint32_t)cur_op; }
    if (PASS == 1) {
        prm.n_runs[u] = count;
        prm.start_i[p] = i;
        prm.start_j[p] = j;
    }
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
