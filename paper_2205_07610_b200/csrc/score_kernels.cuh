// score_kernels.cuh -- lane-group wavefront DP kernels (score + end cell) for sm_100a.
//
// One lane group of P lanes (P in {4,8,16,32}, a power-of-two slice of a warp) advances one execution unit:
// one alignment (int32 arithmetic) or two independent alignments packed into the halves of a half2 register
// (fp16 arithmetic).  Lane t owns K adjacent matrix columns (subject positions) of the current stage and, at
// iteration `it`, computes row r = it - t of its strip, so a stage of P*K columns finishes in m + P - 1 iterations.
// All DP state of a strip lives in registers; the right-most column of lane t reaches lane t+1 through two
// __shfl_up_sync per iteration.  Query symbols come from a small shared-memory ring that is refilled every 128 rows;
// between stages only the stage's right border column (two values per row) goes through a global scratch column.
// Nothing is read or written per cell outside the register file.
//
// Reference semantics reproduced here (pkg/src/waveseq/):
//   cell updates            _kernels.py:113-126 (linear), 259-276 (merged affine), 418-437 (exact affine)
//   edge initialisation     engine.py:210-241, _kernels.py:62-65, refdp.py:53-58,85-90
//   end-cell rule/tie-break _kernels.py:130-145, refdp.py:127-148 (max value; ties -> smallest row, then column)
//   lane hand-off           _kernels.py:156-159, 309-313, 472-477
//   stage chaining          _kernels.py:181-201, 337-357, 502-524
//
// Formulation used for the merged affine state.  With Gs = G + alpha and T = max(Gs - gamma, H), gamma = min(alpha, beta):
//     g  = max(T_up, T_left)                      (= Gs of the cell)
//     d  = H_diag + sigma                         (one fused multiply-add: (H_diag + mismatch) + (match-mismatch)*eq)
//     h  = max(d, g - alpha [, 0])
//     T' = max(d, g - gamma [, 0])
// which is algebraically the reference's x = max(G_up,G_left)-beta; o = max(H_up,H_left)-alpha; g = max(x,o);
// h = max(H_diag+sigma, g [,0]).  Per column the registers hold T and HM = h + mismatch.
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

namespace wsb {

constexpr int kThreads = 128;  // threads per block for all score kernels
constexpr int kQRing = 256;    // query ring rows per lane group (power of two)
constexpr int kQHalf = 128;
constexpr int kPadSubject = 6; // symbol codes that never compare equal to anything
constexpr int kPadQuery = 7;
constexpr int kFlagSubject = 4;
constexpr int kFlagQuery = 5;
constexpr int kNeg32 = -(1 << 30);

enum { AT_GLOBAL = 0, AT_LOCAL = 1, AT_SEMI = 2 };
enum { GAP_LINEAR = 0, GAP_MERGED = 1, GAP_EXACT = 2 };

struct ScoreParams {
    const uint8_t* q_codes; const int64_t* q_off; const int32_t* q_len;
    const uint8_t* s_codes; const int64_t* s_off; const int32_t* s_len;
    const int32_t* pair_q; const int32_t* pair_s;
    const int32_t* units;  // NV pair indices per unit (-1 = empty slot); nullptr = identity (unit u -> pairs NV*u+v)
    int64_t n_units;
    int64_t n_pairs;       // identity mapping: exclusive end of the pair range of this launch
    int64_t pair_base;     // identity mapping: first pair of this launch (a batch may be scored in pieces)
    int32_t* out_score; int32_t* out_i; int32_t* out_j;
    int32_t match, mismatch, alpha, beta;  // beta == alpha for the linear model
    int32_t one = 1;    // the value 1, opaque to the compiler (multiplies that must stay multiplies)
    unsigned long long* block_cycles = nullptr;   // optional: SM cycles every block of the launch spent (clock64 end - start)
    int32_t* redo; int32_t* redo_count;   // packed int16 kernel: pairs it cannot encode (flagged subject symbol) are listed here
    const int32_t* n_pairs_dev;           // re-score launch: units is that list, its length is read from the device
    void* bnd;          // stage border scratch: per lane group bnd_rows x {A, B}
    int64_t bnd_rows;
};

constexpr int kShort16MaxM = 154;    // longest query the packed int16 short-read kernels take (score_short16*.cuh)

using KernelFn = void (*)(const ScoreParams);
struct KernelSel { KernelFn fn; size_t smem; };   // a kernel instantiation and the dynamic shared memory it needs

// ---------------------------------------------------------------- arithmetic policies
// int32 with the substitution score looked up by one IDP.4A: the subject symbol is kept as a profile word (delta =
// match - mismatch in the byte of its code, 0 elsewhere or everywhere for flagged / pad symbols), the query symbol as a
// one-hot byte word (0 for flagged / pad), so H_diag + mismatch + delta * [q == s] is dp4a(profile, onehot, HM_diag).
// Needs |match - mismatch| <= 127; ArI32W below is the unrestricted fallback.
struct ArI32 {
    using V = int32_t;
    static constexpr int NV = 1;
    static __device__ __forceinline__ V splat(int x) { return x; }
    static __device__ __forceinline__ V pack(int a, int) { return a; }
    static __device__ __forceinline__ V neg_inf() { return kNeg32; }
    static __device__ __forceinline__ int get(V a, int) { return a; }
    static __device__ __forceinline__ V add(V a, V b) { return a + b; }
    static __device__ __forceinline__ V vmax(V a, V b) { return max(a, b); }
    template <bool RELU> static __device__ __forceinline__ V diag(V hmd, V q, V s, V) { return __dp4a(s, q, hmd); }
    // max(g + c, d [, 0]); d may or may not already be clamped
    template <bool RELU> static __device__ __forceinline__ V addmax(V g, V c, V d) {
        return RELU ? __viaddmax_s32_relu(g, c, d) : __viaddmax_s32(g, c, d);
    }
    template <bool RELU> static __device__ __forceinline__ V max3(V a, V b, V c) {
        return RELU ? __vimax3_s32_relu(a, b, c) : __vimax3_s32(a, b, c);
    }
    static __device__ __forceinline__ bool any_gt(V a, V b) { return a > b; }
    static __device__ __forceinline__ bool any_ge(V a, V b) { return a >= b; }
    static __device__ __forceinline__ V subj(int a, int, int delta) { return a < 4 ? (V)((unsigned)(delta & 0xff) << (8 * a)) : 0; }
    static __device__ __forceinline__ V query(int a, int) { return a < 4 ? (V)(1u << (8 * a)) : 0; }
    static __device__ __forceinline__ unsigned gt_mask(V a, V b) { return a > b ? 0xffffu : 0u; }
    static __device__ __forceinline__ unsigned ge_mask(V a, V b) { return a >= b ? 0xffffu : 0u; }
    static __device__ __forceinline__ unsigned bits(V a) { return (unsigned)a; }
    static __device__ __forceinline__ int get_bits(unsigned w, int) { return (int)w; }
};

// int32 for any scheme: symbol codes compared directly (compare + select + add per cell)
struct ArI32W : ArI32 {
    template <bool RELU> static __device__ __forceinline__ V diag(V hmd, V q, V s, V delta) {
        return hmd + ((q == s) ? delta : 0);
    }
    static __device__ __forceinline__ V subj(int a, int, int) { return a; }
    static __device__ __forceinline__ V query(int a, int) { return a; }
};

struct ArF16 {
    using V = __half2;
    static constexpr int NV = 2;
    static __device__ __forceinline__ V splat(int x) { return __half2half2(__int2half_rn(x)); }
    static __device__ __forceinline__ V pack(int a, int b) { return __halves2half2(__int2half_rn(a), __int2half_rn(b)); }
    static __device__ __forceinline__ V neg_inf() { return __half2half2(__ushort_as_half((unsigned short)0xFC00)); }
    static __device__ __forceinline__ int get(V a, int v) { return __half2int_rn(v ? __high2half(a) : __low2half(a)); }
    static __device__ __forceinline__ V add(V a, V b) { return __hadd2(a, b); }
    static __device__ __forceinline__ V vmax(V a, V b) { return __hmax2(a, b); }
    template <bool RELU> static __device__ __forceinline__ V diag(V hmd, V q, V s, V delta) {
        const V eq = __heq2(q, s);  // 1.0 / 0.0 per half
        return RELU ? __hfma2_relu(eq, delta, hmd) : __hfma2(eq, delta, hmd);
    }
    // d is already clamped at 0 by diag<true>, so the local variant needs no third operand
    template <bool RELU> static __device__ __forceinline__ V addmax(V g, V c, V d) { return __hmax2(__hadd2(g, c), d); }
    template <bool RELU> static __device__ __forceinline__ V max3(V a, V b, V c) { return __hmax2(__hmax2(a, b), c); }
    static __device__ __forceinline__ bool any_gt(V a, V b) { return __hgt2_mask(a, b) != 0u; }
    static __device__ __forceinline__ bool any_ge(V a, V b) { return __hge2_mask(a, b) != 0u; }
    // symbol codes 0..7 as fp16 integers, both halves in ONE register (the barrier stops the compiler from keeping
    // the halves apart and re-packing them with a PRMT per cell)
    static __device__ __forceinline__ V subj(int a, int b, int) { return codes(a, b); }
    static __device__ __forceinline__ V query(int a, int b) { return codes(a, b); }
    static __device__ __forceinline__ V codes(int a, int b) {
        const unsigned lut_lo = 0x42403C00u, lut_hi = 0x47464544u;  // high bytes of fp16(0..3), fp16(4..7)
        const unsigned ha = __byte_perm(lut_lo, lut_hi, a) & 0xffu, hb = __byte_perm(lut_lo, lut_hi, b) & 0xffu;
        unsigned bits = (ha << 8) | (hb << 24);
        asm volatile("" : "+r"(bits));
        V v; *reinterpret_cast<unsigned*>(&v) = bits; return v;
    }
    static __device__ __forceinline__ unsigned gt_mask(V a, V b) { return __hgt2_mask(a, b); }  // 0xffff per half
    static __device__ __forceinline__ unsigned ge_mask(V a, V b) { return __hge2_mask(a, b); }
    static __device__ __forceinline__ unsigned bits(V a) { return *reinterpret_cast<unsigned*>(&a); }
    static __device__ __forceinline__ int get_bits(unsigned w, int v) {
        return __half2int_rn(__ushort_as_half((unsigned short)(v ? (w >> 16) : (w & 0xffffu))));
    }
};

template <class V> struct alignas(2 * sizeof(V)) Pair2 { V a, b; };

template <int P> __device__ __forceinline__ unsigned group_mask(int lane) {
    return P == 32 ? 0xffffffffu : (((1u << P) - 1u) << (lane & ~(P - 1)));
}

template <class V> __device__ __forceinline__ V shfl_up_v(unsigned mask, V v, int width);
template <> __device__ __forceinline__ int32_t shfl_up_v<int32_t>(unsigned mask, int32_t v, int width) {
    return __shfl_up_sync(mask, v, 1, width);
}
template <> __device__ __forceinline__ __half2 shfl_up_v<__half2>(unsigned mask, __half2 v, int width) {
    return __shfl_up_sync(mask, v, 1, width);
}

// value of register array element idx (idx is not a compile-time constant)
template <class V, int K> __device__ __forceinline__ V select_reg(const V (&a)[K], int idx) {
    V r = a[0];
#pragma unroll
    for (int c = 1; c < K; ++c) if (c == idx) r = a[c];
    return r;
}

// end-cell order of the reference: larger value wins; ties go to the smaller row, then the smaller column
__device__ __forceinline__ bool better_cell(int v, int i, int j, int bv, int bi, int bj) {
    return v > bv || (v == bv && (i < bi || (i == bi && j < bj)));
}

// H(0, j) and H(i, 0) of the reference's edge initialisation (refdp.py:53-58)
__device__ __forceinline__ int edge_h(bool global_edges, int k, int alpha, int beta) {
    return (global_edges && k >= 1) ? -(alpha + beta * (k - 1)) : 0;
}

// dynamic shared memory of one block of score_kernel<AR, P, K, ATYPE, ...>
template <class AR, int P, int K, int ATYPE> constexpr size_t score_smem_bytes() {
    return (ATYPE == AT_LOCAL ? (size_t)AR::NV * ((K + 3) / 4) * kThreads * 16 : 0) +
           (size_t)(kThreads / P) * kQRing * sizeof(typename AR::V);
}

// ---------------------------------------------------------------- the kernel
// MASKED (int32, local only): keep pad columns out of the row maximum explicitly, for schemes where a never-matching
// pad could still raise a score (mismatch > 0 or match < 0); all other instantiations rely on pads being non-improving.
template <class AR, int P, int K, int ATYPE, int GAP, bool MASKED = false>
__global__ void __launch_bounds__(kThreads) score_kernel(const ScoreParams prm) {
    using V = typename AR::V;
    constexpr int NV = AR::NV;
    constexpr int GPB = kThreads / P;  // lane groups per block
    constexpr int W = P * K;           // stage width in columns
    constexpr bool LOCAL = ATYPE == AT_LOCAL;
    constexpr bool GLOBAL_EDGES = ATYPE == AT_GLOBAL;

    constexpr int NCH = (K + 3) / 4;   // 16-byte chunks per row snapshot
    // dynamic shared memory (see score_smem_bytes): row snapshots first (16-byte aligned), then the query rings
    extern __shared__ uint4 smem_dyn[];
    // local alignments: per thread and sub-alignment, the strip's h + mismatch row at its latest record
    uint4 (*snap)[NCH][kThreads] = reinterpret_cast<uint4 (*)[NCH][kThreads]>(smem_dyn);
    V (*qring)[kQRing] = reinterpret_cast<V (*)[kQRing]>(smem_dyn + (LOCAL ? AR::NV * NCH * kThreads : 0));

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int t = tid & (P - 1);
    const int gib = tid / P;
    const unsigned gmask = group_mask<P>(lane);
    const int64_t group_global = (int64_t)blockIdx.x * GPB + gib;
    const int64_t n_groups = (int64_t)gridDim.x * GPB;
    Pair2<V>* bnd = prm.bnd ? reinterpret_cast<Pair2<V>*>(prm.bnd) + group_global * prm.bnd_rows : nullptr;

    const int alpha = prm.alpha, beta = prm.beta, mism = prm.mismatch;
    const int gamma = min(alpha, beta);
    const V c_delta = AR::splat(prm.match - prm.mismatch);
    const V c_mism = AR::splat(mism);
    const V c_nalpha = AR::splat(-alpha);
    const V c_ngamma = AR::splat(-gamma);
    const V c_nbeta = AR::splat(-beta);
    const V c_open_from_hm = AR::splat(-mism - alpha);  // A = H - alpha = HM - mismatch - alpha (exact model)

    // re-score launch of pairs a packed kernel handed back: the unit count sits in device memory
    const int64_t n_units = prm.n_pairs_dev ? (int64_t)((*prm.n_pairs_dev + NV - 1) / NV) : prm.n_units;
    const int64_t n_listed = prm.n_pairs_dev ? (int64_t)*prm.n_pairs_dev : 0;
    const int64_t rounds = (n_units + n_groups - 1) / n_groups;
    for (int64_t rd = 0; rd < rounds; ++rd) {
        const int64_t u = rd * n_groups + group_global;
        int pidx[NV], m[NV], n[NV];
        const uint8_t* qp[NV];
        const uint8_t* sp[NV];
        int mm = 0, nn = 0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            int p = -1;
            if (u < n_units) {
                if (prm.n_pairs_dev) p = u * NV + v < n_listed ? prm.units[u * NV + v] : -1;
                else if (prm.units) p = prm.units[u * NV + v];
                else { const int64_t pp = prm.pair_base + u * NV + v; p = pp < prm.n_pairs ? (int)pp : -1; }
            }
            pidx[v] = p; m[v] = 0; n[v] = 0; qp[v] = nullptr; sp[v] = nullptr;
            if (p >= 0) {
                const int a = prm.pair_q[p], b = prm.pair_s[p];
                m[v] = prm.q_len[a]; n[v] = prm.s_len[b];
                qp[v] = prm.q_codes + prm.q_off[a];
                sp[v] = prm.s_codes + prm.s_off[b];
            }
            mm = max(mm, m[v]); nn = max(nn, n[v]);
        }
        const int mm_w = __reduce_max_sync(0xffffffffu, mm);
        const int nn_w = __reduce_max_sync(0xffffffffu, nn);
        if (mm_w == 0 || nn_w == 0) continue;  // warp-uniform
        const int nstages = (nn_w + W - 1) / W;

        // ---- result tracking state
        int best_v[NV], best_i[NV], best_j[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            best_v[v] = (ATYPE == AT_GLOBAL) ? kNeg32 : 0;
            best_i[v] = 0;
            best_j[v] = (ATYPE == AT_SEMI) ? n[v] : 0;
        }
        V bestvec = AR::splat(0);  // local: per-lane running best value (both sub-alignments)
        int best_c0[NV];           // local: first column - 1 of the strip at the record
#pragma unroll
        for (int v = 0; v < NV; ++v) best_c0[v] = 0;
        (void)bestvec; (void)best_c0;

        for (int st = 0; st < nstages; ++st) {
            // ---- (re)fill the query ring with rows 1..kQRing at the start of a stage
            if (st == 0 || mm_w > kQRing) {
                __syncwarp();
                for (int x = t; x < kQRing; x += P) {
                    int c[2] = {kPadQuery, kPadQuery};
#pragma unroll
                    for (int v = 0; v < NV; ++v)
                        if (x < m[v]) { const int code = qp[v][x]; c[v] = code < 4 ? code : kFlagQuery; }
                    qring[gib][x] = AR::query(c[0], c[1]);
                }
                __syncwarp();
            }
            const int col0 = st * W + t * K;  // columns of this strip are col0+1 .. col0+K (1-based matrix columns)
            V sc[K], T[K], HM[K];
            V EP[GAP == GAP_EXACT ? K : 1];
#pragma unroll
            for (int c = 0; c < K; ++c) {
                int code[2] = {kPadSubject, kPadSubject};
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    if (col0 + c < n[v]) { const int x = sp[v][col0 + c]; code[v] = x < 4 ? x : kFlagSubject; }
                sc[c] = AR::subj(code[0], code[1], prm.match - prm.mismatch);
                const int h0 = edge_h(GLOBAL_EDGES, col0 + c + 1, alpha, beta);
                T[c] = AR::splat(GAP == GAP_EXACT ? kNeg32 : h0);  // exact model: T[] unused, EP holds E - beta
                HM[c] = AR::splat(h0 + mism);
                if (GAP == GAP_EXACT) EP[c] = AR::neg_inf();
            }
            if (GAP == GAP_EXACT) { /* silence unused warnings */ (void)T; }
            const V hm0 = AR::splat(edge_h(GLOBAL_EDGES, col0, alpha, beta) + mism);  // HM(0, col0): diagonal of row 1
            V hm_diag = hm0;
            V tl = AR::neg_inf(), hml = AR::neg_inf();
            // stage 0: (T, HM) of the matrix' left border at the row lane 0 computes next
            V edge_hm = AR::splat(edge_h(GLOBAL_EDGES, 1, alpha, beta) + mism);
            V edge_t = (GAP == GAP_EXACT) ? AR::neg_inf() : AR::splat(edge_h(GLOBAL_EDGES, 1, alpha, beta));
            if (t == 0) {  // left border values for row 1
                if (st == 0) { tl = edge_t; hml = edge_hm; }
                else { const Pair2<V> b = bnd[1]; tl = b.a; hml = b.b; }
            }
            // per-sub-alignment location of column n inside this stage (semiglobal / global capture)
            int cap_c[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int rel = n[v] - 1 - col0;  // register index of column n in this strip, if 0 <= rel < K
                cap_c[v] = (rel >= 0 && rel < K) ? rel : -1;
            }

            const int it_end = mm_w + P - 1;
            for (int it = 1; it <= it_end; ++it) {
                const int r = it - t;
                // ring refill: rows [base+1, base+kQHalf] replace rows that every lane has passed
                if (mm_w > kQRing && it > P && ((it - P) & (kQHalf - 1)) == 0) {
                    const int base = ((it - P) / kQHalf + 1) * kQHalf;  // first 0-based row index to fill
                    if (base < mm_w) {
                        __syncwarp();
                        for (int x = t; x < kQHalf; x += P) {
                            const int row = base + x;
                            int c[2] = {kPadQuery, kPadQuery};
#pragma unroll
                            for (int v = 0; v < NV; ++v)
                                if (row < m[v]) { const int code = qp[v][row]; c[v] = code < 4 ? code : kFlagQuery; }
                            qring[gib][row & (kQRing - 1)] = AR::query(c[0], c[1]);
                        }
                        __syncwarp();
                    }
                }
                V out_t = tl, out_hm = hml;
                if (r >= 1 && r <= mm) {
                    const V q = qring[gib][(r - 1) & (kQRing - 1)];
                    V hd = hm_diag;
                    V left = tl;   // merged/linear: T_left ; exact: F_left - beta
                    V al = (GAP == GAP_EXACT) ? AR::add(hml, c_open_from_hm) : tl;  // exact: H_left - alpha
                    V rm = AR::splat(LOCAL ? 0 : kNeg32);
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        const V d = AR::template diag<LOCAL>(hd, q, sc[c], c_delta);
                        hd = HM[c];
                        V h;
                        if (GAP == GAP_EXACT) {
                            const V e = AR::vmax(EP[c], AR::add(HM[c], c_open_from_hm));
                            const V f = AR::vmax(left, al);
                            h = AR::template max3<LOCAL>(d, e, f);
                            EP[c] = AR::add(e, c_nbeta);
                            left = AR::add(f, c_nbeta);
                            al = AR::add(h, c_nalpha);
                        } else {
                            const V g = AR::vmax(T[c], left);
                            h = AR::template addmax<LOCAL>(g, c_nalpha, d);
                            if (GAP == GAP_MERGED) left = AR::template addmax<LOCAL>(g, c_ngamma, d);
                            else left = h;
                            T[c] = left;
                        }
                        HM[c] = AR::add(h, c_mism);
                        if (LOCAL) rm = AR::vmax(rm, (MASKED && col0 + c >= n[0]) ? AR::splat(kNeg32) : h);
                    }
                    out_t = left;
                    out_hm = HM[K - 1];

                    if (LOCAL) {
                        // Record rows: the strip's row maximum beats the lane's running best (in later stages a tie
                        // also counts when it sits in a smaller row).  The row itself is parked in shared memory with
                        // predicated 16-byte stores; the column is resolved once, after the last stage.  Pad cells
                        // never exceed an earlier real cell, so a pad "record" can only displace a non-winning one.
                        unsigned gtm = AR::gt_mask(rm, bestvec);
                        if (st > 0) {
                            const unsigned gem = AR::ge_mask(rm, bestvec);
#pragma unroll
                            for (int v = 0; v < NV; ++v) if (r < best_i[v]) gtm |= gem & (0xffffu << (16 * v));
                        }
                        bestvec = AR::vmax(bestvec, rm);
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            if (gtm & (0xffffu << (16 * v))) {
                                best_i[v] = r; best_c0[v] = col0;
#pragma unroll
                                for (int ch = 0; ch < NCH; ++ch) {
                                    uint4 w;
                                    w.x = AR::bits(HM[4 * ch]);
                                    w.y = 4 * ch + 1 < K ? AR::bits(HM[4 * ch + 1]) : 0u;
                                    w.z = 4 * ch + 2 < K ? AR::bits(HM[4 * ch + 2]) : 0u;
                                    w.w = 4 * ch + 3 < K ? AR::bits(HM[4 * ch + 3]) : 0u;
                                    snap[v][ch][tid] = w;
                                }
                            }
                        }
                    } else {
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            if (ATYPE == AT_SEMI && r == m[v]) {  // last row: every valid column, increasing j
#pragma unroll
                                for (int c = 0; c < K; ++c) {
                                    const int hv = AR::get(HM[c], v) - mism;
                                    if (col0 + c < n[v] && better_cell(hv, r, col0 + c + 1, best_v[v], best_i[v], best_j[v])) {
                                        best_v[v] = hv; best_i[v] = r; best_j[v] = col0 + c + 1;
                                    }
                                }
                            } else if (cap_c[v] >= 0 && r <= m[v]) {  // this strip holds column n
                                if (ATYPE == AT_SEMI) {
                                    const int hv = AR::get(select_reg<V, K>(HM, cap_c[v]), v) - mism;
                                    if (better_cell(hv, r, n[v], best_v[v], best_i[v], best_j[v])) {
                                        best_v[v] = hv; best_i[v] = r; best_j[v] = n[v];
                                    }
                                } else if (r == m[v]) {
                                    best_v[v] = AR::get(select_reg<V, K>(HM, cap_c[v]), v) - mism;
                                    best_i[v] = r; best_j[v] = n[v];
                                }
                            }
                        }
                    }
                    if (t == P - 1 && st + 1 < nstages) {  // stage border column out
                        Pair2<V> b; b.a = out_t; b.b = out_hm;
                        bnd[r] = b;
                    }
                }
                // hand the strip's right-most column to the next lane; lane 0 takes the stage's left border
                V nt = shfl_up_v<V>(0xffffffffu, out_t, P);
                V nhm = shfl_up_v<V>(0xffffffffu, out_hm, P);
                hm_diag = hml;
                if (st == 0) {  // warp-uniform: left border of the matrix, H(i, 0) walks down by beta per row
                    if (GLOBAL_EDGES) {
                        if (GAP != GAP_EXACT) edge_t = AR::add(edge_t, c_nbeta);
                        edge_hm = AR::add(edge_hm, c_nbeta);
                    }
                    if (t == 0) { nt = edge_t; nhm = edge_hm; }
                } else if (t == 0 && r + 1 <= mm) {
                    const Pair2<V> b = bnd[r + 1];
                    nt = b.a; nhm = b.b;
                }
                tl = nt; hml = nhm;
                if (r == 0) hm_diag = hm0;
            }
            __syncwarp();  // border column stores of this stage are visible to lane 0 in the next stage
        }

        // ---- reduce over the lanes of the group: max value, then smallest row, then smallest column
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            int bv = LOCAL ? AR::get(bestvec, v) : best_v[v];
            int bi = best_i[v];
            int bj = LOCAL ? best_c0[v] : best_j[v];  // local: strips are disjoint, so the strip origin orders columns
            int who = t;
#pragma unroll
            for (int off = P / 2; off >= 1; off >>= 1) {
                const int ov = __shfl_xor_sync(gmask, bv, off, P);
                const int oi = __shfl_xor_sync(gmask, bi, off, P);
                const int oj = __shfl_xor_sync(gmask, bj, off, P);
                const int ow = __shfl_xor_sync(gmask, who, off, P);
                if (better_cell(ov, oi, oj, bv, bi, bj)) { bv = ov; bi = oi; bj = oj; who = ow; }
            }
            if (LOCAL) {
                if (t == who && pidx[v] >= 0) {  // the winning lane finds the first column of its parked row
                    int j = 0;
                    if (bv > 0) {
                        const int target = bv + mism;
                        int pos = K;
#pragma unroll
                        for (int ch = NCH - 1; ch >= 0; --ch) {
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
            } else if (t == 0 && pidx[v] >= 0) {
                prm.out_score[pidx[v]] = bv;
                prm.out_i[pidx[v]] = bi;
                prm.out_j[pidx[v]] = bj;
            }
        }
    }
}

}  // namespace wsb
