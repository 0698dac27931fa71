// traceback_band.cuh -- bounded-memory traceback of ONE large pair: checkpointed tiles.
//
// The reference reaches linear space with Hirschberg / Myers-Miller splits (traceback.py:208-344): forward and reverse
// sweeps over ever smaller sub-matrices, about twice the cells of the plain fill, and a path that is pinned only at score
// level.  This file bounds the memory of a pair whose 0.5 byte/cell direction codes do not fit the scratch
// budget and still returns the SAME path as the full-matrix walk refdp.ref_traceback (refdp.py:158-235), so CIGARs stay
// bit-exact against the oracle:
//
//   pass 1  exact three-state Gotoh over rows 1..i_end, columns 1..j_end (the end cell comes from the score kernels), no
//           codes stored.  The matrix is cut into tiles of R rows x 512 columns (one 32-lane x 16-column stage).  One
//           warp per band of R rows sweeps its tiles left to right; band b + 1 trails band b by one tile (progress
//           counters in global memory), so all bands of a 100 kbp pair are in flight together.  Kept: the bottom row
//           {H, E} of every band (8 bytes per column) and the right column {H - alpha, F - beta} of every tile (8 bytes
//           per row) -- 8 / R + 8 / 512 bytes per cell instead of 0.5.
//   pass 2  one warp follows the path from the end cell: it re-fills the tile the walk stands in from the tile's saved
//           top row and left column -- now writing the four-bit direction codes of that ONE tile (same bit planes as
//           traceback_kernels.cuh) -- lane 0 walks until it leaves the tile, and so on.  A monotone path enters at most
//           m / R + n / 512 + 1 tiles, so pass 2 costs a few percent of pass 1: the whole traceback computes ~1.0x the
//           cells of the matrix where Hirschberg computes ~2x.
#pragma once
#include "traceback_kernels.cuh"

namespace wsb {

constexpr int kBandP = 32, kBandK = 16, kBandW = kBandP * kBandK;

struct BandParams {
    const uint8_t* q;          // query symbols of the whole pair (device)
    const uint8_t* s;
    int32_t rows;              // matrix rows covered: 1 .. rows (the end cell's row)
    int32_t cols;              // matrix columns covered: 1 .. cols
    int32_t band_rows;         // R
    int32_t n_bands;           // ceil(rows / R)
    int2* rowbuf;              // boundary b at rowbuf[b * row_stride + j], j = 0 .. cols: {H(bR, j), E(bR, j)}
    int64_t row_stride;
    int2* colbuf;              // right column of tile column st at colbuf[st * col_stride + i], i = 1 .. rows: {H - alpha, F - beta}
    int64_t col_stride;
    int* progress;             // tiles finished per band
    int* ticket;               // bands are handed out in launch order (a band only ever waits for a band that is running)
    uint32_t* codes;           // pass 2: code block of one tile
    int32_t match, mismatch, alpha, beta;
    int32_t one;
};

struct BandWalk {              // walk state (device memory, one per pair)
    int32_t i, j;              // current cell (absolute row, column); start cell when done
    int32_t state;             // 0 at H, 1 inside a vertical run, 2 inside a horizontal run
    int32_t cur_op, cur_len;   // run being extended (-1: none)
    int32_t done;
    int32_t tiles;             // tiles re-filled by pass 2
    int32_t overflow;          // 1: run buffer too small; 2: the corner of the first tile is not the expected score
    int32_t score;             // in: score of the pair if known (local / semiglobal); out: H(i_end, j_end) of the first tile
    int32_t score_known;
    int64_t cells;             // cells computed by pass 2
    int64_t n_runs;            // runs written so far (reverse order)
    int64_t cap;               // capacity of the run buffer
};

// One tile: rows r0 + 1 .. r0 + m of stage st.  STORE = false (pass 1): leaves the tile's bottom row in rowbuf and its
// right column in colbuf.  STORE = true (pass 2): writes the direction codes of the tile, stage-0 layout of tb_code_at.
template <int ATYPE, bool AFFINE, bool STORE>
__device__ __forceinline__ int band_tile(const BandParams& prm, int band, int st, int t) {
    constexpr int P = kBandP, K = kBandK, W = kBandW, NW = K / 8;
    constexpr bool LOCAL = ATYPE == AT_LOCAL;
    constexpr bool GLOBAL_EDGES = ATYPE == AT_GLOBAL;
    const int r0 = band * prm.band_rows;
    const int m = min(prm.band_rows, prm.rows - r0);
    const int n = prm.cols;
    const uint8_t* qp = prm.q + r0;
    const int2* top = prm.rowbuf + (int64_t)band * prm.row_stride;
    int2* bot = prm.rowbuf + (int64_t)(band + 1) * prm.row_stride;
    const int2* left = prm.colbuf + (int64_t)max(st - 1, 0) * prm.col_stride + r0;   // only read when st > 0
    int2* right = prm.colbuf + (int64_t)st * prm.col_stride + r0;
    const int alpha = prm.alpha, beta = prm.beta, mism = prm.mismatch, one = prm.one;
    const unsigned miss4 = (unsigned)((mism + alpha) & 0xff) * 0x01010101u;
    const unsigned hit = (unsigned)((prm.match + alpha) & 0xff);
    const int nstages = (n + W - 1) / W;
    const int iters = m + P - 1;

    const int col0 = st * W + t * K;
    unsigned prof[K];
    int AL[K], EP[AFFINE ? K : 1];
#pragma unroll
    for (int c = 0; c < K; ++c) {
        unsigned pw = miss4;
        int2 up = make_int2(kNeg32, kNeg32);
        if (col0 + c < n) {
            const int x = prm.s[col0 + c];
            if (x < 4) pw = (miss4 & ~(0xffu << (8 * x))) | (hit << (8 * x));
            up = __ldcg(top + col0 + c + 1);
        }
        prof[c] = pw;
        AL[c] = up.x - alpha;
        if (AFFINE) EP[c] = up.y - beta;
    }
    const int al_top = (col0 <= n ? __ldcg(top + col0).x : kNeg32) - alpha;   // H(r0, col0) - alpha
    int al_diag = al_top, all = kNeg32, fpl = kNeg32;
    int edge = edge_h(GLOBAL_EDGES, r0 + 1, alpha, beta);                     // H(r0 + 1, 0)
    if (t == 0) {
        if (st == 0) { all = edge - alpha; fpl = kNeg32; }
        else { const int2 b = __ldcg(left + 1); all = b.x; fpl = b.y; }
    }
    auto q_at = [&](int it) { return (int)qp[min(max(it - t - 1, 0), m - 1)]; };
    int q_cur = q_at(1), q_nxt = q_at(2);
    for (int it = 1; it <= iters; ++it) {
        const int q_nn = q_at(it + 2);
        const int r = it - t;
        int out_al = all, out_fp = fpl;
        if (r >= 1 && r <= m) {
            const unsigned qsel = q_cur < 4 ? 1u << (8 * q_cur) : 0u;
            int ad = al_diag, fl = fpl, al = all;
            uint32_t words[NW];
#pragma unroll
            for (int w8 = 0; w8 < NW; ++w8) {
                uint32_t wd = 0u, wm = 0u, we = 0u, wf = 0u;
#pragma unroll
                for (int c8 = 0; c8 < 8; ++c8) {
                    const int c = w8 * 8 + c8;
                    const int d = qsel ? __dp4a((int)prof[c], (int)qsel, ad) : ad + (mism + alpha);
                    ad = AL[c];
                    int h, e, f;
                    if (LOCAL) {
                        bool xe = false, xf = false, pd, pm;
                        if (AFFINE) { e = __vibmax_s32(EP[c], AL[c], &xe); f = __vibmax_s32(fl, al, &xf); }
                        else { e = AL[c]; f = al; }
                        const int m1 = __vibmax_s32(d, e, &pd);
                        h = __vibmax_s32(m1, f, &pm);
                        const bool stop = h <= 0;
                        h = max(h, 0);
                        pd = (pd && pm) || stop;
                        pm = pm && !stop;
                        if (STORE) {
                            if (pd) wd += 1u << c8;
                            if (pm) wm += 1u << (8 + c8);
                        }
                        if (AFFINE) {
                            if (STORE) {
                                if (xe) we += 1u << (16 + c8);
                                if (xf) wf += 1u << (24 + c8);
                            }
                            EP[c] = e - beta; fl = f - beta;
                        }
                    } else if (STORE) {
                        if (AFFINE) {
                            e = max_mark(EP[c], AL[c], we, 1u << (16 + c8), one);
                            f = max_mark(fl, al, wf, 1u << (24 + c8), one);
                            EP[c] = e - beta; fl = f - beta;
                        } else { e = AL[c]; f = al; }
                        const int m1 = max_mark(d, e, wd, 1u << c8, one);
                        h = max_mark(m1, f, wm, 1u << (8 + c8), one);
                    } else {
                        if (AFFINE) {
                            e = max(EP[c], AL[c]); f = max(fl, al);
                            EP[c] = e - beta; fl = f - beta;
                        } else { e = AL[c]; f = al; }
                        h = __vimax3_s32(d, e, f);
                    }
                    al = h - alpha;
                    AL[c] = al;
                }
                words[w8] = (wd | wm) | (we | wf);
            }
            if (STORE) {
                uint32_t* dst = prm.codes + ((int64_t)(it - 1) * P + t) * NW;
                *reinterpret_cast<uint2*>(dst) = make_uint2(words[0], words[1]);
            }
            out_al = al;
            out_fp = AFFINE ? fl : kNeg32;
            if (!STORE && t == P - 1 && st + 1 < nstages) right[r] = make_int2(out_al, out_fp);
        }
        int nal = __shfl_up_sync(0xffffffffu, out_al, 1, P);
        int nfp = __shfl_up_sync(0xffffffffu, out_fp, 1, P);
        al_diag = all;
        if (t == 0) {
            if (st == 0) {
                if (GLOBAL_EDGES) edge -= beta;
                nal = edge - alpha; nfp = kNeg32;
            } else if (r + 1 <= m) {
                const int2 b = __ldcg(left + r + 1);
                nal = b.x; nfp = b.y;
            }
        }
        all = nal; fpl = nfp;
        if (r == 0) al_diag = al_top;
        q_cur = q_nxt; q_nxt = q_nn;
    }
    // every lane's registers now hold row m of its strip: the band's bottom boundary for these columns
    if (!STORE) {
#pragma unroll
        for (int c = 0; c < K; ++c)
            if (col0 + c < n) bot[col0 + c + 1] = make_int2(AL[c] + alpha, AFFINE ? EP[c] + beta : kNeg32);
        if (st == 0 && t == 0) bot[0] = make_int2(edge_h(GLOBAL_EDGES, r0 + m, alpha, beta), kNeg32);
        return 0;
    }
    // pass 2: H(r0 + m, n), the tile's corner under the walk (valid in every lane when column n lies in this tile)
    const int cap = n - 1 - st * W;
    const int hv = select_reg<int, K>(AL, min(max(cap - t * K, 0), K - 1)) + alpha;
    return __shfl_sync(0xffffffffu, hv, min(max(cap / K, 0), P - 1));
}

// pass 1: one warp per band, tile after tile; the band above must have finished the tile over this one
template <int ATYPE, bool AFFINE>
__global__ void __launch_bounds__(kThreads) tb_band_sweep_kernel(const BandParams prm) {
    const int t = threadIdx.x & 31;
    int band = 0;
    if (t == 0) band = atomicAdd(prm.ticket, 1);
    band = __shfl_sync(0xffffffffu, band, 0);
    if (band >= prm.n_bands) return;
    const int nstages = (prm.cols + kBandW - 1) / kBandW;
    volatile int* progress = prm.progress;
    for (int st = 0; st < nstages; ++st) {
        if (band > 0) {
            if (t == 0) while (progress[band - 1] <= st) __nanosleep(200);
            __syncwarp();
            __threadfence();
        }
        band_tile<ATYPE, AFFINE, false>(prm, band, st, t);
        __threadfence();
        __syncwarp();
        if (t == 0) progress[band] = st + 1;
        __syncwarp();
    }
}

// boundary 0: the matrix' top row H(0, j), E(0, j) = -inf (refdp.py:53-58); also clears the progress counters
__global__ void tb_band_init_kernel(int2* row0, int cols, int global_edges, int alpha, int beta, int* progress, int n_prog) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j <= cols) row0[j] = make_int2(edge_h(global_edges != 0, j, alpha, beta), kNeg32);
    if (j < n_prog) progress[j] = 0;
}

// pass 2: one warp.  Re-fill the tile under the walk, lane 0 walks it (refdp.py:178-230), repeat.  Runs are appended in
// walk (reverse) order.
template <int ATYPE, bool AFFINE>
__global__ void __launch_bounds__(32) tb_band_walk_kernel(BandParams prm, BandWalk* w, uint32_t* runs_rev) {
    constexpr bool LOCAL = ATYPE == AT_LOCAL;
    const int t = threadIdx.x;
    BandWalk s = *w;
    auto flush = [&]() {
        if (s.n_runs < s.cap) runs_rev[s.n_runs] = ((uint32_t)s.cur_len << 2) | (uint32_t)s.cur_op;
        else s.overflow = 1;
        ++s.n_runs;
    };
    auto emit = [&](int op, int len) {
        if (len <= 0) return;
        if (op == s.cur_op) { s.cur_len += len; return; }
        if (s.cur_op >= 0) flush();
        s.cur_op = op; s.cur_len = len;
    };
    while (!s.done) {
        if (s.i == 0 || s.j == 0) {   // an edge of the matrix (a gap run cannot still be open here: it opened at the edge cell)
            if (ATYPE == AT_GLOBAL) {
                if (s.i == 0 && s.j > 0) { emit(2, s.j); s.j = 0; }
                else if (s.j == 0 && s.i > 0) { emit(1, s.i); s.i = 0; }
            }
            s.done = 1;
            break;
        }
        const int band = (s.i - 1) / prm.band_rows, st = (s.j - 1) / kBandW;
        const int r0 = band * prm.band_rows, c0 = st * kBandW;
        const int mb = min(prm.band_rows, prm.rows - r0);
        // columns right of the walk are never visited again
        prm.cols = s.j;
        const int corner = band_tile<ATYPE, AFFINE, true>(prm, band, st, t);
        __threadfence();
        __syncwarp();
        if (s.tiles == 0) {   // the first tile ends in the end cell: its corner is the score
            if (s.score_known && corner != s.score) { s.overflow = 2; s.done = 1; break; }
            s.score = corner;
        }
        ++s.tiles;
        s.cells += (int64_t)mb * (s.j - c0);
        if (t == 0) {
            while (s.i > r0 && s.j > c0) {
                const uint32_t cd = tb_code_at<LOCAL>(prm.codes, s.i - r0, s.j - c0, mb, kBandP, kBandK);
                if (s.state == 0) {
                    const uint32_t origin = cd & 3u;
                    if (origin == 0u) { s.done = 1; break; }            // local stop: H(i, j) == 0
                    if (origin == 1u) { emit(0, 1); --s.i; --s.j; continue; }
                    s.state = origin == 2u ? 1 : 2;
                }
                if (s.state == 1) { emit(1, 1); --s.i; if (!(cd & 4u)) s.state = 0; }
                else { emit(2, 1); --s.j; if (!(cd & 8u)) s.state = 0; }
            }
        }
        s.i = __shfl_sync(0xffffffffu, s.i, 0);
        s.j = __shfl_sync(0xffffffffu, s.j, 0);
        s.done = __shfl_sync(0xffffffffu, s.done, 0);
        __syncwarp();
    }
    if (t == 0) {
        if (s.cur_op >= 0) { flush(); s.cur_op = -1; s.cur_len = 0; }
        *w = s;
    }
}

__global__ void tb_band_reverse_kernel(const uint32_t* rev, int64_t n, uint32_t* out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) out[k] = rev[n - 1 - k];
}

}  // namespace wsb
