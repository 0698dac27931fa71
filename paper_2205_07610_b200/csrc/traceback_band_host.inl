// traceback_band_host.inl -- host side of the bounded-memory traceback of one large pair (traceback_band.cuh).
// Included by traceback_host.inl.
#include "traceback_band.cuh"

using BandSweepFn = void (*)(const BandParams);
using BandWalkFn = void (*)(BandParams, BandWalk*, uint32_t*);
template <int ATYPE> static void tb_band_pick_gap(bool affine, BandSweepFn& sweep, BandWalkFn& walk) {
    if (affine) { sweep = tb_band_sweep_kernel<ATYPE, true>; walk = tb_band_walk_kernel<ATYPE, true>; }
    else { sweep = tb_band_sweep_kernel<ATYPE, false>; walk = tb_band_walk_kernel<ATYPE, false>; }
}
static void tb_band_pick(int atype, bool affine, BandSweepFn& sweep, BandWalkFn& walk) {
    if (atype == AT_GLOBAL) tb_band_pick_gap<AT_GLOBAL>(affine, sweep, walk);
    else if (atype == AT_LOCAL) tb_band_pick_gap<AT_LOCAL>(affine, sweep, walk);
    else tb_band_pick_gap<AT_SEMI>(affine, sweep, walk);
}

// grow the run buffer of a batch to hold `total` runs, keeping what is already there
static int tb_reserve_runs(wsb_ctx* ctx, TracebackState& tb, int64_t total, int64_t hint) {
    if (total <= tb.runs_cap) return WSB_OK;
    const int64_t want = std::max<int64_t>(total * 3 / 2 + 1024, hint);
    uint32_t* bigger = nullptr;
    CUDA_TRY(ctx, ctx->alloc((void**)&bigger, sizeof(uint32_t) * (size_t)want));
    if (tb.d_runs && tb.total_runs)
        CUDA_TRY(ctx, cudaMemcpyAsync(bigger, tb.d_runs, sizeof(uint32_t) * (size_t)tb.total_runs, cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (tb.d_runs) ctx->release(tb.d_runs);
    tb.d_runs = bigger; tb.runs_cap = want;
    return WSB_OK;
}

// Height R of the checkpoint bands of a rows x cols problem under a scratch budget: the smallest multiple of 32 (at
// least 128, at most 8192) whose boundary rows fit next to the tile columns.
static int tb_band_rows(int64_t rows, int64_t cols, size_t budget_bytes) {
    const int64_t nst = (cols + kBandW - 1) / kBandW;
    const double col_bytes = 8.0 * (double)(rows + 2) * (double)nst;
    const double left = std::max((double)budget_bytes - col_bytes, (double)budget_bytes / 4);
    int64_t nb_max = std::max<int64_t>(2, (int64_t)(left / (8.0 * (double)(cols + 1))));
    int64_t R = (rows + nb_max - 1) / nb_max;
    R = std::min<int64_t>(8192, std::max<int64_t>(128, (R + 31) / 32 * 32));
    return (int)R;
}

// Traceback of pair p through checkpointed tiles.  Needs the pair's score and end cell in b->d_score / d_i / d_j.
// Appends the runs at tb.total_runs, sets run_off[p] and the start cell.
static int tb_band_pair(wsb_batch* b, const wsb_scheme* sch, int atype, int64_t p, size_t budget_bytes, float* ms,
                        int* launches) {
    wsb_ctx* ctx = b->ctx;
    TracebackState& tb = b->tb;
    const bool affine = sch->gap_model == WSB_GAP_AFFINE;
    const int beta_eff = affine ? sch->gap_extend : sch->gap_open;
    cudaStream_t st = ctx->stream;

    // global: the end cell is (m, n) and the score comes out of the walk's first tile; local / semiglobal: both come from
    // the score kernels (same tie-break as everywhere else)
    int32_t pq = 0, ps = 0, ei = b->m[p], ej = b->n[p], known = 0;
    int64_t qo = 0, so = 0;
    CUDA_TRY(ctx, cudaMemcpyAsync(&pq, b->d_pq + p, 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(&ps, b->d_ps + p, 4, cudaMemcpyDeviceToHost, st));
    if (atype != AT_GLOBAL) {
        CUDA_TRY(ctx, cudaMemcpyAsync(&ei, b->d_i + p, 4, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(ctx, cudaMemcpyAsync(&ej, b->d_j + p, 4, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(ctx, cudaMemcpyAsync(&known, b->d_score + p, 4, cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    CUDA_TRY(ctx, cudaMemcpyAsync(&qo, b->d_qoff + pq, 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(&so, b->d_soff + ps, 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));

    const int64_t rows = ei, cols = ej;
    BandWalk w{};
    w.i = ei; w.j = ej; w.state = 0; w.cur_op = -1; w.cur_len = 0; w.done = 0; w.tiles = 0; w.overflow = 0; w.n_runs = 0;
    w.cap = rows + cols + 2;
    w.score = known; w.score_known = atype != AT_GLOBAL; w.cells = 0;

    std::vector<void*> blocks;
    auto cleanup = [&]() { for (void* x : blocks) ctx->release(x); blocks.clear(); };
    auto grab = [&](void** out, size_t bytes) {
        cudaError_t e = ctx->alloc(out, bytes);
        if (e == cudaSuccess) blocks.push_back(*out);
        return e;
    };
#define BAND_TRY(expr)                                                                             \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            ctx->last_error = std::string(#expr) + ": " + cudaGetErrorString(e_);                  \
            cleanup();                                                                             \
            return e_ == cudaErrorMemoryAllocation ? WSB_E_NOMEM : WSB_E_CUDA;                     \
        }                                                                                          \
    } while (0)

    uint32_t* d_rev = nullptr;
    BandWalk* d_w = nullptr;
    BAND_TRY(grab((void**)&d_w, sizeof(BandWalk)));
    BAND_TRY(cudaEventRecord(ctx->ev0, st));
    if (rows > 0 && cols > 0) {
        const int R = tb_band_rows(rows, cols, budget_bytes);
        const int nb = (int)((rows + R - 1) / R);
        const int nst = (int)((cols + kBandW - 1) / kBandW);
        BandParams prm{};
        prm.q = b->d_qcodes + qo; prm.s = b->d_scodes + so;
        prm.rows = (int32_t)rows; prm.cols = (int32_t)cols; prm.band_rows = R; prm.n_bands = nb;
        prm.row_stride = cols + 1; prm.col_stride = rows + 2;
        prm.match = sch->match; prm.mismatch = sch->mismatch; prm.alpha = sch->gap_open; prm.beta = beta_eff; prm.one = 1;
        const size_t row_bytes = sizeof(int2) * (size_t)prm.row_stride * (size_t)(nb + 1);
        const size_t col_bytes = sizeof(int2) * (size_t)prm.col_stride * (size_t)std::max(nst - 1, 1);
        const size_t code_bytes = sizeof(uint32_t) * (size_t)tb_code_words(R, kBandW, kBandP, kBandK);
        BAND_TRY(grab((void**)&prm.rowbuf, row_bytes));
        BAND_TRY(grab((void**)&prm.colbuf, col_bytes));
        BAND_TRY(grab((void**)&prm.codes, code_bytes));
        BAND_TRY(grab((void**)&prm.progress, sizeof(int) * (size_t)(nb + 1)));
        BAND_TRY(grab((void**)&d_rev, sizeof(uint32_t) * (size_t)w.cap));
        prm.ticket = prm.progress + nb;
        b->tb_band_peak = std::max<int64_t>(b->tb_band_peak, (int64_t)(row_bytes + col_bytes + code_bytes + 4 * (size_t)w.cap));
        BandSweepFn sweep; BandWalkFn walk;
        tb_band_pick(atype, affine, sweep, walk);
        const int init_n = (int)std::max<int64_t>(cols + 1, nb + 1);
        tb_band_init_kernel<<<(init_n + 255) / 256, 256, 0, st>>>(prm.rowbuf, (int)cols, atype == AT_GLOBAL, sch->gap_open,
                                                                  beta_eff, prm.progress, nb + 1);
        BAND_TRY(cudaGetLastError());
        if (nb > 1 || nst > 1) {   // a single tile needs no checkpoints
            sweep<<<(nb + kThreads / 32 - 1) / (kThreads / 32), kThreads, 0, st>>>(prm);
            BAND_TRY(cudaGetLastError());
        }
        BAND_TRY(cudaMemcpyAsync(d_w, &w, sizeof(BandWalk), cudaMemcpyHostToDevice, st));
        walk<<<1, 32, 0, st>>>(prm, d_w, d_rev);
        BAND_TRY(cudaGetLastError());
        BAND_TRY(cudaMemcpyAsync(&w, d_w, sizeof(BandWalk), cudaMemcpyDeviceToHost, st));
        BAND_TRY(cudaStreamSynchronize(st));
        if (launches) *launches += 3;
        b->tb_band_cells += ((nb > 1 || nst > 1) ? rows * cols : 0) + w.cells;
        b->tb_band_tiles += w.tiles;
        if (w.overflow || !w.done) {
            ctx->last_error = w.overflow == 2 ? "bounded-memory traceback: the end cell's value differs from the score pass"
                                              : "bounded-memory traceback: walk did not finish";
            cleanup();
            return WSB_E_CUDA;
        }
        if (atype == AT_GLOBAL) {
            const int32_t sc = w.score;
            BAND_TRY(cudaMemcpyAsync(b->d_score + p, &sc, 4, cudaMemcpyHostToDevice, st));
            BAND_TRY(cudaMemcpyAsync(b->d_i + p, &ei, 4, cudaMemcpyHostToDevice, st));
            BAND_TRY(cudaMemcpyAsync(b->d_j + p, &ej, 4, cudaMemcpyHostToDevice, st));
        }
    }
    ++b->tb_band_pairs;
    int rc = tb_reserve_runs(ctx, tb, tb.total_runs + w.n_runs, 0);
    if (rc) { cleanup(); return rc; }
    if (w.n_runs > 0) {
        tb_band_reverse_kernel<<<(unsigned)((w.n_runs + 255) / 256), 256, 0, st>>>(d_rev, w.n_runs, tb.d_runs + tb.total_runs);
        BAND_TRY(cudaGetLastError());
        if (launches) *launches += 1;
    }
    const int32_t si = w.i, sj = w.j;
    BAND_TRY(cudaMemcpyAsync(tb.d_qs + p, &si, 4, cudaMemcpyHostToDevice, st));
    BAND_TRY(cudaMemcpyAsync(tb.d_ss + p, &sj, 4, cudaMemcpyHostToDevice, st));
    BAND_TRY(cudaMemcpyAsync(tb.d_run_off + p, &tb.total_runs, 8, cudaMemcpyHostToDevice, st));
    BAND_TRY(cudaEventRecord(ctx->ev1, st));
    BAND_TRY(cudaEventSynchronize(ctx->ev1));
    if (ms) { float t = 0.f; BAND_TRY(cudaEventElapsedTime(&t, ctx->ev0, ctx->ev1)); *ms += t; }
    tb.total_runs += w.n_runs;
#undef BAND_TRY
    cleanup();
    return WSB_OK;
}
