// traceback_host.inl -- host side of the traceback path (included at the end of wsb200.cu).
//
// wsb_batch_traceback = score pass (end cells, same kernels and tie-break as score-only mode) + per chunk of pairs:
// direction-code fill -> walk pass 1 (run counts, start cells) -> prefix sum -> walk pass 2 (runs, forward order).
// Pairs are processed in chunks so that the 0.5 byte/cell code scratch stays inside a fixed budget
// (WSB_TB_SCRATCH_MB, default 16 GiB).
#include <cub/device/device_scan.cuh>

#include "traceback_fill16.cuh"
#include "traceback_band_host.inl"

struct TbShape { int P, K; };
static const TbShape kTbShapes[] = {{8, 16}, {8, 32}, {32, 16}, {16, 16}, {8, 24}};   // index 4: packed int16 fill only

static int tb_pick_shape(int max_n, bool packed16) {
    static const char* force = getenv("WSB_TB_SHAPE");  // tuning aid
    if (force && force[0]) return std::min(packed16 ? 4 : 3, std::max(0, atoi(force)));
    if (max_n <= 128) return 0;
    // int32 fill: (8,32); (16,16) = index 3 doubles the resident warps but measured 2 % slower at 250 bp.  The packed int16
    // fill is the other way round (1529 vs 1453 GCUPS on cfg3): its (8,32) form needs 198 registers
    if (packed16 && max_n <= 192) return 4;   // (8,24): 150 bp reads fill 78 % of the strip instead of 59 % of 256 columns
    if (max_n <= 256) return packed16 ? 3 : 1;
    return 2;
}

using TbFillFn = void (*)(const TbParams);
template <int P, int K> static TbFillFn tb_pick_fill(int atype, bool affine) {
    switch (atype) {
        case AT_GLOBAL: return affine ? tb_fill_kernel<P, K, AT_GLOBAL, true> : tb_fill_kernel<P, K, AT_GLOBAL, false>;
        case AT_LOCAL: return affine ? tb_fill_kernel<P, K, AT_LOCAL, true> : tb_fill_kernel<P, K, AT_LOCAL, false>;
        default: return affine ? tb_fill_kernel<P, K, AT_SEMI, true> : tb_fill_kernel<P, K, AT_SEMI, false>;
    }
}

// schemes beyond the signed-byte profile (tb_fill_kernel's WIDE form): one shape, any length
static TbFillFn tb_pick_fill_wide(int atype, bool affine) {
    switch (atype) {
        case AT_GLOBAL: return affine ? tb_fill_kernel<32, 16, AT_GLOBAL, true, true> : tb_fill_kernel<32, 16, AT_GLOBAL, false, true>;
        case AT_LOCAL: return affine ? tb_fill_kernel<32, 16, AT_LOCAL, true, true> : tb_fill_kernel<32, 16, AT_LOCAL, false, true>;
        default: return affine ? tb_fill_kernel<32, 16, AT_SEMI, true, true> : tb_fill_kernel<32, 16, AT_SEMI, false, true>;
    }
}

// packed int16 fill (traceback_fill16.cuh): batches of one stage, two alignments per thread
template <int P, int K, bool AFFINE> static TbFillFn tb_pick_fill16_gap(int atype, bool ragged) {
    if (atype == AT_GLOBAL) return ragged ? tb_fill16_kernel<P, K, AT_GLOBAL, true, AFFINE> : tb_fill16_kernel<P, K, AT_GLOBAL, false, AFFINE>;
    if (atype == AT_LOCAL) return ragged ? tb_fill16_kernel<P, K, AT_LOCAL, true, AFFINE> : tb_fill16_kernel<P, K, AT_LOCAL, false, AFFINE>;
    return ragged ? tb_fill16_kernel<P, K, AT_SEMI, true, AFFINE> : tb_fill16_kernel<P, K, AT_SEMI, false, AFFINE>;
}
template <int P, int K> static TbFillFn tb_pick_fill16_shape(int atype, bool ragged, bool affine) {
    return affine ? tb_pick_fill16_gap<P, K, true>(atype, ragged) : tb_pick_fill16_gap<P, K, false>(atype, ragged);
}
static TbFillFn tb_pick_fill16(int shape, int atype, bool ragged, bool affine) {
    if (shape == 0) return tb_pick_fill16_shape<8, 16>(atype, ragged, affine);
    if (shape == 1) return tb_pick_fill16_shape<8, 32>(atype, ragged, affine);
    if (shape == 3) return tb_pick_fill16_shape<16, 16>(atype, ragged, affine);
    if (shape == 4) return tb_pick_fill16_shape<8, 24>(atype, ragged, affine);
    return nullptr;
}

template <int PASS> static void tb_launch_walk(int atype, const TbParams& prm, cudaStream_t stream) {
    const int thr = 128;
    const unsigned grid = (unsigned)((prm.n_pairs + thr - 1) / thr);
    switch (atype) {
        case AT_GLOBAL: tb_walk_kernel<AT_GLOBAL, PASS><<<grid, thr, 0, stream>>>(prm); break;
        case AT_LOCAL: tb_walk_kernel<AT_LOCAL, PASS><<<grid, thr, 0, stream>>>(prm); break;
        default: tb_walk_kernel<AT_SEMI, PASS><<<grid, thr, 0, stream>>>(prm); break;
    }
}

extern "C" int wsb_batch_traceback(wsb_batch* b, const wsb_scheme* sch, int atype, float* kernel_ms, int32_t* n_launches) {
    if (!b) return WSB_E_ARG;
    std::lock_guard<std::recursive_mutex> lock_(b->ctx->mu);
    int rc = check_scheme(sch, atype);
    if (rc) return rc;
    wsb_ctx* ctx = b->ctx;
    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const bool affine = sch->gap_model == WSB_GAP_AFFINE;
    const int beta_eff = affine ? sch->gap_extend : sch->gap_open;
    // the fill kernels look sigma + alpha up in a signed-byte profile; schemes beyond it take the compare / select form
    const bool wide_tb = std::abs(sch->match + sch->gap_open) > 127 || std::abs(sch->mismatch + sch->gap_open) > 127;
    const int64_t np = b->n_pairs;
    TracebackState& tb = b->tb;
    tb.valid = false;

    size_t budget_words = (size_t)16384 << 18;  // 16 GiB in 32-bit words (a B200 carries 180 GB)
    if (const char* e = getenv("WSB_TB_SCRATCH_MB")) { const long mb = atol(e); if (mb > 0) budget_words = (size_t)mb << 18; }
    if (b->tb_scratch_bytes > 0) budget_words = (size_t)std::max<int64_t>(b->tb_scratch_bytes / 4, 1);
    // pairs whose direction codes alone exceed the budget take the checkpointed-tile path (traceback_band.cuh)
    auto is_giant = [&](int64_t p) {
        const int m_ = b->m[p], n_ = b->n[p];
        return m_ > 0 && n_ > 0 && (size_t)tb_code_words(m_, n_, kBandP, kBandK) > budget_words;
    };
    bool any_giant = false;
    if (b->uniform) any_giant = is_giant(0);
    else for (int64_t p = 0; p < np && !any_giant; ++p) any_giant = is_giant(p);
    if (wide_tb && any_giant) {   // the checkpointed-tile path (traceback_band.cuh) has the byte profile only
        b->ctx->last_error = "traceback beyond the code budget needs |match + gap_open| and |mismatch + gap_open| <= 127";
        return WSB_E_SCHEME;
    }
    b->tb_band_pairs = b->tb_band_cells = b->tb_band_tiles = b->tb_band_peak = 0;

    // 1. end cells with the score kernels (identical tie-break); per-pair length faults surface here
    float score_ms = 0.f;
    int32_t score_launches = 0;
    // (global / semiglobal: the fill kernel finds them itself, only the plan and the empty-side pairs are needed -- unless
    // a giant pair needs its end cell before any code is written)
    rc = batch_score_impl(b, sch, atype, WSB_VARIANT_AUTO, kernel_ms ? &score_ms : nullptr, &score_launches,
                          /*plan_only=*/atype == AT_GLOBAL || (atype == AT_SEMI && !any_giant));
    if (rc) return rc;
    const Plan* score_plan = b->last_plan;

    if (!tb.d_qs) CUDA_TRY(ctx, ctx->alloc((void**)&tb.d_qs, sizeof(int32_t) * (size_t)np));
    if (!tb.d_ss) CUDA_TRY(ctx, ctx->alloc((void**)&tb.d_ss, sizeof(int32_t) * (size_t)np));
    if (!tb.d_run_off) CUDA_TRY(ctx, ctx->alloc((void**)&tb.d_run_off, sizeof(int64_t) * (size_t)(np + 1)));

    // 2. chunks of consecutive pairs under the scratch budget
    int max_m = 0, max_n = 0;
    if (b->uniform) { max_m = b->m[0]; max_n = b->n[0]; }
    else for (int64_t p = 0; p < np; ++p) { max_m = std::max(max_m, b->m[p]); max_n = std::max(max_n, b->n[p]); }
    // two alignments per thread in int16 halves where the batch allows it
    static const bool no16 = getenv("WSB_TB_NO16") != nullptr;   // tuning aid
    const bool can16 = !no16 && !wide_tb && max_m > 0 && max_n > 0 &&
                       tb_fill16_range_ok(max_m, max_n, sch->match, sch->mismatch, sch->gap_open, beta_eff);
    // equal-sized pairs without rejected ones share every bound; anything else takes the masked (ragged) form
    const bool ragged16 = !b->uniform || !(!score_plan || score_plan->status.empty() || score_plan->status[0] == 0);
    const int shape = wide_tb ? 2 : tb_pick_shape(max_n, can16);
    const int P = kTbShapes[shape].P, K = kTbShapes[shape].K;
    TbFillFn fill = wide_tb    ? tb_pick_fill_wide(atype, affine)
                  : shape == 0 ? tb_pick_fill<8, 16>(atype, affine)
                  : shape == 1 ? tb_pick_fill<8, 32>(atype, affine)
                  : shape == 2 ? tb_pick_fill<32, 16>(atype, affine)
                  : shape == 3 ? tb_pick_fill<16, 16>(atype, affine) : tb_pick_fill<8, 32>(atype, affine);   // 4: never launched
    TbFillFn fill16 = (can16 && max_n <= P * K) ? tb_pick_fill16(shape, atype, ragged16, affine) : nullptr;

    int per_sm = 0;
    CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fill, kThreads, 0));
    per_sm = std::max(per_sm, 1);
    const int gpb = kThreads / P;
    const int max_grid = ctx->sm_count * per_sm;
    int max_grid16 = 0;
    if (fill16) {
        int per_sm16 = 0;
        CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm16, fill16, kThreads, 0));
        max_grid16 = ctx->sm_count * std::max(per_sm16, 1);
    }
    const bool multi_stage = max_n > P * K;
    const int64_t bnd_rows = multi_stage ? (int64_t)max_m + 2 : 0;
    const size_t bnd_need = (size_t)bnd_rows * sizeof(int2) * (size_t)max_grid * gpb;
    if (bnd_need > b->bnd_bytes) {
        if (b->d_bnd) { ctx->release(b->d_bnd); b->d_bnd = nullptr; b->bnd_bytes = 0; }
        CUDA_TRY(ctx, ctx->alloc(&b->d_bnd, bnd_need));
        b->bnd_bytes = bnd_need;
    }

    cudaEvent_t e0 = ctx->ev0, e1 = ctx->ev1;
    float total_ms = score_ms;
    int launches = score_launches;
    uint32_t* d_codes = nullptr;
    uint32_t* d_run_tmp = nullptr;
    int64_t* d_code_off = nullptr;
    int32_t* d_cnt = nullptr;
    int64_t* d_chunk_off = nullptr;
    void* d_scan_tmp = nullptr;
    size_t scan_tmp_bytes = 0, codes_cap = 0;
    int64_t chunk_cap = 0;
    std::vector<int64_t> code_off;
    tb.total_runs = 0;
    int status = WSB_OK;
    auto cleanup = [&]() {
        if (d_codes) ctx->release(d_codes);
        if (d_run_tmp) ctx->release(d_run_tmp);
        if (d_code_off) ctx->release(d_code_off);
        if (d_cnt) ctx->release(d_cnt);
        if (d_chunk_off) ctx->release(d_chunk_off);
        if (d_scan_tmp) ctx->release(d_scan_tmp);
    };
#define TB_TRY(expr)                                                                               \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            ctx->last_error = std::string(#expr) + ": " + cudaGetErrorString(e_);                  \
            cleanup();                                                                             \
            return e_ == cudaErrorMemoryAllocation ? WSB_E_NOMEM : WSB_E_CUDA;                     \
        }                                                                                          \
    } while (0)

    // first traceback after creation with the upload still in flight: chunks end on upload-piece boundaries and each fill
    // waits only for its own piece, so the fill of piece k runs while pieces k+1.. are still on the bus
    const bool by_piece = b->upload_pending && b->n_pieces > 1;
    int piece = 0;
    int64_t first = 0;
    while (first < np) {
        if (any_giant && is_giant(first) && !(score_plan && !score_plan->status.empty() && score_plan->status[first] != 0)) {
            int band_launches = 0;
            float band_ms = 0.f;
            const int brc = tb_band_pair(b, sch, atype, first, budget_words * 4, &band_ms, &band_launches);
            if (brc) { cleanup(); return brc; }
            total_ms += band_ms;
            launches += band_launches;
            ++first;
            continue;
        }
        // grow the chunk until the code budget is reached
        code_off.clear();
        int64_t words = 0, count = 0;
        if (by_piece) while (piece + 1 < b->n_pieces && b->piece_end[piece] <= first) ++piece;
        const int64_t chunk_stop = by_piece ? std::max(b->piece_end[piece], first + 1) : np;
        // equal-sized pairs: the code offsets are an arithmetic progression, generated on the device (no per-pair host loop)
        const bool regular = b->uniform && max_m > 0 && max_n > 0 && !ragged16;
        const int64_t w_each = regular ? tb_code_words(max_m, max_n, P, K) : 0;
        if (regular) {
            count = std::min(std::min(np, chunk_stop) - first, std::max<int64_t>(1, (int64_t)budget_words / std::max<int64_t>(w_each, 1)));
            words = w_each * count;
        }
        while (!regular && first + count < std::min(np, chunk_stop)) {
            const int64_t p = first + count;
            const bool faulty = score_plan && score_plan->status[p] != 0;
            const int64_t w = (b->m[p] > 0 && b->n[p] > 0 && !faulty) ? tb_code_words(b->m[p], b->n[p], P, K) : 0;
            if (count > 0 && (words + w > (int64_t)budget_words || (any_giant && !faulty && is_giant(p)))) break;
            code_off.push_back(faulty ? -1 : words);
            words += w;
            ++count;
        }
        if ((size_t)words > codes_cap) {
            if (d_codes) ctx->release(d_codes);
            d_codes = nullptr;
            TB_TRY(ctx->alloc((void**)&d_codes, sizeof(uint32_t) * (size_t)std::max<int64_t>(words, 1)));
            codes_cap = (size_t)words;
        }
        if (count > chunk_cap) {
            if (d_code_off) ctx->release(d_code_off);
            if (d_cnt) ctx->release(d_cnt);
            if (d_chunk_off) ctx->release(d_chunk_off);
            if (d_run_tmp) ctx->release(d_run_tmp);
            d_code_off = nullptr; d_cnt = nullptr; d_chunk_off = nullptr; d_run_tmp = nullptr;
            TB_TRY(ctx->alloc((void**)&d_run_tmp, sizeof(uint32_t) * (size_t)kTbTmpRuns * (size_t)count));
            TB_TRY(ctx->alloc((void**)&d_code_off, sizeof(int64_t) * (size_t)count));
            TB_TRY(ctx->alloc((void**)&d_cnt, sizeof(int32_t) * (size_t)(count + 1)));
            TB_TRY(ctx->alloc((void**)&d_chunk_off, sizeof(int64_t) * (size_t)(count + 1)));
            chunk_cap = count;
            size_t need = 0;
            TB_TRY(cub::DeviceScan::ExclusiveSum(nullptr, need, d_cnt, d_chunk_off, (int)(count + 1), ctx->stream));
            if (need > scan_tmp_bytes) {
                if (d_scan_tmp) ctx->release(d_scan_tmp);
                d_scan_tmp = nullptr;
                TB_TRY(ctx->alloc(&d_scan_tmp, need));
                scan_tmp_bytes = need;
            }
        }
        if (regular) {
            fill_progression_kernel<int64_t><<<(unsigned)((count + 255) / 256), 256, 0, ctx->stream>>>(d_code_off, (int64_t)0, w_each, count);
            TB_TRY(cudaGetLastError());
        } else {
            TB_TRY(cudaMemcpyAsync(d_code_off, code_off.data(), sizeof(int64_t) * (size_t)count, cudaMemcpyHostToDevice, ctx->stream));
        }

        TbParams prm;
        prm.q_codes = b->d_qcodes; prm.q_off = b->d_qoff; prm.q_len = b->d_qlen;
        prm.s_codes = b->d_scodes; prm.s_off = b->d_soff; prm.s_len = b->d_slen;
        prm.pair_q = b->d_pq; prm.pair_s = b->d_ps;
        prm.first_pair = first; prm.n_pairs = count;
        prm.code_off = d_code_off; prm.codes = d_codes;
        prm.match = sch->match; prm.mismatch = sch->mismatch; prm.alpha = sch->gap_open; prm.beta = beta_eff;
        prm.bnd = bnd_rows ? (int2*)b->d_bnd : nullptr; prm.bnd_rows = bnd_rows;
        prm.end_i = b->d_i; prm.end_j = b->d_j; prm.start_i = tb.d_qs; prm.start_j = tb.d_ss;
        prm.w_score = b->d_score; prm.w_i = b->d_i; prm.w_j = b->d_j;
        prm.n_runs = d_cnt; prm.run_off = d_chunk_off; prm.runs = nullptr;
        prm.tb_p = P; prm.tb_k = K; prm.one = 1; prm.run_tmp = d_run_tmp;
        prm.lane_major = fill16 ? 1 : 0;

        if (by_piece) TB_TRY(b->wait_piece(ctx->stream, piece));
        TB_TRY(cudaEventRecord(e0, ctx->stream));
        if (fill16) {
            const int64_t units = (count + 1) / 2;
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((units + gpb - 1) / gpb, max_grid16));
            fill16<<<grid, kThreads, 0, ctx->stream>>>(prm);
        } else {
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((count + gpb - 1) / gpb, max_grid));
            fill<<<grid, kThreads, 0, ctx->stream>>>(prm);
        }
        TB_TRY(cudaGetLastError());
        TB_TRY(cudaMemsetAsync(d_cnt + count, 0, sizeof(int32_t), ctx->stream));
        tb_launch_walk<1>(atype, prm, ctx->stream);
        TB_TRY(cudaGetLastError());
        size_t tmp = scan_tmp_bytes;
        TB_TRY(cub::DeviceScan::ExclusiveSum(d_scan_tmp, tmp, d_cnt, d_chunk_off, (int)(count + 1), ctx->stream));
        int64_t chunk_runs = 0;
        TB_TRY(cudaMemcpyAsync(&chunk_runs, d_chunk_off + count, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        TB_TRY(cudaStreamSynchronize(ctx->stream));
        if (tb.total_runs + chunk_runs > tb.runs_cap) {  // grow the run buffer, keeping what earlier chunks wrote
            const int grc = tb_reserve_runs(ctx, tb, tb.total_runs + chunk_runs,
                                            (int64_t)((double)(tb.total_runs + chunk_runs) * np / (first + count)) + 1024);
            if (grc) { cleanup(); return grc; }
        }
        prm.runs = tb.d_runs + tb.total_runs;
        tb_launch_walk<2>(atype, prm, ctx->stream);
        TB_TRY(cudaGetLastError());
        // global run offsets of this chunk = chunk prefix + runs of earlier chunks
        add_base_kernel<<<(unsigned)((count + 255) / 256), 256, 0, ctx->stream>>>(d_chunk_off, tb.total_runs, count,
                                                                                  tb.d_run_off + first);
        TB_TRY(cudaGetLastError());
        TB_TRY(cudaEventRecord(e1, ctx->stream));
        TB_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        TB_TRY(cudaEventElapsedTime(&ms, e0, e1));
        total_ms += ms;
        launches += 5;
        tb.total_runs += chunk_runs;
        first += count;
    }
    b->upload_pending = false;
    TB_TRY(cudaMemcpyAsync(tb.d_run_off + np, &tb.total_runs, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    TB_TRY(cudaStreamSynchronize(ctx->stream));
#undef TB_TRY
    cleanup();
    tb.valid = true;
    if (kernel_ms) *kernel_ms = total_ms;
    if (n_launches) *n_launches = launches;
    return status;
}

extern "C" int wsb_batch_set_tb_scratch(wsb_batch* b, int64_t bytes) {
    if (!b || bytes < 0) return WSB_E_ARG;
    b->tb_scratch_bytes = bytes;
    return WSB_OK;
}

extern "C" int wsb_batch_tb_info(const wsb_batch* b, int64_t* out4) {
    if (!b || !out4) return WSB_E_ARG;
    out4[0] = b->tb_band_pairs; out4[1] = b->tb_band_cells; out4[2] = b->tb_band_tiles; out4[3] = b->tb_band_peak;
    return WSB_OK;
}

extern "C" int64_t wsb_batch_total_runs(const wsb_batch* b) { return (b && b->tb.valid) ? b->tb.total_runs : -1; }

extern "C" int wsb_batch_fetch_traceback(wsb_batch* b, int32_t* out_score, int32_t* q_start, int32_t* q_end,
                                         int32_t* s_start, int32_t* s_end, uint32_t* cigar, int64_t cigar_cap,
                                         int64_t* cigar_off, int32_t* status) {
    if (!b || !out_score || !q_start || !q_end || !s_start || !s_end || !cigar_off) return WSB_E_ARG;
    if (!b->tb.valid) return WSB_E_ARG;
    wsb_ctx* ctx = b->ctx;
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const int64_t np = b->n_pairs;
    const size_t bytes = sizeof(int32_t) * (size_t)np;
    CUDA_TRY(ctx, cudaMemcpyAsync(cigar_off, b->tb.d_run_off, sizeof(int64_t) * (size_t)(np + 1), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (b->tb.total_runs > cigar_cap || (!cigar && b->tb.total_runs > 0)) return WSB_E_CAPACITY;
    CUDA_TRY(ctx, cudaMemcpyAsync(out_score, b->d_score, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(q_start, b->tb.d_qs, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(s_start, b->tb.d_ss, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(q_end, b->d_i, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(s_end, b->d_j, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (b->tb.total_runs > 0)
        CUDA_TRY(ctx, cudaMemcpyAsync(cigar, b->tb.d_runs, sizeof(uint32_t) * (size_t)b->tb.total_runs, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (status) {
        if (b->last_plan) std::memcpy(status, b->last_plan->status.data(), bytes);
        else std::memset(status, 0, bytes);
    }
    return WSB_OK;
}

extern "C" int wsb_traceback_batch(wsb_ctx* ctx, const wsb_scheme* scheme, int align_type, const uint8_t* q_codes,
                                   const int64_t* q_off, const int32_t* q_len, int64_t n_q, const uint8_t* s_codes,
                                   const int64_t* s_off, const int32_t* s_len, int64_t n_s, const int32_t* pair_q,
                                   const int32_t* pair_s, int64_t n_pairs, int32_t* out_score, int32_t* q_start,
                                   int32_t* q_end, int32_t* s_start, int32_t* s_end, uint32_t* cigar, int64_t cigar_cap,
                                   int64_t* cigar_off, int32_t* status) {
    if (!ctx) return WSB_E_ARG;
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    wsb_batch* b = nullptr;
    int rc = wsb_batch_create(ctx, q_codes, q_off, q_len, n_q, s_codes, s_off, s_len, n_s, pair_q, pair_s, n_pairs, &b);
    if (rc) return rc;
    rc = wsb_batch_traceback(b, scheme, align_type, nullptr, nullptr);
    if (!rc) rc = wsb_batch_fetch_traceback(b, out_score, q_start, q_end, s_start, s_end, cigar, cigar_cap, cigar_off, status);
    wsb_batch_destroy(b);
    return rc;
}
