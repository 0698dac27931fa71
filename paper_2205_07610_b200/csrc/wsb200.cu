// wsb200.cu -- host side of libwsb200.so: contexts, resident batches, the length-bucketing planner, kernel dispatch
// and the C ABI declared in include/wsb200.h.  No CPU compute path exists here: every alignment runs in the CUDA
// kernels of score_kernels.cuh / traceback_kernels.cuh.
#include "../../include/wsb200.h"
#include <chrono>
#include "score_kernels.cuh"
#include "score_short.cuh"
#include "score_long.cuh"
#include "traceback_kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <numeric>
#include <atomic>
#include <condition_variable>
#include <string>
#include <thread>
#include <tuple>
#include <type_traits>
#include <vector>

#include "hostpack.h"

using namespace wsb;

// ------------------------------------------------------------------------------------------------ objects
struct wsb_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // host-to-device uploads of a batch run here, overlapping the kernels of earlier pieces
    cudaStream_t dl_stream = nullptr;    // device-to-host result downloads of finished pieces (wsb_batch_score_fetch)
    cudaEvent_t dl_ev[16] = {};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // launch groups of the long-read kernel run side by side on these streams (fork after ev0, join before ev1)
    static constexpr int kAux = 6;
    cudaStream_t aux[kAux] = {};
    cudaEvent_t aux_done[kAux] = {};
    unsigned int* d_queues = nullptr;  // work-queue heads of the long-read launches
    int32_t* d_cflags = nullptr;       // cluster launches of the long-read kernel: kLongCf ints per cluster, kLongCfClusters per cluster size
    std::string last_error;
    // Host threads that pack large byte pools into the 2-bit layout before they cross the bus (hostpack.cpp); 0 = pools go up
    // as they are.  -1 = default: WSB_HOST_PACK_THREADS, else min(16, cores - 1).  wsb_ctx_set_host_pack_threads overrides.
    int host_pack_threads = -1;
    int cluster16 = -1;                // 1: the device schedules clusters of 16 blocks x 16 warps of the long-read kernel (non-portable
                                       // size); -1: not probed yet (probe_cluster16)
    // One context serves every host thread that aligns on its GPU (the reference runs independent alignments
    // concurrently, batch.py:213-240): each entry point that touches the context's streams, events, queues or block
    // cache holds this lock for its whole duration.  Recursive: the one-shot calls nest the batch calls.
    std::recursive_mutex mu;
    // Device-memory cache: batches come and go with every run_batch call, and cudaMalloc/cudaFree of GB-sized pools
    // cost tens of milliseconds each, so freed blocks are kept (size-bucketed, 2 MiB granularity) and reused.
    std::multimap<size_t, void*> free_blocks;
    std::map<void*, size_t> live_blocks;
    size_t cached_bytes = 0;

    cudaError_t alloc(void** out, size_t bytes) {
        const size_t gran = (size_t)2 << 20;
        const size_t want = std::max<size_t>(gran, (bytes + gran - 1) / gran * gran);
        auto it = free_blocks.lower_bound(want);
        if (it != free_blocks.end() && it->first <= want + want / 4) {
            *out = it->second; live_blocks[*out] = it->first; cached_bytes -= it->first; free_blocks.erase(it);
            return cudaSuccess;
        }
        cudaError_t e = cudaMalloc(out, want);
        if (e != cudaSuccess) {  // give the cache back and retry once
            (void)cudaGetLastError();
            trim();
            e = cudaMalloc(out, want);
        }
        if (e == cudaSuccess) live_blocks[*out] = want;
        return e;
    }
    void release(void* p) {
        if (!p) return;
        auto it = live_blocks.find(p);
        if (it == live_blocks.end()) { cudaFree(p); return; }
        free_blocks.emplace(it->second, p); cached_bytes += it->second; live_blocks.erase(it);
        if (cached_bytes > ((size_t)24 << 30)) trim();
    }
    void trim() {
        for (auto& kv : free_blocks) cudaFree(kv.second);
        free_blocks.clear(); cached_bytes = 0;
    }
};

struct LaunchGroup {  // pairs that run in one kernel launch
    int variant = 0;  // WSB_VARIANT_F16X2 | WSB_VARIANT_I32
    int shape = 0;    // index into the (P, K) shape table of the variant
    int gap = 0;      // GAP_LINEAR | GAP_MERGED | GAP_EXACT
    int64_t n_units = 0;
    int64_t unit_off = 0;  // offset (in int32) into the plan's unit array; -1 = identity mapping
    int max_m = 0, max_n = 0;
    int long_nw = 0;       // > 0: long-read kernel with this many warps per block (score_long.cuh)
    bool long16 = false;   // long-read kernel, packed int16: units are two pairs of identical shape (score_long16.cuh)
    int cluster = 1;       // long-read kernel: thread blocks per pair (a cluster of 2, 4 or 8 for the giants of a batch)
};

struct Plan {
    std::vector<LaunchGroup> groups;
    int32_t* d_units = nullptr;   // from the context's block cache (cudaMalloc + cudaFree per call cost more than a cfg1-sized launch)
    std::vector<int32_t> h_units; // source of the upload: lives as long as the plan, so no synchronisation after queueing the copy
    std::vector<int32_t> status;  // per pair
    bool any_error = false;
    // geometry counters of the plan (wsb_batch_plan_stats): the GPU counterpart of EngineStats (engine.py:109-146)
    int64_t st_stages = 0, st_iters = 0, st_updates = 0, st_pairs = 0;
    int64_t st_q_max = 0, st_q_add = 0, st_q_lookup = 0;   // thread-instructions x 4 (packed kernels advance two cells per instruction)
};

// Host-packed upload of a batch whose pools arrive as one-byte codes: T worker threads turn each upload piece into the
// 2-bit layout inside a page-locked staging block; whichever worker finishes a piece last queues its copy, the expanding
// kernel and the piece's event on the copy stream (pieces complete in order: every worker walks them in order).  A
// consumer that wants to wait for piece k on a stream first waits, on the host, until that event HAS been recorded
// (cudaStreamWaitEvent on an event nobody recorded yet returns at once).  A slice with a flagged symbol (no 2-bit
// encoding) goes up as plain bytes.
struct HostPacker {
    static constexpr int kMaxPieces = 16;
    std::vector<std::thread> workers;
    std::mutex mu;
    std::condition_variable cv;
    int queued = 0;                       // packed pieces whose event is recorded (guarded by mu); they complete in order
    int n_packed = 0;                     // pieces 0 .. n_packed-1 are packed; the rest go up as plain bytes, a chunk behind every
                                          // packed piece (all of them queued once the last packed piece is)
    std::atomic<int> done[kMaxPieces];    // workers that finished piece k
    std::atomic<int> flagged[kMaxPieces][2];
    bool raw_done[kMaxPieces] = {};       // plain-byte pieces whose event is recorded (touched by the queueing worker only)
    std::atomic<int> error{0};            // first cudaError_t a worker saw
    std::atomic<long long> bytes{0};      // bytes queued for the bus
    void* host_stage = nullptr;           // page-locked, from wsb_pinned_alloc
    HostPacker() { for (auto& d : done) d.store(0); for (auto& f : flagged) { f[0].store(0); f[1].store(0); } }
    void wait_queued(int k) { const int need = std::min(k, n_packed - 1); std::unique_lock<std::mutex> lk(mu); cv.wait(lk, [&] { return queued > need; }); }
    void join() { for (auto& t : workers) if (t.joinable()) t.join(); workers.clear(); }
};
extern "C" int wsb_pinned_alloc(size_t bytes, void** out);
extern "C" void wsb_pinned_free(void* p);

struct wsb_batch {
    wsb_ctx* ctx = nullptr;
    HostPacker* packer = nullptr;
    // stream `s` waits for upload piece k (host-packed uploads: the piece's event is first awaited on the host)
    cudaError_t wait_piece(cudaStream_t s, int k) {
        if (packer) {
            packer->wait_queued(k);
            if (packer->error.load()) return (cudaError_t)packer->error.load();
        }
        return cudaStreamWaitEvent(s, piece_ev[k], 0);
    }
    void finish_packer() {   // all pieces queued; bytes accounted
        if (!packer) return;
        packer->join();
        h2d_bytes += packer->bytes.exchange(0);
    }
    int64_t n_q = 0, n_s = 0, n_pairs = 0;
    uint8_t *d_qcodes = nullptr, *d_scodes = nullptr;
    int64_t *d_qoff = nullptr, *d_soff = nullptr;
    int32_t *d_qlen = nullptr, *d_slen = nullptr, *d_pq = nullptr, *d_ps = nullptr;
    int32_t *d_score = nullptr, *d_i = nullptr, *d_j = nullptr;
    // per pair lengths (host).  Regular batches (pair i = (i, i), equal-length reads) keep one value instead of a vector.
    struct LenVec {
        std::vector<int32_t> v;
        int32_t uni = -1;
        int32_t operator[](int64_t p) const { return uni >= 0 ? uni : v[(size_t)p]; }
        int32_t& slot(int64_t p) { return v[(size_t)p]; }
        void resize(size_t k) { v.resize(k); }
    };
    LenVec m, n;
    bool uniform = false;       // every pair has the same (m, n)
    int64_t total_cells = 0;
    std::map<std::tuple<int, int, int, int, int, int, int>, Plan> plans;
    const Plan* last_plan = nullptr;
    void* d_bnd = nullptr;
    size_t bnd_bytes = 0;
    int32_t* d_redo_long = nullptr;   // packed int16 long-read kernel: same, re-scored by the int32 long-read kernel
    int32_t* d_redo = nullptr;   // packed int16 kernel: list of pairs to re-score (slot 0 = count, list from slot 4)
    unsigned long long* d_cycles = nullptr;   // per-block SM cycles of the last packed int16 short launch (wsb_batch_kernel_cycles)
    int cycles_blocks = 0;
    // Piecewise upload: piece k covers pairs [piece_end[k-1], piece_end[k]) and is complete (pools included) once
    // piece_ev[k] has fired on the copy stream; the first score call after creation launches piece by piece.
    static constexpr int kMaxPieces = 16;
    int n_pieces = 0;
    int n_pieces_usable = 0;             // 1: score only after the whole upload (packed pools with flagged positions)
    void* stage_blocks[4] = {};          // packed-pool staging areas, released with the batch
    int64_t piece_end[kMaxPieces] = {};
    cudaEvent_t piece_ev[kMaxPieces] = {};
    bool upload_pending = false;
    int64_t h2d_bytes = 0;               // bytes that actually crossed the bus at creation (generated arrays excluded)
    TracebackState tb;  // traceback_kernels.cuh
    // bounded-memory traceback of giant pairs (traceback_band.cuh): scratch budget override and counters of the last call
    int64_t tb_scratch_bytes = 0;
    int64_t tb_band_pairs = 0, tb_band_cells = 0, tb_band_tiles = 0, tb_band_peak = 0;
};

#define CUDA_TRY(ctx, expr)                                                                        \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            (ctx)->last_error = std::string(#expr) + ": " + cudaGetErrorString(e_);                \
            return e_ == cudaErrorMemoryAllocation ? WSB_E_NOMEM : WSB_E_CUDA;                     \
        }                                                                                          \
    } while (0)

// ------------------------------------------------------------------------------------------------ small helpers
extern "C" const char* wsb_strerror(int status) {
    switch (status) {
        case WSB_OK: return "ok";
        case WSB_E_CUDA: return "CUDA runtime or kernel launch failure";
        case WSB_E_ARG: return "invalid argument";
        case WSB_E_NOMEM: return "out of memory";
        case WSB_E_LENGTH: return "sequence lengths exceed the supported score range (max_step*(m+n) >= 2^29)";
        case WSB_E_RANGE: return "problem exceeds the packed half2 value range";
        case WSB_E_SCHEME: return "packed affine mode requires a merged-state-exact scheme";
        case WSB_E_CAPACITY: return "output buffer too small";
        case WSB_E_NODEVICE: return "no CUDA device available";
        default: return "unknown status";
    }
}

extern "C" const char* wsb_version(void) { return "wsb200 0.1.0 (sm_100a)"; }

extern "C" int wsb_device_count(int* count) {
    if (!count) return WSB_E_ARG;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) { *count = 0; (void)cudaGetLastError(); return WSB_E_NODEVICE; }
    *count = n;
    return n > 0 ? WSB_OK : WSB_E_NODEVICE;
}

static int max_step(const wsb_scheme* s) {
    return std::max({std::abs(s->match), std::abs(s->mismatch), s->gap_open, s->gap_extend, 1});
}

extern "C" int wsb_merged_state_exact(const wsb_scheme* s) {
    if (!s) return 0;
    const int worst = std::min(s->mismatch, s->match);
    if (s->match < s->mismatch) return 0;
    if (s->gap_open + s->gap_extend < -worst) return 0;
    if (2 * s->gap_extend < -worst) return 0;
    return 1;
}

extern "C" int wsb_f16_range_ok(const wsb_scheme* s, int32_t m, int32_t n) {
    if (!s) return 0;
    // every finite value the kernel forms is bounded by max_step*(m+n) plus one open/extend/mismatch shift
    const int64_t bound = (int64_t)max_step(s) * ((int64_t)m + n) + std::abs(s->mismatch) + s->gap_open + s->gap_extend;
    return bound <= 2048 ? 1 : 0;
}

extern "C" int wsb_plan_shards(const int32_t* q_len, const int32_t* s_len, const int32_t* pair_q, const int32_t* pair_s,
                               int64_t n_pairs, int32_t n_shards, int32_t* shard_of, int64_t* shard_cells) {
    if (!q_len || !s_len || !pair_q || !pair_s || !shard_of || n_pairs < 0 || n_shards < 1) return WSB_E_ARG;
    std::vector<int64_t> cells((size_t)n_pairs);
    bool uniform = true;
    for (int64_t p = 0; p < n_pairs; ++p) {
        cells[p] = (int64_t)q_len[pair_q[p]] * s_len[pair_s[p]];
        if (cells[p] != cells[0]) uniform = false;
    }
    std::vector<int64_t> load((size_t)n_shards, 0);
    if (uniform) {  // contiguous equal blocks keep the pools' locality
        for (int64_t p = 0; p < n_pairs; ++p) {
            const int k = (int)std::min<int64_t>(n_shards - 1, p * n_shards / std::max<int64_t>(n_pairs, 1));
            shard_of[p] = k; load[k] += cells[p];
        }
    } else {  // longest-processing-time first: biggest pair to the least loaded shard
        std::vector<int64_t> order((size_t)n_pairs);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return cells[a] > cells[b]; });
        for (int64_t p : order) {
            int k = 0;
            for (int x = 1; x < n_shards; ++x) if (load[x] < load[k]) k = x;
            shard_of[p] = k; load[k] += cells[p];
        }
    }
    if (shard_cells) for (int k = 0; k < n_shards; ++k) shard_cells[k] = load[k];
    return WSB_OK;
}

// ------------------------------------------------------------------------------------------------ context
// Gather sequences ids[0 .. n_ids) of a pool into a compact pool (host only): the per-GPU shards of run_batch upload
// only the sequences their pairs reference ("sliced to the referenced subset"; the reference's workers share
// one read-only copy, batch.py:213-240).
extern "C" int wsb_compact_pool(const uint8_t* codes, const int64_t* off, const int32_t* len, const int64_t* ids,
                                int64_t n_ids, uint8_t* out_codes, int64_t* out_off) {
    if (!codes || !off || !len || !ids || !out_off || n_ids < 0) return WSB_E_ARG;
    int64_t at = 0;
    for (int64_t k = 0; k < n_ids; ++k) {
        if (ids[k] < 0 || len[ids[k]] < 0) return WSB_E_ARG;
        out_off[k] = at; at += len[ids[k]];
    }
    if (at > 0 && !out_codes) return WSB_E_ARG;
    const int nthr = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<unsigned>(8u, std::max(1u, std::thread::hardware_concurrency())), at / (4 << 20) + 1));
    auto work = [&](int t) {
        for (int64_t k = n_ids * t / nthr, hi = n_ids * (t + 1) / nthr; k < hi; ++k)
            std::memcpy(out_codes + out_off[k], codes + off[ids[k]], (size_t)len[ids[k]]);
    };
    if (nthr == 1) work(0);
    else {
        std::vector<std::thread> th;
        for (int t = 0; t < nthr; ++t) th.emplace_back(work, t);
        for (auto& x : th) x.join();
    }
    return WSB_OK;
}

extern "C" int wsb_ctx_create(int device, wsb_ctx** out) {
    if (!out) return WSB_E_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) { (void)cudaGetLastError(); return WSB_E_NODEVICE; }
    if (device < 0 || device >= n) return WSB_E_ARG;
    wsb_ctx* c = new (std::nothrow) wsb_ctx();
    if (!c) return WSB_E_NOMEM;
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        // created third, before the six launch-group streams: a process has 8 hardware connections by default
        // (CUDA_DEVICE_MAX_CONNECTIONS) and streams beyond that share one; a download stream that shares the upload stream's
        // connection queues every later upload piece behind a download that is waiting for its kernel (measured: the
        // piecewise pipeline degrades to upload + kernel, 18 -> 22 ms per 4 M pairs)
        cudaStreamCreateWithFlags(&c->dl_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess) {
        (void)cudaGetLastError();
        delete c;
        return WSB_E_CUDA;
    }
    bool ok = cudaMalloc((void**)&c->d_queues, 64 * sizeof(unsigned int)) == cudaSuccess &&
              cudaMalloc((void**)&c->d_cflags, 4 * kLongCfClusters * kLongCf * sizeof(int32_t)) == cudaSuccess &&
              cudaMemset(c->d_cflags, 0, 4 * kLongCfClusters * kLongCf * sizeof(int32_t)) == cudaSuccess;
    for (int k = 0; k < wsb_ctx::kAux && ok; ++k)
        ok = cudaStreamCreateWithFlags(&c->aux[k], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&c->aux_done[k], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) { (void)cudaGetLastError(); wsb_ctx_destroy(c); return WSB_E_CUDA; }
    *out = c;
    return WSB_OK;
}

extern "C" void wsb_ctx_destroy(wsb_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    c->trim();
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    for (int k = 0; k < wsb_ctx::kAux; ++k) {
        if (c->aux[k]) cudaStreamDestroy(c->aux[k]);
        if (c->aux_done[k]) cudaEventDestroy(c->aux_done[k]);
    }
    if (c->d_queues) cudaFree(c->d_queues);
    if (c->d_cflags) cudaFree(c->d_cflags);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->dl_stream) cudaStreamDestroy(c->dl_stream);
    for (cudaEvent_t e : c->dl_ev) if (e) cudaEventDestroy(e);
    delete c;
}

extern "C" const char* wsb_last_error(const wsb_ctx* c) { return c ? c->last_error.c_str() : "null context"; }
extern "C" int wsb_ctx_sm_count(const wsb_ctx* c) { return c ? c->sm_count : 0; }
extern "C" int wsb_ctx_set_host_pack_threads(wsb_ctx* c, int threads) {
    if (!c || threads < -1) return WSB_E_ARG;
    std::lock_guard<std::recursive_mutex> lock_(c->mu);
    c->host_pack_threads = threads;
    return WSB_OK;
}
extern "C" const char* wsb_host_pack_isa(void) { return hostpack_isa(); }

// ------------------------------------------------------------------------------------------------ batch
// Metadata arrays of regular batches (equal-length reads laid out back to back, pair i = (i, i)) are arithmetic
// progressions: those are generated on the device instead of crossing the bus (40 bytes per pair at 150 bp).
template <class T> static bool is_progression(const T* a, int64_t n, T& a0, T& d) {
    a0 = n > 0 ? a[0] : T(0);
    d = n > 1 ? T(a[1] - a[0]) : T(0);
    for (int64_t k = 0; k < n; ++k)
        if (a[k] != T(a0 + d * T(k))) return false;
    return true;
}
template <class T> __global__ void fill_progression_kernel(T* dst, T a0, T d, int64_t n) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) dst[k] = T(a0 + d * T(k));
}

template <class T> static int upload(wsb_ctx* ctx, T** dst, const T* src, int64_t count) {
    *dst = nullptr;
    const size_t bytes = sizeof(T) * (size_t)std::max<int64_t>(count, 1);
    CUDA_TRY(ctx, ctx->alloc((void**)dst, bytes));
    if (count > 0) CUDA_TRY(ctx, cudaMemcpyAsync(*dst, src, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice, ctx->copy_stream));
    return WSB_OK;
}
template <class T> static int generate(wsb_ctx* ctx, T** dst, T a0, T d, int64_t count) {
    *dst = nullptr;
    CUDA_TRY(ctx, ctx->alloc((void**)dst, sizeof(T) * (size_t)std::max<int64_t>(count, 1)));
    if (count > 0) {
        fill_progression_kernel<T><<<(unsigned)((count + 255) / 256), 256, 0, ctx->copy_stream>>>(*dst, a0, d, count);
        CUDA_TRY(ctx, cudaGetLastError());
    }
    return WSB_OK;
}

extern "C" void wsb_batch_destroy(wsb_batch* b) {
    if (!b) return;
    std::lock_guard<std::recursive_mutex> lock_(b->ctx->mu);
    cudaSetDevice(b->ctx->device);
    if (b->packer) b->packer->join();    // its workers queue work on the copy stream
    cudaStreamSynchronize(b->ctx->copy_stream);
    cudaStreamSynchronize(b->ctx->stream);
    if (b->packer) { if (b->packer->host_stage) wsb_pinned_free(b->packer->host_stage); delete b->packer; b->packer = nullptr; }
    for (int k = 0; k < wsb_batch::kMaxPieces; ++k) if (b->piece_ev[k]) cudaEventDestroy(b->piece_ev[k]);
    if (b->d_cycles) b->ctx->release(b->d_cycles);
    for (void* p : {(void*)b->d_qcodes, (void*)b->d_scodes, (void*)b->d_qoff, (void*)b->d_soff, (void*)b->d_qlen,
                    (void*)b->d_slen, (void*)b->d_pq, (void*)b->d_ps, (void*)b->d_score, (void*)b->d_i, (void*)b->d_j,
                    b->d_bnd, (void*)b->d_redo, (void*)b->d_redo_long, b->stage_blocks[0], b->stage_blocks[1], b->stage_blocks[2], b->stage_blocks[3]})
        if (p) b->ctx->release(p);
    for (auto& kv : b->plans) if (kv.second.d_units) b->ctx->release(kv.second.d_units);
    // traceback buffers come from the context's block cache
    for (void* p : {(void*)b->tb.d_qs, (void*)b->tb.d_ss, (void*)b->tb.d_run_off, (void*)b->tb.d_runs}) if (p) b->ctx->release(p);
    b->tb.d_qs = b->tb.d_ss = nullptr; b->tb.d_run_off = nullptr; b->tb.d_runs = nullptr;
    b->tb.release();
    delete b;
}

// 2-bit packed pools (the reference's Sequence.data layout, core.py:78-87: four symbols per byte, low bits first, here
// over the concatenated pool) are expanded on the device: a quarter of the bytes cross the bus.
__global__ void unpack2_kernel(const uint8_t* packed_slice, int64_t first_byte, int64_t sym_lo, int64_t sym_hi, uint8_t* codes) {
    // one thread per packed byte of the slice; symbols outside [sym_lo, sym_hi) belong to a neighbouring slice
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t byte = first_byte + k;
    const int64_t s0 = byte * 4;
    if (s0 >= sym_hi) return;
    const unsigned v = packed_slice[k];
    if (s0 >= sym_lo && s0 + 3 < sym_hi && (reinterpret_cast<uintptr_t>(codes + s0) & 3) == 0) {
        *reinterpret_cast<uchar4*>(codes + s0) = make_uchar4(v & 3, (v >> 2) & 3, (v >> 4) & 3, (v >> 6) & 3);
        return;
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
        if (s0 + x >= sym_lo && s0 + x < sym_hi) codes[s0 + x] = (v >> (2 * x)) & 3;
}
__global__ void set_flags_kernel(const int64_t* idx, int64_t n, int64_t limit, uint8_t* codes) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n && idx[k] >= 0 && idx[k] < limit) codes[idx[k]] = 4;
}

struct PackedPools {   // optional: pools given in the 2-bit layout (+ sorted-or-not lists of flagged symbol positions)
    const uint8_t* q_packed = nullptr; const int64_t* q_flags = nullptr; int64_t n_q_flags = 0;
    const uint8_t* s_packed = nullptr; const int64_t* s_flags = nullptr; int64_t n_s_flags = 0;
    // optional: the caller vouches for a regular batch (read k of either pool at k * length, pair i = (i, i)); the
    // metadata arrays may then be null and nothing is scanned
    int32_t uniform_q_len = -1, uniform_s_len = -1;
};

static int batch_create_impl(wsb_ctx* ctx, const uint8_t* q_codes, const int64_t* q_off, const int32_t* q_len,
                             int64_t n_q, const uint8_t* s_codes, const int64_t* s_off, const int32_t* s_len,
                             int64_t n_s, const int32_t* pair_q, const int32_t* pair_s, int64_t n_pairs,
                             const PackedPools& pk, wsb_batch** out) {
    const bool vouched = pk.uniform_q_len >= 0 && pk.uniform_s_len >= 0;
    if (!ctx || !out || (!q_codes && !pk.q_packed) || (!s_codes && !pk.s_packed) ||
        (!vouched && (!q_off || !q_len || !s_off || !s_len || !pair_q || !pair_s)) ||
        n_q <= 0 || n_s <= 0 || n_pairs <= 0 || n_pairs > (int64_t)0x7fffffff || (vouched && (n_pairs > n_q || n_pairs > n_s)))
        return WSB_E_ARG;
    *out = nullptr;
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    wsb_batch* b = new (std::nothrow) wsb_batch();
    if (!b) return WSB_E_NOMEM;
    b->ctx = ctx; b->n_q = n_q; b->n_s = n_s; b->n_pairs = n_pairs;

    // metadata scans, one host thread each: furthest sequence end of either pool (pools need not be packed in order)
    // and the arithmetic-progression test of the six index / offset / length arrays
    int64_t q_total = 0, s_total = 0;
    int64_t o0[2] = {0, 0}, od[2] = {0, 0};
    int32_t l0[2] = {0, 0}, ld[2] = {0, 0}, p0[2] = {0, 0}, pd[2] = {0, 0};
    bool ap_off[2] = {false, false}, ap_len[2] = {false, false}, ap_pair[2] = {false, false};
    {
        auto total_q = [&] { int64_t x = 0; for (int64_t k = 0; k < n_q; ++k) x = std::max(x, q_off[k] + q_len[k]); q_total = x; };
        auto total_s = [&] { int64_t x = 0; for (int64_t k = 0; k < n_s; ++k) x = std::max(x, s_off[k] + s_len[k]); s_total = x; };
        if (vouched) {
            q_total = n_q * pk.uniform_q_len; s_total = n_s * pk.uniform_s_len;
            for (int k = 0; k < 2; ++k) { ap_off[k] = ap_len[k] = ap_pair[k] = true; p0[k] = 0; pd[k] = 1; ld[k] = 0; o0[k] = 0; }
            od[0] = l0[0] = pk.uniform_q_len; od[1] = l0[1] = pk.uniform_s_len;
        } else if (n_pairs >= 65536) {
            std::thread th[8] = {
                std::thread(total_q), std::thread(total_s),
                std::thread([&] { ap_off[0] = is_progression(q_off, n_q, o0[0], od[0]); }),
                std::thread([&] { ap_off[1] = is_progression(s_off, n_s, o0[1], od[1]); }),
                std::thread([&] { ap_len[0] = is_progression(q_len, n_q, l0[0], ld[0]); }),
                std::thread([&] { ap_len[1] = is_progression(s_len, n_s, l0[1], ld[1]); }),
                std::thread([&] { ap_pair[0] = is_progression(pair_q, n_pairs, p0[0], pd[0]); }),
                std::thread([&] { ap_pair[1] = is_progression(pair_s, n_pairs, p0[1], pd[1]); })};
            for (auto& x : th) x.join();
        } else { total_q(); total_s(); }
    }
    // regular batch: identity pair list over equal-length reads -> nothing to validate or tabulate per pair
    const bool regular = ap_pair[0] && p0[0] == 0 && pd[0] == 1 && ap_pair[1] && p0[1] == 0 && pd[1] == 1 && ap_len[0] &&
                         ld[0] == 0 && ap_len[1] && ld[1] == 0 && n_pairs <= n_q && n_pairs <= n_s && l0[0] >= 0 && l0[1] >= 0;
    // per-pair lengths, index validation and the uniformity test, split over host threads
    if (!regular) {
        try { b->m.resize((size_t)n_pairs); b->n.resize((size_t)n_pairs); } catch (...) { delete b; return WSB_E_NOMEM; }
    }
    const int nthr = regular ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency())), n_pairs / 65536 + 1));
    std::vector<int> bad(nthr, 0), uni(nthr, 1);
    std::vector<int64_t> cells(nthr, 0);
    const int m0 = regular ? l0[0] : (pair_q[0] >= 0 && pair_q[0] < n_q) ? q_len[pair_q[0]] : -1;
    const int n0 = regular ? l0[1] : (pair_s[0] >= 0 && pair_s[0] < n_s) ? s_len[pair_s[0]] : -1;
    auto work = [&](int k) {
        const int64_t lo = n_pairs * k / nthr, hi = n_pairs * (k + 1) / nthr;
        int64_t acc = 0;
        for (int64_t p = lo; p < hi; ++p) {
            const int a = pair_q[p], c = pair_s[p];
            if (a < 0 || a >= n_q || c < 0 || c >= n_s) { bad[k] = 1; b->m.slot(p) = b->n.slot(p) = 0; continue; }
            const int mm = q_len[a], nn = s_len[c];
            if (mm < 0 || nn < 0) { bad[k] = 1; continue; }
            b->m.slot(p) = mm; b->n.slot(p) = nn;
            acc += (int64_t)mm * nn;
            if (mm != m0 || nn != n0) uni[k] = 0;
        }
        cells[k] = acc;
    };
    if (regular) {
        b->m.uni = l0[0]; b->n.uni = l0[1];
        cells[0] = (int64_t)n_pairs * l0[0] * l0[1];
    } else if (nthr == 1) work(0);
    else {
        std::vector<std::thread> th;
        for (int k = 0; k < nthr; ++k) th.emplace_back(work, k);
        for (auto& x : th) x.join();
    }
    b->uniform = true;
    for (int k = 0; k < nthr; ++k) {
        if (bad[k]) { delete b; return WSB_E_ARG; }
        if (!uni[k]) b->uniform = false;
        b->total_cells += cells[k];
    }

    // Pieces: the pairs are cut into up to eight ranges; piece k needs the pool bytes up to the furthest sequence end
    // any pair of pieces 0..k references, so the pools go up in address order, one slice per piece, and a piece can be
    // scored while the slices of later pieces are still on the bus.  (Arbitrary pair lists degrade gracefully: the
    // first piece then simply waits for most of the pool.)
    int n_pieces = 1;
    if (n_pairs >= 262144 && q_total + s_total >= ((int64_t)32 << 20)) {
        static const int want = [] { const char* e = getenv("WSB_PIECES"); return e ? atoi(e) : 8; }();   // tuning aid
        n_pieces = std::min<int>(wsb_batch::kMaxPieces, std::max(1, want));
    }
    // Half-size pieces at both ends (one piece more): the first kernels start after half a piece's upload, and only half a
    // piece's kernels remain once the last byte has landed.
    const bool half_ends = n_pieces >= 4 && n_pieces < wsb_batch::kMaxPieces;
    const int whole_pieces = n_pieces;
    if (half_ends) ++n_pieces;
    b->n_pieces = n_pieces;
    std::vector<int64_t> need_q((size_t)n_pieces, 0), need_s((size_t)n_pieces, 0);
    {
        auto piece_work = [&](int k) {
            const int64_t lo = k == 0 ? 0 : b->piece_end[k - 1], hi = b->piece_end[k];
            int64_t mq = 0, msq = 0;
            for (int64_t p = lo; p < hi; ++p) {
                const int a = pair_q[p], c = pair_s[p];
                mq = std::max(mq, q_off[a] + q_len[a]);
                msq = std::max(msq, s_off[c] + s_len[c]);
            }
            need_q[k] = mq; need_s[k] = msq;
        };
        for (int k = 0; k < n_pieces; ++k)   // boundaries on multiples of 2048 pairs (packed units never straddle pieces)
            b->piece_end[k] = k + 1 == n_pieces ? n_pairs
                              : std::min<int64_t>(n_pairs, ((half_ends ? n_pairs * (2 * k + 1) / (2 * whole_pieces) : n_pairs * (k + 1) / n_pieces) + 2047) / 2048 * 2048);
        // the arithmetic shortcut holds only for reads stored back to back from offset 0 (always true for the vouched
        // uniform entry); strided or prefixed pools with an identity pair list take the scan below
        const bool back_to_back = regular && ap_off[0] && o0[0] == 0 && od[0] == l0[0] && ap_off[1] && o0[1] == 0 && od[1] == l0[1];
        if (n_pieces == 1) { need_q[0] = q_total; need_s[0] = s_total; }
        else if (back_to_back) {   // pair p needs the pool bytes up to (p + 1) * length
            for (int k = 0; k < n_pieces; ++k) { need_q[k] = b->piece_end[k] * l0[0]; need_s[k] = b->piece_end[k] * l0[1]; }
            need_q[n_pieces - 1] = q_total; need_s[n_pieces - 1] = s_total;
        } else {
            std::vector<std::thread> th;
            for (int k = 0; k < n_pieces; ++k) th.emplace_back(piece_work, k);
            for (auto& x : th) x.join();
            for (int k = 1; k < n_pieces; ++k) { need_q[k] = std::max(need_q[k], need_q[k - 1]); need_s[k] = std::max(need_s[k], need_s[k - 1]); }
            need_q[n_pieces - 1] = q_total; need_s[n_pieces - 1] = s_total;
        }
    }
    int rc;
    {
#define UPG(dst, src, cnt, ap, a0, d) \
        if ((rc = (ap) ? generate(ctx, &b->dst, a0, d, cnt) : upload(ctx, &b->dst, src, cnt)) != WSB_OK) { wsb_batch_destroy(b); return rc; } \
        if (!(ap)) b->h2d_bytes += (int64_t)sizeof(*src) * (cnt);
        UPG(d_qoff, q_off, n_q, ap_off[0], o0[0], od[0]) UPG(d_soff, s_off, n_s, ap_off[1], o0[1], od[1])
        UPG(d_qlen, q_len, n_q, ap_len[0], l0[0], ld[0]) UPG(d_slen, s_len, n_s, ap_len[1], l0[1], ld[1])
        UPG(d_pq, pair_q, n_pairs, ap_pair[0], p0[0], pd[0]) UPG(d_ps, pair_s, n_pairs, ap_pair[1], p0[1], pd[1])
#undef UPG
    }
    auto fail = [&](cudaError_t e) {
        ctx->last_error = cudaGetErrorString(e);
        wsb_batch_destroy(b);
        return e == cudaErrorMemoryAllocation ? WSB_E_NOMEM : WSB_E_CUDA;
    };
    cudaError_t e;
    if ((e = ctx->alloc((void**)&b->d_qcodes, (size_t)std::max<int64_t>(q_total, 1) + 64)) != cudaSuccess) return fail(e);
    if ((e = ctx->alloc((void**)&b->d_scodes, (size_t)std::max<int64_t>(s_total, 1) + 64)) != cudaSuccess) return fail(e);
    // pool slices, address-ordered; a packed pool goes up as packed bytes into a staging area and is expanded per slice
    uint8_t *stage_q = nullptr, *stage_s = nullptr;
    int64_t *dflags_q = nullptr, *dflags_s = nullptr;
    if (pk.q_packed && (e = ctx->alloc((void**)&stage_q, (size_t)(q_total / 4 + 2))) != cudaSuccess) return fail(e);
    if (pk.s_packed && (e = ctx->alloc((void**)&stage_s, (size_t)(s_total / 4 + 2))) != cudaSuccess) return fail(e);
    auto send = [&](const uint8_t* codes, const uint8_t* packed, uint8_t* stage, uint8_t* dst, int64_t lo, int64_t hi) -> cudaError_t {
        if (hi <= lo) return cudaSuccess;
        if (!packed) { b->h2d_bytes += hi - lo; return cudaMemcpyAsync(dst + lo, codes + lo, (size_t)(hi - lo), cudaMemcpyHostToDevice, ctx->copy_stream); }
        const int64_t b0 = lo / 4, b1 = (hi + 3) / 4;   // packed bytes covering symbols [lo, hi)
        b->h2d_bytes += b1 - b0;
        cudaError_t r = cudaMemcpyAsync(stage + b0, packed + b0, (size_t)(b1 - b0), cudaMemcpyHostToDevice, ctx->copy_stream);
        if (r != cudaSuccess) return r;
        unpack2_kernel<<<(unsigned)((b1 - b0 + 255) / 256), 256, 0, ctx->copy_stream>>>(stage + b0, b0, lo, hi, dst);
        return cudaGetLastError();
    };
    // Host-packed upload: byte pools of a piecewise batch are packed by worker threads, piece by piece (see HostPacker)
    int pack_threads = 0;
    if (!pk.q_packed && !pk.s_packed && n_pieces > 1) {
        pack_threads = ctx->host_pack_threads;
        if (pack_threads < 0) {
            static const int dflt = [] {
                const char* ev = getenv("WSB_HOST_PACK_THREADS");
                // one core stays free for the thread that launches the kernels of the pieces as they land (cfg2 on 16 cores:
                // 20.2 ms per call with 15 packers, 21-24 ms with 16)
                const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
                return ev ? atoi(ev) : (int)std::min(16u, hw > 2 ? hw - 1 : hw);
            }();
            pack_threads = dflt;
        }
        pack_threads = std::max(0, std::min(pack_threads, 64));
    }
    if (pack_threads > 0) {
        const int64_t qb = q_total / 4 + 2, sb = s_total / 4 + 2;
        if ((e = ctx->alloc((void**)&stage_q, (size_t)qb)) != cudaSuccess) return fail(e);
        if ((e = ctx->alloc((void**)&stage_s, (size_t)sb)) != cudaSuccess) return fail(e);
        b->stage_blocks[0] = stage_q; b->stage_blocks[1] = stage_s;
        for (int k = 0; k < n_pieces; ++k)
            if ((e = cudaEventCreateWithFlags(&b->piece_ev[k], cudaEventDisableTiming)) != cudaSuccess) return fail(e);
        HostPacker* hp = new (std::nothrow) HostPacker();
        if (!hp) return fail(cudaErrorMemoryAllocation);
        b->packer = hp;
        if (wsb_pinned_alloc((size_t)(qb + sb), &hp->host_stage) != WSB_OK) return fail(cudaErrorMemoryAllocation);
        uint8_t* const hq = static_cast<uint8_t*>(hp->host_stage);
        uint8_t* const hs = hq + qb;
        // metadata queued above (and everything else on the copy stream so far) precedes piece 0's event, as before
        const int T = pack_threads;
        const int device = ctx->device;
        cudaStream_t cs = ctx->copy_stream;
        // WSB_HOST_PACK_RAW=r lets the last r pieces travel as plain bytes meanwhile, in chunks queued behind each packed piece.
        // Off by default: on the bench host the copy engine's reads and the packers' reads share the memory system, and
        // every mix measured slower than packing everything (cfg2, 16 threads: 20.6 ms packed, 23-25 ms with 1-3 plain
        // pieces, 24.3 ms all plain).
        static const int raw_env = [] { const char* ev = getenv("WSB_HOST_PACK_RAW"); return ev ? atoi(ev) : 0; }();
        int n_raw = raw_env;
        n_raw = std::max(0, std::min(n_raw, n_pieces - 1));
        const int n_packed = n_pieces - n_raw;
        hp->n_packed = n_packed;
        uint8_t *dq = b->d_qcodes, *dsc = b->d_scodes;
        cudaEvent_t* evs = b->piece_ev;
        static const bool trace = getenv("WSB_TRACE") != nullptr;
        const auto t_start = std::chrono::steady_clock::now();
        auto worker = [=](int t) {
            int64_t lo[2] = {0, 0};       // symbols of either pool already covered by earlier pieces
            for (int k = 0; k < n_packed; ++k) {
                const int64_t hi[2] = {std::max(lo[0], need_q[k]), std::max(lo[1], need_s[k])};
                int64_t pb0[2], pb1[2];   // packed bytes this piece adds (a byte shared with the previous piece stays as it is)
                for (int v = 0; v < 2; ++v) {
                    pb0[v] = (lo[v] + 3) / 4; pb1[v] = (hi[v] + 3) / 4;
                    if (pb1[v] > pb0[v]) {
                        const int64_t span = pb1[v] - pb0[v];
                        const int64_t a = pb0[v] + span * t / T / 64 * 64, z = t + 1 == T ? pb1[v] : pb0[v] + span * (t + 1) / T / 64 * 64;
                        if (z > a && hostpack_range(v ? s_codes : q_codes, v ? s_total : q_total, v ? hs : hq, a, z)) hp->flagged[k][v].store(1);
                    }
                }
                if (hp->done[k].fetch_add(1) + 1 == T) {   // last one out queues the piece
                    cudaError_t ce = cudaSetDevice(device);
                    for (int v = 0; v < 2 && ce == cudaSuccess; ++v) {
                        if (hi[v] <= lo[v]) continue;
                        const uint8_t* codes = v ? s_codes : q_codes;
                        uint8_t* dst = v ? dsc : dq;
                        if (hp->flagged[k][v].load()) {   // a flagged symbol: this slice travels as plain bytes
                            hp->bytes += hi[v] - lo[v];
                            ce = cudaMemcpyAsync(dst + lo[v], codes + lo[v], (size_t)(hi[v] - lo[v]), cudaMemcpyHostToDevice, cs);
                            continue;
                        }
                        uint8_t* hst = v ? hs : hq;
                        uint8_t* dstage = v ? stage_s : stage_q;
                        if (pb1[v] > pb0[v]) {
                            hp->bytes += pb1[v] - pb0[v];
                            ce = cudaMemcpyAsync(dstage + pb0[v], hst + pb0[v], (size_t)(pb1[v] - pb0[v]), cudaMemcpyHostToDevice, cs);
                            if (ce != cudaSuccess) break;
                        }
                        // a byte shared with the previous piece is on the device already -- unless that piece's slice went up
                        // as plain bytes (flagged): then the few symbols of the shared byte are copied as bytes too
                        const int64_t u0 = lo[v] / 4, u1 = (hi[v] + 3) / 4;
                        int64_t sym_lo = lo[v];
                        if (u0 < pb0[v] && k > 0 && hp->flagged[k - 1][v].load()) {
                            const int64_t edge = std::min(hi[v], pb0[v] * 4);
                            hp->bytes += edge - lo[v];
                            ce = cudaMemcpyAsync(dst + lo[v], codes + lo[v], (size_t)(edge - lo[v]), cudaMemcpyHostToDevice, cs);
                            if (ce != cudaSuccess) break;
                            sym_lo = edge;
                        }
                        if (hi[v] > sym_lo) {
                            const int64_t f0 = sym_lo / 4;
                            unpack2_kernel<<<(unsigned)((u1 - f0 + 255) / 256), 256, 0, cs>>>(dstage + f0, f0, sym_lo, hi[v], dst);
                            ce = cudaGetLastError();
                        }
                    }
                    if (ce == cudaSuccess) ce = cudaEventRecord(evs[k], cs);
                    if (n_raw > 0 && ce == cudaSuccess) {
                        // the plain-byte region (everything behind the last packed piece), cut into n_packed chunks: chunk k
                        // follows packed piece k on the same stream (one copy engine serves host-to-device traffic, so a
                        // long plain copy on a second stream would stall the packed pieces behind it)
                        int64_t r0[2] = {0, 0};
                        for (int j = 0; j < n_packed; ++j) { r0[0] = std::max(r0[0], need_q[j]); r0[1] = std::max(r0[1], need_s[j]); }
                        const int64_t tot[2] = {q_total, s_total};
                        int64_t c_lo[2], c_hi[2];
                        for (int v = 0; v < 2; ++v) {
                            const int64_t span = std::max<int64_t>(0, tot[v] - r0[v]);
                            c_lo[v] = r0[v] + span * k / n_packed; c_hi[v] = k + 1 == n_packed ? tot[v] : r0[v] + span * (k + 1) / n_packed;
                            if (c_hi[v] > c_lo[v] && ce == cudaSuccess) {
                                hp->bytes += c_hi[v] - c_lo[v];
                                ce = cudaMemcpyAsync((v ? dsc : dq) + c_lo[v], (v ? s_codes : q_codes) + c_lo[v], (size_t)(c_hi[v] - c_lo[v]),
                                                     cudaMemcpyHostToDevice, cs);
                            }
                        }
                        // a plain piece is complete once the chunks up to its end are on the stream
                        for (int j = n_packed; j < n_pieces && ce == cudaSuccess; ++j) {
                            const bool now = k + 1 == n_packed || (c_hi[0] >= need_q[j] && c_hi[1] >= need_s[j]);
                            if (now && !hp->raw_done[j]) { hp->raw_done[j] = true; ce = cudaEventRecord(evs[j], cs); }
                        }
                    }
                    if (ce != cudaSuccess) { int zero = 0; hp->error.compare_exchange_strong(zero, (int)ce); }
                    { std::lock_guard<std::mutex> lk(hp->mu); hp->queued = k + 1; }
                    hp->cv.notify_all();
                    if (trace) fprintf(stderr, "[wsb] host pack: piece %d queued at %.2f ms (%s, %d threads)\n", k,
                                       std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(), hostpack_isa(), T);
                }
                lo[0] = hi[0]; lo[1] = hi[1];
            }
        };
        try {
            for (int t = 0; t < T; ++t) hp->workers.emplace_back(worker, t);
        } catch (...) {
            // could not start every worker: nobody would ever complete a piece.  Let the started ones run out (they only
            // pack), then fall back to the plain upload below.
            hp->join();
            for (auto& d : hp->done) d.store(0);
            pack_threads = 0;
        }
    }
    int64_t done_q = 0, done_s = 0;
    for (int k = 0; k < n_pieces && pack_threads == 0; ++k) {
        if ((e = send(q_codes, pk.q_packed, stage_q, b->d_qcodes, done_q, need_q[k])) != cudaSuccess) return fail(e);
        done_q = std::max(done_q, need_q[k]);
        if ((e = send(s_codes, pk.s_packed, stage_s, b->d_scodes, done_s, need_s[k])) != cudaSuccess) return fail(e);
        done_s = std::max(done_s, need_s[k]);
        if (k + 1 == n_pieces) {   // flagged positions (rare) are stamped once everything is expanded
            if (pk.q_packed && pk.n_q_flags > 0) {
                if ((e = ctx->alloc((void**)&dflags_q, sizeof(int64_t) * (size_t)pk.n_q_flags)) != cudaSuccess) return fail(e);
                if ((e = cudaMemcpyAsync(dflags_q, pk.q_flags, sizeof(int64_t) * (size_t)pk.n_q_flags, cudaMemcpyHostToDevice, ctx->copy_stream)) != cudaSuccess) return fail(e);
                set_flags_kernel<<<(unsigned)((pk.n_q_flags + 255) / 256), 256, 0, ctx->copy_stream>>>(dflags_q, pk.n_q_flags, q_total, b->d_qcodes);
            }
            if (pk.s_packed && pk.n_s_flags > 0) {
                if ((e = ctx->alloc((void**)&dflags_s, sizeof(int64_t) * (size_t)pk.n_s_flags)) != cudaSuccess) return fail(e);
                if ((e = cudaMemcpyAsync(dflags_s, pk.s_flags, sizeof(int64_t) * (size_t)pk.n_s_flags, cudaMemcpyHostToDevice, ctx->copy_stream)) != cudaSuccess) return fail(e);
                set_flags_kernel<<<(unsigned)((pk.n_s_flags + 255) / 256), 256, 0, ctx->copy_stream>>>(dflags_s, pk.n_s_flags, s_total, b->d_scodes);
            }
        }
        if (!b->piece_ev[k] && (e = cudaEventCreateWithFlags(&b->piece_ev[k], cudaEventDisableTiming)) != cudaSuccess) return fail(e);
        if ((e = cudaEventRecord(b->piece_ev[k], ctx->copy_stream)) != cudaSuccess) return fail(e);
    }
    if (pack_threads == 0 && b->packer) {   // workers could not be started: plain upload done above
        if (b->packer->host_stage) wsb_pinned_free(b->packer->host_stage);
        delete b->packer; b->packer = nullptr;
    }
    // staging areas are only touched by work already queued on the copy stream: hand them back to the cache now, the
    // next user of those blocks is ordered behind this batch on the same streams
    b->stage_blocks[0] = stage_q; b->stage_blocks[1] = stage_s; b->stage_blocks[2] = dflags_q; b->stage_blocks[3] = dflags_s;
    b->upload_pending = true;
    if ((pk.q_packed && pk.n_q_flags > 0) || (pk.s_packed && pk.n_s_flags > 0)) b->n_pieces_usable = 1;  // flags land last
    for (int32_t** p : {&b->d_score, &b->d_i, &b->d_j}) {
        e = ctx->alloc((void**)p, sizeof(int32_t) * (size_t)n_pairs);
        if (e != cudaSuccess) return fail(e);
    }
    *out = b;
    return WSB_OK;
}

extern "C" int wsb_batch_create_async(wsb_ctx* ctx, const uint8_t* q_codes, const int64_t* q_off, const int32_t* q_len,
                                      int64_t n_q, const uint8_t* s_codes, const int64_t* s_off, const int32_t* s_len,
                                      int64_t n_s, const int32_t* pair_q, const int32_t* pair_s, int64_t n_pairs,
                                      wsb_batch** out) {
    if (!q_codes || !s_codes) return WSB_E_ARG;
    return batch_create_impl(ctx, q_codes, q_off, q_len, n_q, s_codes, s_off, s_len, n_s, pair_q, pair_s, n_pairs, PackedPools(), out);
}

extern "C" int wsb_batch_create_packed_async(wsb_ctx* ctx, const uint8_t* q_packed, const int64_t* q_flag_pos, int64_t n_q_flags,
                                             const int64_t* q_off, const int32_t* q_len, int64_t n_q,
                                             const uint8_t* s_packed, const int64_t* s_flag_pos, int64_t n_s_flags,
                                             const int64_t* s_off, const int32_t* s_len, int64_t n_s,
                                             const int32_t* pair_q, const int32_t* pair_s, int64_t n_pairs, wsb_batch** out) {
    if (!q_packed || !s_packed || n_q_flags < 0 || n_s_flags < 0 || (n_q_flags > 0 && !q_flag_pos) || (n_s_flags > 0 && !s_flag_pos))
        return WSB_E_ARG;
    PackedPools pk;
    pk.q_packed = q_packed; pk.q_flags = q_flag_pos; pk.n_q_flags = n_q_flags;
    pk.s_packed = s_packed; pk.s_flags = s_flag_pos; pk.n_s_flags = n_s_flags;
    return batch_create_impl(ctx, nullptr, q_off, q_len, n_q, nullptr, s_off, s_len, n_s, pair_q, pair_s, n_pairs, pk, out);
}

extern "C" int wsb_batch_create_uniform_async(wsb_ctx* ctx, const uint8_t* q_codes, const uint8_t* q_packed, int32_t q_len,
                                              const uint8_t* s_codes, const uint8_t* s_packed, int32_t s_len, int64_t n_pairs,
                                              wsb_batch** out) {
    if (q_len < 0 || s_len < 0 || (!q_codes == !q_packed) || (!s_codes == !s_packed) || (!q_codes != !s_codes)) return WSB_E_ARG;
    PackedPools pk;
    pk.q_packed = q_packed; pk.s_packed = s_packed; pk.uniform_q_len = q_len; pk.uniform_s_len = s_len;
    return batch_create_impl(ctx, q_codes, nullptr, nullptr, n_pairs, s_codes, nullptr, nullptr, n_pairs, nullptr, nullptr, n_pairs, pk, out);
}

extern "C" int wsb_batch_create(wsb_ctx* ctx, const uint8_t* q_codes, const int64_t* q_off, const int32_t* q_len,
                                int64_t n_q, const uint8_t* s_codes, const int64_t* s_off, const int32_t* s_len,
                                int64_t n_s, const int32_t* pair_q, const int32_t* pair_s, int64_t n_pairs,
                                wsb_batch** out) {
    if (!ctx) return WSB_E_ARG;
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    int rc = wsb_batch_create_async(ctx, q_codes, q_off, q_len, n_q, s_codes, s_off, s_len, n_s, pair_q, pair_s, n_pairs, out);
    if (rc) return rc;
    (*out)->finish_packer();
    cudaError_t e = cudaStreamSynchronize(ctx->copy_stream);  // host arrays may be reused by the caller after return
    if (e != cudaSuccess) { ctx->last_error = cudaGetErrorString(e); wsb_batch_destroy(*out); *out = nullptr; return WSB_E_CUDA; }
    return WSB_OK;
}

extern "C" int64_t wsb_batch_total_cells(const wsb_batch* b) { return b ? b->total_cells : 0; }
// SM cycles of the last packed int16 short-read launch of this batch (largest per-block clock64 span), 0 if there was none
extern "C" int64_t wsb_batch_kernel_cycles(wsb_batch* b) {
    if (!b || !b->d_cycles || b->cycles_blocks <= 0) return 0;
    std::lock_guard<std::recursive_mutex> lock_(b->ctx->mu);
    std::vector<unsigned long long> h((size_t)b->cycles_blocks);
    if (cudaSetDevice(b->ctx->device) != cudaSuccess) return 0;
    if (cudaMemcpyAsync(h.data(), b->d_cycles, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, b->ctx->stream) != cudaSuccess) return 0;
    if (cudaStreamSynchronize(b->ctx->stream) != cudaSuccess) return 0;
    unsigned long long mx = 0;
    for (auto v : h) mx = std::max(mx, v);
    return (int64_t)mx;
}
extern "C" int64_t wsb_batch_h2d_bytes(const wsb_batch* b) { return b ? b->h2d_bytes + (b->packer ? (int64_t)b->packer->bytes.load() : 0) : 0; }

extern "C" int wsb_batch_plan_stats(const wsb_batch* b, int64_t* out8) {
    if (!b || !out8 || !b->last_plan) return WSB_E_ARG;
    const Plan& pl = *b->last_plan;
    out8[0] = pl.st_stages; out8[1] = pl.st_iters; out8[2] = pl.st_updates;
    out8[3] = pl.st_q_max / 4; out8[4] = pl.st_q_add / 4; out8[5] = pl.st_q_lookup / 4;
    out8[6] = (int64_t)pl.groups.size(); out8[7] = pl.st_pairs;
    return WSB_OK;
}
extern "C" int wsb_batch_has_faults(const wsb_batch* b) { return (b && b->last_plan && b->last_plan->any_error) ? 1 : 0; }

// Page-locked host blocks for result downloads, recycled process-wide (cudaHostAlloc of tens of MB costs milliseconds).
#include <mutex>
static std::mutex g_pin_mu;
static std::multimap<size_t, void*> g_pin_free;
static std::map<void*, size_t> g_pin_live;
extern "C" int wsb_pinned_alloc(size_t bytes, void** out) {
    if (!out) return WSB_E_ARG;
    const size_t want = std::max<size_t>(4096, (bytes + 4095) / 4096 * 4096);
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        auto it = g_pin_free.lower_bound(want);
        if (it != g_pin_free.end() && it->first <= want + want / 2) {
            *out = it->second; g_pin_live[*out] = it->first; g_pin_free.erase(it);
            return WSB_OK;
        }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, want, cudaHostAllocDefault) != cudaSuccess) { (void)cudaGetLastError(); *out = nullptr; return WSB_E_NOMEM; }
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_live[p] = want;
    *out = p;
    return WSB_OK;
}
extern "C" void wsb_pinned_free(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_live.find(p);
    if (it == g_pin_live.end()) return;
    size_t held = 0;
    for (auto& kv : g_pin_free) held += kv.first;
    if (held + it->second > ((size_t)1 << 30)) cudaFreeHost(p);   // keep at most 1 GiB parked
    else g_pin_free.emplace(it->second, p);
    g_pin_live.erase(it);
}

// ------------------------------------------------------------------------------------------------ kernel shapes
struct Shape { int P, K; };
// packed half2 shapes: short reads in a single stage; (8,32) also chains stages for longer packed reads.
// (4,38) halves the wavefront ramp of 150 bp reads but needs ~200 registers: measured slower than (8,19) on B200
// (2 instead of 4 resident blocks per SM), so it is only reachable through WSB_FORCE_SHAPE=3.
static const Shape kShapesF16[] = {{4, 16}, {8, 19}, {8, 32}, {4, 38}, {16, 16}};
// int32 shapes: narrow groups for short reads, full warps with wide stages for long reads
static const Shape kShapesI32[] = {{8, 16}, {16, 16}, {32, 16}, {8, 19}};
// packed int16 short-read kernels.  (16, 10) is the LATENCY shape: twice the lanes per unit, strips half as long; 22 % more
// instructions per cell, but a batch that leaves most SMs with less than one block of (8, K) groups finishes ~20 % sooner.
// Chosen per launch group, latency_shape().
static const Shape kShapesS16[] = {{8, 16}, {8, 19}, {16, 10}};
static Shape shape_of(int variant, int shape);
constexpr int kNumShapesF16 = 3, kNumShapesI32 = 4;  // shapes the planner may choose
constexpr int kNumShapes = 5;  // bucket array bound

static Shape shape_of(int variant, int shape) {
    return variant == WSB_VARIANT_F16X2 ? kShapesF16[shape] : variant == WSB_VARIANT_S16X2 ? kShapesS16[shape] : kShapesI32[shape];
}

// A packed int16 short-read launch group of at most 1.5 blocks of (8, K) lane groups per SM runs on (16, 10) lane groups
// instead: twice the blocks, strips half as long (WSB_S16_LAT = 0: never, 2: always; tuning aid).  Measured (B200, 150 bp,
// kernel time, (8, 19) against (16, 10)): 2 000 pairs 35 / 28 us (global linear), 48 / 37 us (local affine); 4 700 pairs
// 35 / 31 and 45 / 39; 6 000 pairs 40 / 36 and 52 / 48; at 10 000 pairs the wide shape's 22 % extra instructions lose:
// 54 / 59 and 72 / 81 us.
static int latency_shape(int shape, int64_t n_units, int max_m, int sm_count) {
    static const char* lat = getenv("WSB_S16_LAT");
    const int mode = (lat && lat[0]) ? atoi(lat) : 1;
    if (mode == 0 || max_m < 2) return shape;
    return (mode >= 2 || n_units * 2 <= (int64_t)sm_count * 3 * (kThreads / 8)) ? 2 : shape;
}

static double padded_cost(const Shape& s, int m, int n) {
    const int w = s.P * s.K;
    const int stages = (n + w - 1) / w;
    return (double)(m + s.P - 1) * stages * w;
}

static int best_shape(const Shape* shapes, int count, int table_size, int m, int n) {
    static const char* force = getenv("WSB_FORCE_SHAPE");  // tuning aid: index into the shape table
    if (force && force[0]) return std::min(table_size - 1, std::max(0, atoi(force)));
    int best = 0;
    double bc = padded_cost(shapes[0], m, n);
    for (int k = 1; k < count; ++k) {
        const double c = padded_cost(shapes[k], m, n);
        if (c < bc) { bc = c; best = k; }
    }
    return best;
}


template <class AR, int P, int K, int GAP> static KernelSel pick_atype(int atype, bool masked) {
    switch (atype) {
        case AT_GLOBAL: return {score_kernel<AR, P, K, AT_GLOBAL, GAP>, score_smem_bytes<AR, P, K, AT_GLOBAL>()};
        case AT_LOCAL:
            if constexpr (!std::is_same<AR, ArF16>::value) {
                if (masked) return {score_kernel<AR, P, K, AT_LOCAL, GAP, true>, score_smem_bytes<AR, P, K, AT_LOCAL>()};
            }
            return {score_kernel<AR, P, K, AT_LOCAL, GAP>, score_smem_bytes<AR, P, K, AT_LOCAL>()};
        default: return {score_kernel<AR, P, K, AT_SEMI, GAP>, score_smem_bytes<AR, P, K, AT_SEMI>()};
    }
}

template <class AR, int P, int K> static KernelSel pick_gap(int atype, int gap, bool masked) {
    if (gap == GAP_LINEAR) return pick_atype<AR, P, K, GAP_LINEAR>(atype, masked);
    if (gap == GAP_MERGED) return pick_atype<AR, P, K, GAP_MERGED>(atype, masked);
    if constexpr (!std::is_same<AR, ArF16>::value) return pick_atype<AR, P, K, GAP_EXACT>(atype, masked);
    return {nullptr, 0};  // the packed kernels have no exact three-state model
}

template <int P, int K> static KernelSel pick_short(int gap) {
    if (gap == GAP_LINEAR) return {f16_local_short_kernel<P, K, GAP_LINEAR>, short_smem_bytes<P, K>()};
    return {f16_local_short_kernel<P, K, GAP_MERGED>, short_smem_bytes<P, K>()};
}

template <int GAP, bool CLUSTER> static LongFn pick_long_atype(int atype) {
    switch (atype) {
        case AT_GLOBAL: return score_long_kernel<AT_GLOBAL, GAP, CLUSTER>;
        case AT_LOCAL: return score_long_kernel<AT_LOCAL, GAP, CLUSTER>;
        default: return score_long_kernel<AT_SEMI, GAP, CLUSTER>;
    }
}
static LongFn pick_long(int atype, int gap, bool cluster) {
    if (gap == GAP_LINEAR) return cluster ? pick_long_atype<GAP_LINEAR, true>(atype) : pick_long_atype<GAP_LINEAR, false>(atype);
    if (gap == GAP_MERGED) return cluster ? pick_long_atype<GAP_MERGED, true>(atype) : pick_long_atype<GAP_MERGED, false>(atype);
    return nullptr;
}

// Can a cluster of 16 blocks x 16 warps of the long-read kernel be resident?  (non-portable cluster size: opt-in per kernel)
static bool probe_cluster16(wsb_ctx* ctx) {
    if (ctx->cluster16 >= 0) return ctx->cluster16 == 1;
    ctx->cluster16 = 0;
    LongFn fn = pick_long(AT_LOCAL, GAP_MERGED, true);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16); cfg.blockDim = dim3(kLongMaxWarps * 32);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n >= 1) ctx->cluster16 = 1;
    }
    (void)cudaGetLastError();
    return ctx->cluster16 == 1;
}

// The packed int16 short-read kernels live in their own translation unit (wsb200_s16.cu, built with -Xptxas -O1: ptxas'
// default scheduling costs those two kernels 3-4 %, every other kernel is at its best with the default).
namespace wsb {
KernelSel pick_short16_local(int shape, int gap, int alpha, int gamma);
KernelSel pick_short16_global(int shape, int gap, int alpha, int gamma, bool ragged);
}

namespace wsb { LongFn pick_long16(int atype, int gap, int alpha, int gamma); }   // score_long16.cuh, compiled in wsb200_s16.cu

// short_ok: every unit of the launch fits one stage and the short kernel's query buffer
static KernelSel pick_kernel(int variant, int shape, int atype, int gap, bool masked, bool short_ok, bool wide,
                             int alpha = 0, int gamma = 0, bool ragged = true) {
    static const char* no_short = getenv("WSB_NO_SHORT");  // tuning aid: force the general kernel
    if (variant == WSB_VARIANT_S16X2 && atype == AT_GLOBAL) {
        return pick_short16_global(shape, gap, alpha, gamma, ragged);
    }
    if (variant == WSB_VARIANT_S16X2) {
        return pick_short16_local(shape, gap, alpha, gamma);
    }
    if (variant == WSB_VARIANT_F16X2 && atype == AT_LOCAL && short_ok && !(no_short && no_short[0])) {
        switch (shape) {
            case 0: return pick_short<4, 16>(gap);
            case 1: return pick_short<8, 19>(gap);
            case 2: return pick_short<8, 32>(gap);
            case 3: return pick_short<4, 38>(gap);
            default: return pick_short<16, 16>(gap);
        }
    }
    if (variant == WSB_VARIANT_F16X2) {
        switch (shape) {
            case 0: return pick_gap<ArF16, 4, 16>(atype, gap, masked);
            case 1: return pick_gap<ArF16, 8, 19>(atype, gap, masked);
            case 2: return pick_gap<ArF16, 8, 32>(atype, gap, masked);
            case 3: return pick_gap<ArF16, 4, 38>(atype, gap, masked);
            default: return pick_gap<ArF16, 16, 16>(atype, gap, masked);
        }
    }
    if (wide) return pick_gap<ArI32W, 8, 16>(atype, gap, masked);  // |match - mismatch| > 127: compare/select kernel
    switch (shape) {
        case 0: return pick_gap<ArI32, 8, 16>(atype, gap, masked);
        case 1: return pick_gap<ArI32, 16, 16>(atype, gap, masked);
        case 2: return pick_gap<ArI32, 32, 16>(atype, gap, masked);
        default: return pick_gap<ArI32, 8, 19>(atype, gap, masked);
    }
}


// Per-cell instruction mix of the kernel a launch group runs, in quarter thread-instructions per matrix cell: {max, add /
// sub, substitution lookup}.  These are the cell bodies of the kernels; tests/test_cpu_host.py pins the
// packed int16 rows against the SASS of the built library.
static void op_mix_q(const LaunchGroup& g, int atype, int& qmax, int& qadd, int& qlook) {
    const bool local = atype == AT_LOCAL, merged = g.gap == GAP_MERGED, exact = g.gap == GAP_EXACT;
    if (g.long_nw > 0) {
        if (g.long16) { qmax = (merged ? 4 : 2) + (local ? 1 : 0); qadd = merged ? 6 : 4; qlook = 2; }
        else { qmax = (merged ? 8 : 4) + (local ? 2 : 0); qadd = merged ? 8 : 4; qlook = 4; }
        return;
    }
    if (g.variant == WSB_VARIANT_S16X2) {   // PRMT + VIADD + (2 | 1) VIMNMX3 + (2 | 1) VIADD per two cells, local: + half a VIMNMX3
        qmax = (merged ? 4 : 2) + (local ? 1 : 0); qadd = merged ? 6 : 4; qlook = 2;
        return;
    }
    if (g.variant == WSB_VARIANT_F16X2) {
        const Shape sh = kShapesF16[g.shape];
        const bool short_ok = local && g.max_n <= sh.P * sh.K && g.max_m <= kShortQRows - 4 * sh.P - 2;
        if (short_ok) { qmax = merged ? 5 : 3; qadd = merged ? 8 : 6; qlook = 2; }
        else { qmax = (merged ? 6 : 4) + (local ? 2 : 0); qadd = merged ? 8 : 6; qlook = 2; }
        return;
    }
    qmax = (exact ? 12 : merged ? 12 : 8) + (local ? 4 : 0); qadd = exact ? 20 : 4; qlook = 4;
}

// ------------------------------------------------------------------------------------------------ planner
// Length-bucketing partitioner: classify every pair (variant by value range, kernel shape by padded work), sort each
// class by work so neighbouring lane groups (and the two halves of a packed unit) carry near-equal loads, and emit one
// launch group per (variant, shape).  Replaces batch._plan_units / _chunk_units (batch.py:118-164).
static int build_plan(wsb_batch* b, const wsb_scheme* sch, int atype, int variant, Plan& plan, bool want_s16) {
    wsb_ctx* ctx = b->ctx;
    const int64_t np = b->n_pairs;
    const bool affine = sch->gap_model == WSB_GAP_AFFINE;
    const bool merged_ok = !affine || wsb_merged_state_exact(sch);
    // the packed kernel's junk-cell argument needs never-matching pads to be non-improving
    const bool f16_scheme_ok = merged_ok && sch->mismatch <= 0 && sch->match >= 0;
    const int gap_i32 = !affine ? GAP_LINEAR : (wsb_merged_state_exact(sch) ? GAP_MERGED : GAP_EXACT);
    const int gap_f16 = !affine ? GAP_LINEAR : GAP_MERGED;
    const int ms = max_step(sch);
    const int beta_eff_plan = affine ? sch->gap_extend : sch->gap_open;
    const bool wide_scheme = std::abs(sch->match - sch->mismatch) > 127;
    // (the snapshot of the packed int16 kernel holds T - alpha: it needs every gap step to cost something)
    const bool s16_ok = want_s16 && atype == AT_LOCAL && f16_scheme_ok && std::abs(sch->match) <= 127 &&
                        std::abs(sch->mismatch) <= 127 && sch->gap_open >= 1 && (!affine || sch->gap_extend >= 1);
    // global alignment of short reads: no pad argument needed (pads sit right of / below every real cell), values in 16 bits
    const bool s16g_ok = want_s16 && atype == AT_GLOBAL && merged_ok && !wide_scheme && std::abs(sch->match) <= 127 &&
                         std::abs(sch->mismatch) <= 127;
    plan.status.assign((size_t)np, 0);

    if (variant == WSB_VARIANT_F16X2 && !merged_ok) return WSB_E_SCHEME;

    auto classify = [&](int m, int n, int& var, int& shape, int& status) {
        status = 0; var = -1; shape = 0;
        if (m == 0 || n == 0) return;  // empty side: resolved on the host below, never launched
        if ((int64_t)ms * ((int64_t)m + n) >= (1ll << 29)) { status = WSB_E_LENGTH; return; }
        const bool fits = f16_scheme_ok && wsb_f16_range_ok(sch, m, n);
        if (variant == WSB_VARIANT_F16X2 && !fits) { status = WSB_E_RANGE; return; }
        if (variant == WSB_VARIANT_AUTO && fits && s16_ok && n <= 152 && m <= kShort16MaxM) {
            var = WSB_VARIANT_S16X2; shape = n <= 128 ? 0 : 1;
            static const char* s16_shape = getenv("WSB_S16_SHAPE");   // tuning aid: lane-group shape / occupancy of the packed int16 kernel
            if (s16_shape && s16_shape[0]) shape = std::min(1, std::max(0, atoi(s16_shape)));   // packed int16 DPX kernel: same pairs as the half2 short kernel
        } else if (variant == WSB_VARIANT_AUTO && s16g_ok && n <= 152 && m <= kShort16MaxM &&
                   (int64_t)std::abs(sch->match) * std::min(m, n) + std::abs(sch->mismatch) <= 16000 &&
                   3ll * sch->gap_open + (int64_t)beta_eff_plan * (m + n) + std::abs(sch->mismatch) <= 16000) {
            var = WSB_VARIANT_S16X2; shape = n <= 128 ? 0 : 1;
        } else if (variant != WSB_VARIANT_I32 && fits) { var = WSB_VARIANT_F16X2; shape = best_shape(kShapesF16, kNumShapesF16, 5, m, n); }
        else { var = WSB_VARIANT_I32; shape = wide_scheme ? 0 : best_shape(kShapesI32, kNumShapesI32, 4, m, n); }
    };
    // The long-read kernel (score_long.cuh) takes the int32 pairs that would otherwise run full-warp stages: it needs
    // byte-sized substitution scores, the merged (or linear) gap state and, for local alignment, non-improving pads.
    static const char* no_long = getenv("WSB_NO_LONG");
    const bool long_scheme_ok = !(no_long && no_long[0]) && gap_i32 != GAP_EXACT && std::abs(sch->match) <= 127 &&
                                std::abs(sch->mismatch) <= 127 && (atype != AT_LOCAL || (sch->mismatch <= 0 && sch->match >= 0));
    auto long_ok = [&](int var, int shape, int m, int n) {
        (void)shape;
        if (!long_scheme_ok || var != WSB_VARIANT_I32 || m < 64) return false;
        static const char* thr = getenv("WSB_LONG_MIN_N");  // tuning aid: take everything wider than this
        if (thr && thr[0]) return n > atoi(thr);
        // 512-column stages: below ~2 kbp the narrow lane groups of score_kernel win unless the width fits well
        // (measured crossover, tools/len_sweep.py)
        const int64_t padded = (int64_t)((n + kLongW - 1) / kLongW) * kLongW;
        return n > 2048 || (n > 512 && padded * 100 <= (int64_t)n * 115);
    };

    // geometry counters: per unit the stages of its subject, the wavefront trips of its sweep(s) and the cell updates the
    // lockstep sweep executes, padding included (the reference's definition, tests/test_engine.py:223-233)
    auto account_plan = [&](Plan& pl, const std::vector<int32_t>& unit_list) {
        for (const LaunchGroup& g : pl.groups) {
            const int nv = (g.long_nw > 0) ? (g.long16 ? 2 : 1) : (g.variant == WSB_VARIANT_I32 ? 1 : 2);
            const int P = g.long_nw > 0 ? 32 : shape_of(g.variant, g.shape).P;
            const int W = g.long_nw > 0 ? kLongW : P * shape_of(g.variant, g.shape).K;
            int qmax, qadd, qlook;
            op_mix_q(g, atype, qmax, qadd, qlook);
            for (int64_t u = 0; u < g.n_units; ++u) {
                int mu = 0, nu = 0, live = 0;
                for (int v = 0; v < nv; ++v) {
                    int64_t pr;
                    if (g.unit_off < 0) { pr = u * nv + v; if (pr >= np) pr = -1; }
                    else pr = unit_list[(size_t)(g.unit_off + u * nv + v)];
                    if (pr < 0) continue;
                    mu = std::max(mu, (int)b->m[pr]); nu = std::max(nu, (int)b->n[pr]); ++live;
                }
                if (!live) continue;
                const int64_t stages = (nu + W - 1) / W;
                const int64_t updates = stages * (int64_t)mu * W * nv;
                pl.st_stages += stages; pl.st_iters += stages * (mu + P - 1); pl.st_updates += updates; pl.st_pairs += live;
                pl.st_q_max += updates * qmax; pl.st_q_add += updates * qadd; pl.st_q_lookup += updates * qlook;
                if (g.unit_off < 0) {   // identical units: multiply instead of looping over millions of them
                    const int64_t rest = g.n_units - 1 - (np % nv ? 1 : 0);
                    if (u == 0 && rest > 0) {
                        pl.st_stages += stages * rest; pl.st_iters += stages * (mu + P - 1) * rest; pl.st_updates += updates * rest;
                        pl.st_pairs += (int64_t)live * rest;
                        pl.st_q_max += updates * qmax * rest; pl.st_q_add += updates * qadd * rest; pl.st_q_lookup += updates * qlook * rest;
                        u += rest;
                    }
                }
            }
        }
    };

    if (b->uniform) {
        int var, shape, status;
        classify(b->m[0], b->n[0], var, shape, status);
        if (status) { std::fill(plan.status.begin(), plan.status.end(), status); plan.any_error = true; return WSB_OK; }
        if (var < 0) return WSB_OK;
        if (!long_ok(var, shape, b->m[0], b->n[0])) {
            LaunchGroup g;
            g.variant = var; g.shape = shape; g.gap = var == WSB_VARIANT_I32 ? gap_i32 : gap_f16;
            g.n_units = var == WSB_VARIANT_I32 ? np : (np + 1) / 2;
            g.unit_off = -1; g.max_m = b->m[0]; g.max_n = b->n[0];
            if (var == WSB_VARIANT_S16X2) g.shape = latency_shape(g.shape, g.n_units, g.max_m, ctx->sm_count);
            plan.groups.push_back(g);
            account_plan(plan, std::vector<int32_t>());
            return WSB_OK;
        }
    }

    // general path: bucket, sort by work (descending), pair neighbours
    std::vector<int64_t> bucket[3][kNumShapes];   // class 0 = half2, 1 = int32, 2 = packed int16
    std::vector<int64_t> long_pairs;
    double long_iters = 0.0;  // single-warp iterations of all long-class pairs
    for (int64_t p = 0; p < np; ++p) {
        int var, shape, status;
        classify(b->m[p], b->n[p], var, shape, status);
        if (status) { plan.status[p] = status; plan.any_error = true; continue; }
        if (var < 0) continue;
        if (long_ok(var, shape, b->m[p], b->n[p])) {
            long_pairs.push_back(p);
            long_iters += (double)((b->n[p] + kLongW - 1) / kLongW) * (b->m[p] + 31);
        } else {
            bucket[var == WSB_VARIANT_F16X2 ? 0 : var == WSB_VARIANT_S16X2 ? 2 : 1][shape].push_back(p);
        }
    }
    std::vector<int32_t> units;
    auto by_work = [&](int64_t x, int64_t y) {
        const int64_t cx = (int64_t)b->m[x] * b->n[x], cy = (int64_t)b->m[y] * b->n[y];
        if (cx != cy) return cx > cy;
        return b->n[x] > b->n[y];
    };
    // long-read pairs: warps per pair.  A pair must not outlast a fraction of the whole launch's makespan (so the
    // giants of a skewed batch get up to 16 warps), beyond that the cheapest count in warp-iterations wins (pipeline
    // fill of ~80 rows per extra warp, idle warps when the stage count is not a multiple).
    if (!long_pairs.empty()) {
        // Packed int16 units: two long pairs of identical shape whose values fit 16 bits run in the halves of one
        // register set (score_long16.cuh); everything else runs one pair per block / cluster in int32.
        static const char* no_l16 = getenv("WSB_NO_LONG16");  // tuning aid
        const bool l16_scheme = variant == WSB_VARIANT_AUTO && !(no_l16 && no_l16[0]);
        std::vector<int64_t> cand, singles;
        for (int64_t p : long_pairs) {
            // 16-bit value range: scores rise by at most match per diagonal step, and no value falls below the all-gap
            // path (2 alpha + beta (m + n)) by more than one open / mismatch (local: nothing falls below -alpha)
            const int64_t mm = b->m[p], nn = b->n[p];
            const int64_t hi = (int64_t)std::max(sch->match, 0) * std::min(mm, nn) + sch->gap_open + beta_eff_plan;
            const int64_t lo = atype == AT_LOCAL ? sch->gap_open
                                                 : 3ll * sch->gap_open + (int64_t)beta_eff_plan * (mm + nn) + std::abs(sch->mismatch);
            const bool fits16 = l16_scheme && hi <= 32000 && lo <= 32000;
            (fits16 ? cand : singles).push_back(p);
        }
        // A unit is two pairs of identical shape.  (The kernel also takes local pairs of different shapes -- the shorter
        // alignment then sees pads -- but pairing near-equal neighbours of a skewed batch measured 8 % slower than
        // running them one per block in int32: cfg5 2942 vs 3196 GCUPS.)
        std::stable_sort(cand.begin(), cand.end(), [&](int64_t x, int64_t y) {
            if (b->n[x] != b->n[y]) return b->n[x] > b->n[y];
            return b->m[x] > b->m[y];
        });
        std::vector<std::pair<int64_t, int64_t>> twins;   // units of the packed kernel
        for (size_t k = 0; k < cand.size();) {
            if (k + 1 < cand.size() && b->n[cand[k]] == b->n[cand[k + 1]] && b->m[cand[k]] == b->m[cand[k + 1]]) {
                twins.emplace_back(cand[k], cand[k + 1]); k += 2;
            } else { singles.push_back(cand[k]); ++k; }
        }
        // class index = log2(warps per pair): 0..4 -> 1..16 warps in one block, 5..8 -> clusters of 2, 4, 8, 16 blocks x 16 warps
        // (16: the non-portable cluster size, where the device schedules it)
        std::vector<int64_t> by_class[9];
        std::vector<std::pair<int64_t, int64_t>> twins_by_class[5];
        const double machine_warps = (double)ctx->sm_count * 20.0;
        const double makespan = std::max(long_iters / machine_warps, 1.0);
        static const char* no_cluster = getenv("WSB_NO_CLUSTER");  // tuning aid
        // Clusters of 16 blocks (non-portable size) are opt-in (WSB_CLUSTER16=1): measured on cfg5's 8-way shards they lose
        // (a shard holds ~16 pairs of that class; 7 clusters of 16 are co-resident against 15 of 8: 164 ms per shard
        // against 140 ms), and on the whole batch too (679 against 622 ms).
        static const char* want_cluster16 = getenv("WSB_CLUSTER16");
        const int max_class = (no_cluster && no_cluster[0]) ? 4 : (want_cluster16 && want_cluster16[0] == '1' && probe_cluster16(ctx)) ? 8 : 7;
        auto pick_class = [&](int64_t p, int top) {
            const int stages = (b->n[p] + kLongW - 1) / kLongW;
            const double t1 = (double)stages * (b->m[p] + 31);
            // warps per pair come from powers of two: blocks then spread evenly over the four schedulers of an SM
            // ... but a cluster only up to about twice the pair's proportional share of the machine, or a few giants that
            // dominate the batch would queue behind each other in half-idle clusters
            static const double share_factor = [] { const char* e = getenv("WSB_SHARE_CAP"); return e ? atof(e) : 2.0; }();   // tuning aid
            const double share_cap = std::max(1.0, share_factor * t1 / std::max(long_iters, 1.0) * machine_warps);
            int lo = 0;
            // (the step to 16 blocks is taken as soon as 128 warps no longer cover the stages in one round: a 100 kbp subject
            // has 196 stages)
            while (lo < top && ((2 << lo) <= stages || (lo == 7 && stages > (1 << lo))) && (lo < 4 || (double)(2 << lo) <= share_cap) &&
                   t1 / (1 << lo) > 0.25 * makespan) ++lo;
            int best = lo;
            double best_cost = 1e300;
            for (int c = lo; c <= std::min(lo + 1, std::min(top, 4)); ++c) {   // one block: also weigh the next size up
                const int nw = 1 << c;
                if (nw > stages) break;
                const double rounds = (double)((stages + nw - 1) / nw);
                const double cost = nw * (rounds * (b->m[p] + 31) + (nw - 1) * 100.0);
                if (cost < best_cost * 0.999) { best_cost = cost; best = c; }
            }
            if (lo > 4) best = lo;
            return best;
        };
        for (int64_t p : singles) by_class[pick_class(p, max_class)].push_back(p);
        for (auto& tw : twins) twins_by_class[pick_class(tw.first, 4)].push_back(tw);
        for (int c = 4; c >= 0; --c) {
            auto& v = twins_by_class[c];
            if (v.empty()) continue;
            std::stable_sort(v.begin(), v.end(), [&](const std::pair<int64_t, int64_t>& x, const std::pair<int64_t, int64_t>& y) {
                return by_work(x.first, y.first);
            });
            LaunchGroup g;
            g.variant = WSB_VARIANT_I32; g.shape = 2; g.gap = gap_i32; g.long_nw = 1 << c; g.long16 = true;
            g.unit_off = (int64_t)units.size();
            g.n_units = (int64_t)v.size();
            for (auto& tw : v) {
                g.max_m = std::max({g.max_m, b->m[tw.first], b->m[tw.second]});
                g.max_n = std::max({g.max_n, b->n[tw.first], b->n[tw.second]});
                units.push_back((int32_t)tw.first); units.push_back((int32_t)tw.second);
            }
            plan.groups.push_back(g);
        }
        for (int c = 8; c >= 0; --c) {
            auto& v = by_class[c];
            if (v.empty()) continue;
            std::stable_sort(v.begin(), v.end(), by_work);
            LaunchGroup g;
            g.variant = WSB_VARIANT_I32; g.shape = 2; g.gap = gap_i32;
            g.long_nw = c <= 4 ? 1 << c : kLongMaxWarps;
            g.cluster = c <= 4 ? 1 : 1 << (c - 4);
            g.unit_off = (int64_t)units.size();
            g.n_units = (int64_t)v.size();
            for (int64_t p : v) {
                g.max_m = std::max(g.max_m, b->m[p]); g.max_n = std::max(g.max_n, b->n[p]);
                units.push_back((int32_t)p);
            }
            plan.groups.push_back(g);
        }
    }
    for (int cls = 0; cls < 3; ++cls)
        for (int s = 0; s < kNumShapes; ++s) {
            auto& v = bucket[cls][s];
            if (v.empty()) continue;
            std::stable_sort(v.begin(), v.end(), by_work);
            LaunchGroup g;
            g.variant = cls == 0 ? WSB_VARIANT_F16X2 : cls == 2 ? WSB_VARIANT_S16X2 : WSB_VARIANT_I32;
            g.shape = s; g.gap = cls == 1 ? gap_i32 : gap_f16;
            g.unit_off = (int64_t)units.size();
            for (int64_t p : v) { g.max_m = std::max(g.max_m, b->m[p]); g.max_n = std::max(g.max_n, b->n[p]); }
            if (cls != 1) {
                g.n_units = ((int64_t)v.size() + 1) / 2;
                if (cls == 2) g.shape = latency_shape(g.shape, g.n_units, g.max_m, ctx->sm_count);
                for (size_t k = 0; k < v.size(); k += 2) {
                    units.push_back((int32_t)v[k]);
                    units.push_back(k + 1 < v.size() ? (int32_t)v[k + 1] : -1);
                }
            } else {
                g.n_units = (int64_t)v.size();
                for (int64_t p : v) units.push_back((int32_t)p);
            }
            plan.groups.push_back(g);
        }
    account_plan(plan, units);
    if (!units.empty()) {
        plan.h_units = std::move(units);
        CUDA_TRY(ctx, ctx->alloc((void**)&plan.d_units, plan.h_units.size() * sizeof(int32_t)));
        CUDA_TRY(ctx, cudaMemcpyAsync(plan.d_units, plan.h_units.data(), plan.h_units.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                      ctx->stream));
    }
    return WSB_OK;
}

// pairs with an empty side never reach the device (engine.py:281-288); fill their slots after the kernels
__global__ void empty_side_kernel(const int32_t* pair_q, const int32_t* pair_s, const int32_t* q_len, const int32_t* s_len,
                                  int64_t n_pairs, int atype, int affine, int alpha, int beta, int32_t* out_score,
                                  int32_t* out_i, int32_t* out_j) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_pairs) return;
    const int m = q_len[pair_q[p]], n = s_len[pair_s[p]];
    if (m != 0 && n != 0) return;
    if (atype == AT_GLOBAL) {
        const int len = m == 0 ? n : m;
        const int cost = len <= 0 ? 0 : (affine ? alpha + (len - 1) * beta : alpha * len);
        out_score[p] = -cost; out_i[p] = m; out_j[p] = n;
    } else if (atype == AT_LOCAL) {
        out_score[p] = 0; out_i[p] = 0; out_j[p] = 0;
    } else {
        out_score[p] = 0; out_i[p] = 0; out_j[p] = m == 0 ? n : 0;
    }
}

static int check_scheme(const wsb_scheme* s, int atype) {
    if (!s) return WSB_E_ARG;
    if (atype < 0 || atype > 2) return WSB_E_ARG;
    if (s->gap_model != WSB_GAP_LINEAR && s->gap_model != WSB_GAP_AFFINE) return WSB_E_ARG;
    if (s->gap_open < 0 || s->gap_extend < 0) return WSB_E_ARG;
    return WSB_OK;
}

// plan_only: build (or reuse) the plan and resolve empty-side pairs, but launch no score kernel (the traceback fill of
// global / semiglobal alignments produces score and end cell itself)
struct FetchDst { int32_t* score = nullptr; int32_t* i = nullptr; int32_t* j = nullptr; bool done = false; bool mapped = false; };

// 16-byte vector copies of three result arrays into page-locked host memory (unified addressing: same pointer on the device)
__global__ void results_home_kernel(const int32_t* s0, const int32_t* s1, const int32_t* s2, int32_t* d0, int32_t* d1, int32_t* d2,
                                    int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x, first = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(s0) | reinterpret_cast<uintptr_t>(s1) | reinterpret_cast<uintptr_t>(s2) |
                       reinterpret_cast<uintptr_t>(d0) | reinterpret_cast<uintptr_t>(d1) | reinterpret_cast<uintptr_t>(d2)) & 15) == 0;
    const int64_t n4 = vec ? n / 4 : 0;
    for (int64_t k = first; k < n4; k += stride) {
        reinterpret_cast<int4*>(d0)[k] = reinterpret_cast<const int4*>(s0)[k];
        reinterpret_cast<int4*>(d1)[k] = reinterpret_cast<const int4*>(s1)[k];
        reinterpret_cast<int4*>(d2)[k] = reinterpret_cast<const int4*>(s2)[k];
    }
    for (int64_t k = n4 * 4 + first; k < n; k += stride) { d0[k] = s0[k]; d1[k] = s1[k]; d2[k] = s2[k]; }
}

static int batch_score_impl(wsb_batch* b, const wsb_scheme* sch, int atype, int variant, float* kernel_ms,
                            int32_t* n_launches, bool plan_only, FetchDst* fetch = nullptr) {
    if (!b) return WSB_E_ARG;
    std::lock_guard<std::recursive_mutex> lock_(b->ctx->mu);
    int rc = check_scheme(sch, atype);
    if (rc) return rc;
    if (variant < WSB_VARIANT_AUTO || variant > WSB_VARIANT_S16X2) return WSB_E_ARG;
    // S16X2 is routed like AUTO; both give short local pairs to the packed int16 kernel (WSB_NO_S16: tuning aid, AUTO then
    // keeps the half2 short kernel)
    static const char* no_s16 = getenv("WSB_NO_S16");
    const bool want_s16 = variant == WSB_VARIANT_S16X2 || (variant == WSB_VARIANT_AUTO && !(no_s16 && no_s16[0]));
    if (variant == WSB_VARIANT_S16X2) variant = WSB_VARIANT_AUTO;
    wsb_ctx* ctx = b->ctx;
    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const bool affine = sch->gap_model == WSB_GAP_AFFINE;
    const int beta_eff = affine ? sch->gap_extend : sch->gap_open;

    auto key = std::make_tuple(sch->match, sch->mismatch, sch->gap_open, sch->gap_extend, sch->gap_model, atype,
                               want_s16 ? (int)WSB_VARIANT_S16X2 : variant);
    auto it = b->plans.find(key);
    if (it == b->plans.end()) {
        Plan plan;
        rc = build_plan(b, sch, atype, variant, plan, want_s16);
        if (rc) { if (plan.d_units) ctx->release(plan.d_units); return rc; }
        it = b->plans.emplace(key, std::move(plan)).first;
    }
    const Plan& plan = it->second;
    b->last_plan = &plan;

    bool any_l16 = false;
    int l16_gap = GAP_MERGED;
    int64_t l16_rows = 0;
    size_t l16_bnd_off = 0;
    const int l16_redo_nw = 4, l16_redo_grid = ctx->sm_count * 2;
    // launch geometry + border scratch (every launch group owns a slice: long-read groups run concurrently)
    struct Geo { KernelFn fn; LongFn lfn; size_t smem; int grid; int64_t bnd_rows; size_t bnd_off; };
    std::vector<Geo> geo;
    size_t bnd_need = 0;
    for (const LaunchGroup& g : plan.groups) {
        if (g.long_nw > 0) {
            LongFn lfn = g.long16 ? pick_long16(atype, g.gap, sch->gap_open, affine ? std::min(sch->gap_open, sch->gap_extend) : sch->gap_open)
                                  : pick_long(atype, g.gap, g.cluster > 1);
            if (!lfn) return WSB_E_SCHEME;
            int grid = 1;
            if (g.cluster > 1) {  // one pair per cluster: as many clusters as the device can co-schedule
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3((unsigned)(g.cluster * std::min<int64_t>(g.n_units, 1024)));
                cfg.blockDim = dim3((unsigned)(g.long_nw * 32));
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = (unsigned)g.cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                cfg.attrs = at; cfg.numAttrs = 1;
                int max_clusters = 0;
                if (g.cluster > 8) CUDA_TRY(ctx, cudaFuncSetAttribute(lfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                CUDA_TRY(ctx, cudaOccupancyMaxActiveClusters(&max_clusters, lfn, &cfg));
                max_clusters = std::max(1, std::min(max_clusters, kLongCfClusters));   // flag blocks per cluster size
                grid = g.cluster * (int)std::min<int64_t>(g.n_units, max_clusters);
            } else {
                int per_sm = 0;
                CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lfn, g.long_nw * 32, 0));
                per_sm = std::max(per_sm, 1);
                static const char* occ = getenv("WSB_LONG_MAX_BLOCKS");  // tuning aid: cap resident blocks per SM
                if (occ && occ[0]) per_sm = std::max(1, std::min(per_sm, atoi(occ)));
                grid = (int)std::max<int64_t>(1, std::min<int64_t>(g.n_units, (int64_t)ctx->sm_count * per_sm));
            }
            const int64_t rows = ((int64_t)g.max_m + 31) / 32 * 32 + 64;
            geo.push_back({nullptr, lfn, 0, grid, rows, bnd_need});
            bnd_need += (size_t)rows * sizeof(int2) * (size_t)(g.long_nw * g.cluster + 1) * (size_t)(grid / g.cluster);
            continue;
        }
        const Shape sh = shape_of(g.variant, g.shape);
        const bool short_ok = g.max_n <= sh.P * sh.K && g.max_m <= kShortQRows - 4 * sh.P - 2;
        const KernelSel sel = pick_kernel(g.variant, g.shape, atype, g.gap, sch->mismatch > 0 || sch->match < 0, short_ok,
                                          std::abs(sch->match - sch->mismatch) > 127, sch->gap_open,
                                          affine ? std::min(sch->gap_open, sch->gap_extend) : sch->gap_open,
                                          /*ragged=*/g.unit_off >= 0 || g.max_m < 2 * sh.P);
        KernelFn fn = sel.fn;
        if (!fn) return WSB_E_SCHEME;
        CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel.smem));
        int per_sm = 0;
        CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, sel.smem));
        per_sm = std::max(per_sm, 1);
        const int gpb = kThreads / sh.P;
        const int64_t blocks_needed = (g.n_units + gpb - 1) / gpb;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks_needed, (int64_t)ctx->sm_count * per_sm));
        const bool multi_stage = g.max_n > sh.P * sh.K;
        const int64_t rows = multi_stage ? (int64_t)g.max_m + 2 : 0;
        geo.push_back({fn, nullptr, sel.smem, grid, rows, bnd_need});
        bnd_need += ((size_t)rows * 8u * (size_t)grid * gpb + 255) / 256 * 256;
    }
    {   // the packed int16 long-read kernel may hand pairs back: scratch for their int32 re-score launch
        int64_t rows16 = 0;
        for (size_t k = 0; k < plan.groups.size(); ++k) if (plan.groups[k].long16) rows16 = std::max(rows16, geo[k].bnd_rows);
        if (rows16 > 0 && !plan_only) {
            l16_bnd_off = bnd_need;
            bnd_need += (size_t)rows16 * sizeof(int2) * (size_t)(l16_redo_nw + 1) * (size_t)l16_redo_grid;
            if (!b->d_redo_long) CUDA_TRY(ctx, ctx->alloc((void**)&b->d_redo_long, sizeof(int32_t) * (size_t)(b->n_pairs + 8)));
            CUDA_TRY(ctx, cudaMemsetAsync(b->d_redo_long, 0, 16, ctx->stream));
        }
    }
    if (bnd_need > b->bnd_bytes) {
        if (b->d_bnd) { ctx->release(b->d_bnd); b->d_bnd = nullptr; b->bnd_bytes = 0; }
        CUDA_TRY(ctx, ctx->alloc(&b->d_bnd, bnd_need));
        b->bnd_bytes = bnd_need;
    }
    if (plan.groups.size() > 63) return WSB_E_ARG;  // cannot happen: at most 16 + 10 launch groups per plan
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_queues, 0, 64 * sizeof(unsigned int), ctx->stream));

    // first call after creation: the uploads may still be in flight on the copy stream
    const bool piecewise = b->upload_pending && b->n_pieces > 1 && b->n_pieces_usable != 1 && !plan_only && plan.groups.size() == 1 &&
                           plan.groups[0].unit_off < 0 && plan.groups[0].long_nw == 0;
    // plan_only (traceback of global / semiglobal batches): the caller fills chunk by chunk and waits per upload piece itself
    const bool defer_upload = plan_only && b->upload_pending && b->n_pieces > 1 && b->n_pieces_usable != 1;
    if (b->upload_pending && !piecewise && !defer_upload && b->n_pieces > 0)
        CUDA_TRY(ctx, b->wait_piece(ctx->stream, b->n_pieces - 1));

    bool any_s16 = false;
    int s16_gap = GAP_MERGED;
    for (const LaunchGroup& g : plan.groups) any_s16 = any_s16 || g.variant == WSB_VARIANT_S16X2;
    if (any_s16 && !plan_only) {   // list of pairs the packed int16 kernel hands back (flagged subject symbols)
        if (!b->d_redo) CUDA_TRY(ctx, ctx->alloc((void**)&b->d_redo, sizeof(int32_t) * (size_t)(b->n_pairs + 8)));
        CUDA_TRY(ctx, cudaMemsetAsync(b->d_redo, 0, 16, ctx->stream));
    }
    any_s16 = false;

    CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    int launches = 0, n_aux = 0;
    bool aux_used[wsb_ctx::kAux] = {};
    for (size_t k = 0; k < plan.groups.size() && !plan_only; ++k) {
        const LaunchGroup& g = plan.groups[k];
        if (g.long_nw > 0) {  // long-read groups, largest warps-per-pair first, each on its own stream
            const int a = n_aux++ % wsb_ctx::kAux;
            if (!aux_used[a]) { CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->aux[a], ctx->ev0, 0)); aux_used[a] = true; }
            LongParams lp;
            lp.q_codes = b->d_qcodes; lp.q_off = b->d_qoff; lp.q_len = b->d_qlen;
            lp.s_codes = b->d_scodes; lp.s_off = b->d_soff; lp.s_len = b->d_slen;
            lp.pair_q = b->d_pq; lp.pair_s = b->d_ps;
            lp.units = plan.d_units + g.unit_off; lp.n_units = g.n_units;
            lp.out_score = b->d_score; lp.out_i = b->d_i; lp.out_j = b->d_j;
            lp.match = sch->match; lp.mismatch = sch->mismatch; lp.alpha = sch->gap_open; lp.beta = beta_eff;
            lp.bnd = reinterpret_cast<int2*>((char*)b->d_bnd + geo[k].bnd_off); lp.bnd_rows = geo[k].bnd_rows;
            lp.queue = ctx->d_queues + k; lp.one = 1;
            lp.redo = b->d_redo_long ? b->d_redo_long + 4 : nullptr; lp.redo_count = b->d_redo_long; lp.n_units_dev = nullptr;
            if (g.long16) { any_l16 = true; l16_gap = g.gap; l16_rows = std::max(l16_rows, geo[k].bnd_rows); }
            lp.cflags = ctx->d_cflags + (size_t)kLongCfClusters * kLongCf * (size_t)(g.cluster == 2 ? 0 : g.cluster == 4 ? 1 : g.cluster == 8 ? 2 : 3);
            if (g.cluster > 1) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3((unsigned)geo[k].grid); cfg.blockDim = dim3((unsigned)(g.long_nw * 32));
                cfg.dynamicSmemBytes = 0; cfg.stream = ctx->aux[a];
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = (unsigned)g.cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                cfg.attrs = at; cfg.numAttrs = 1;
                static const bool trace_cl = getenv("WSB_TRACE") != nullptr;
                if (trace_cl) fprintf(stderr, "[wsb] long-read launch: %lld pairs on clusters of %d blocks, grid %d\n", (long long)g.n_units, g.cluster, geo[k].grid);
                CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, geo[k].lfn, lp));
            } else {
                geo[k].lfn<<<geo[k].grid, g.long_nw * 32, 0, ctx->aux[a]>>>(lp);
            }
            CUDA_TRY(ctx, cudaGetLastError());
            ++launches;
            continue;
        }
        ScoreParams prm;
        prm.q_codes = b->d_qcodes; prm.q_off = b->d_qoff; prm.q_len = b->d_qlen;
        prm.s_codes = b->d_scodes; prm.s_off = b->d_soff; prm.s_len = b->d_slen;
        prm.pair_q = b->d_pq; prm.pair_s = b->d_ps;
        prm.units = g.unit_off >= 0 ? plan.d_units + g.unit_off : nullptr;
        prm.n_units = g.n_units; prm.n_pairs = b->n_pairs; prm.pair_base = 0;
        prm.redo = b->d_redo ? b->d_redo + 4 : nullptr; prm.redo_count = b->d_redo; prm.n_pairs_dev = nullptr;
        if (g.variant == WSB_VARIANT_S16X2) {
            any_s16 = true; s16_gap = g.gap;
            if (!piecewise) {   // one launch carries the group: its blocks report their cycle counts
                if (!b->d_cycles) CUDA_TRY(ctx, ctx->alloc((void**)&b->d_cycles, sizeof(unsigned long long) * 4096));
                b->cycles_blocks = std::min(geo[k].grid, 4096);
                if (geo[k].grid <= 4096) prm.block_cycles = b->d_cycles;
            }
        }
        prm.out_score = b->d_score; prm.out_i = b->d_i; prm.out_j = b->d_j;
        prm.match = sch->match; prm.mismatch = sch->mismatch; prm.alpha = sch->gap_open; prm.beta = beta_eff;
        prm.bnd = geo[k].bnd_rows ? (char*)b->d_bnd + geo[k].bnd_off : nullptr; prm.bnd_rows = geo[k].bnd_rows;
        if (piecewise) {  // uniform batch, identity unit mapping: one launch per uploaded piece, as its slice lands
            const int nv = g.variant == WSB_VARIANT_I32 ? 1 : 2;
            const Shape sh = shape_of(g.variant, g.shape);
            const int gpb = kThreads / sh.P;
            const int64_t full_blocks = (g.n_units + gpb - 1) / gpb;
            const int64_t resident = full_blocks <= geo[k].grid ? (int64_t)1 << 40 : geo[k].grid;  // grid cap = resident blocks
            for (int pc = 0; pc < b->n_pieces; ++pc) {
                const int64_t lo = pc == 0 ? 0 : b->piece_end[pc - 1], hi = b->piece_end[pc];
                if (hi <= lo) continue;
                CUDA_TRY(ctx, b->wait_piece(ctx->stream, pc));
                prm.pair_base = lo; prm.n_pairs = hi; prm.n_units = (hi - lo + nv - 1) / nv;
                const int64_t blocks = (prm.n_units + gpb - 1) / gpb;
                const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, resident));
                geo[k].fn<<<grid, kThreads, geo[k].smem, ctx->stream>>>(prm);
                CUDA_TRY(ctx, cudaGetLastError());
                ++launches;
                if (fetch && fetch->score && fetch->mapped && pc < 16) {   // results of this piece go home while later pieces upload and run
                    if (!ctx->dl_ev[pc]) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->dl_ev[pc], cudaEventDisableTiming));
                    CUDA_TRY(ctx, cudaEventRecord(ctx->dl_ev[pc], ctx->stream));
                    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->dl_stream, ctx->dl_ev[pc], 0));
                    // a small kernel stores the piece into the page-locked (device-visible) destination: a copy-engine
                    // download would queue behind the batch's own pending uploads and block this thread until they drained
                    results_home_kernel<<<32, 256, 0, ctx->dl_stream>>>(b->d_score + lo, b->d_i + lo, b->d_j + lo, fetch->score + lo,
                                                                        fetch->i + lo, fetch->j + lo, hi - lo);
                    CUDA_TRY(ctx, cudaGetLastError());
                    fetch->done = true;
                }
            }
            continue;
        }
        geo[k].fn<<<geo[k].grid, kThreads, geo[k].smem, ctx->stream>>>(prm);
        CUDA_TRY(ctx, cudaGetLastError());
        ++launches;
    }
    if (any_s16 && atype == AT_GLOBAL) {   // global: the general int32 kernel takes the listed pairs (one pair per unit)
        const int gap32 = !affine ? GAP_LINEAR : (wsb_merged_state_exact(sch) ? GAP_MERGED : GAP_EXACT);
        const bool wide32 = std::abs(sch->match - sch->mismatch) > 127;
        const KernelSel sel = pick_kernel(WSB_VARIANT_I32, wide32 ? 0 : 3, atype, gap32, false, false, wide32);
        if (!sel.fn) return WSB_E_SCHEME;
        CUDA_TRY(ctx, cudaFuncSetAttribute(sel.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel.smem));
        ScoreParams prm = {};
        prm.q_codes = b->d_qcodes; prm.q_off = b->d_qoff; prm.q_len = b->d_qlen;
        prm.s_codes = b->d_scodes; prm.s_off = b->d_soff; prm.s_len = b->d_slen;
        prm.pair_q = b->d_pq; prm.pair_s = b->d_ps;
        prm.units = b->d_redo + 4; prm.n_pairs_dev = b->d_redo; prm.n_units = 0; prm.n_pairs = b->n_pairs;
        prm.out_score = b->d_score; prm.out_i = b->d_i; prm.out_j = b->d_j;
        prm.match = sch->match; prm.mismatch = sch->mismatch; prm.alpha = sch->gap_open; prm.beta = beta_eff;
        prm.bnd = nullptr; prm.bnd_rows = 0;   // one stage: n <= 152 = 8 x 19 (the wide kernel's 8 x 16 would need borders)
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((b->n_pairs + 15) / 16, (int64_t)ctx->sm_count * 2));
        sel.fn<<<grid, kThreads, sel.smem, ctx->stream>>>(prm);
        CUDA_TRY(ctx, cudaGetLastError());
        ++launches;
    } else if (any_s16) {   // re-score what the packed int16 kernel could not encode, with the half2 short kernel
        const KernelSel sel = s16_gap == GAP_LINEAR
            ? KernelSel{f16_local_short_kernel<8, 19, GAP_LINEAR, true>, short_smem_bytes<8, 19>()}
            : KernelSel{f16_local_short_kernel<8, 19, GAP_MERGED, true>, short_smem_bytes<8, 19>()};
        CUDA_TRY(ctx, cudaFuncSetAttribute(sel.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel.smem));
        ScoreParams prm = {};
        prm.q_codes = b->d_qcodes; prm.q_off = b->d_qoff; prm.q_len = b->d_qlen;
        prm.s_codes = b->d_scodes; prm.s_off = b->d_soff; prm.s_len = b->d_slen;
        prm.pair_q = b->d_pq; prm.pair_s = b->d_ps;
        prm.units = b->d_redo + 4; prm.n_pairs_dev = b->d_redo; prm.n_units = 0; prm.n_pairs = b->n_pairs;
        prm.out_score = b->d_score; prm.out_i = b->d_i; prm.out_j = b->d_j;
        prm.match = sch->match; prm.mismatch = sch->mismatch; prm.alpha = sch->gap_open; prm.beta = beta_eff;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((b->n_pairs / 2 + 15) / 16, (int64_t)ctx->sm_count * 2));
        sel.fn<<<grid, kThreads, sel.smem, ctx->stream>>>(prm);
        CUDA_TRY(ctx, cudaGetLastError());
        ++launches;
    }
    if (!defer_upload) b->upload_pending = false;
    for (int a = 0; a < wsb_ctx::kAux; ++a)
        if (aux_used[a]) {
            CUDA_TRY(ctx, cudaEventRecord(ctx->aux_done[a], ctx->aux[a]));
            CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->aux_done[a], 0));
        }
    if (any_l16) {   // pairs the packed int16 long-read kernel handed back (flagged subject symbols): int32 long-read kernel
        LongFn lfn = pick_long(atype, l16_gap, false);
        if (!lfn) return WSB_E_SCHEME;
        LongParams lp = {};
        lp.q_codes = b->d_qcodes; lp.q_off = b->d_qoff; lp.q_len = b->d_qlen;
        lp.s_codes = b->d_scodes; lp.s_off = b->d_soff; lp.s_len = b->d_slen;
        lp.pair_q = b->d_pq; lp.pair_s = b->d_ps;
        lp.units = b->d_redo_long + 4; lp.n_units = 0; lp.n_units_dev = b->d_redo_long;
        lp.out_score = b->d_score; lp.out_i = b->d_i; lp.out_j = b->d_j;
        lp.match = sch->match; lp.mismatch = sch->mismatch; lp.alpha = sch->gap_open; lp.beta = beta_eff;
        lp.bnd = reinterpret_cast<int2*>((char*)b->d_bnd + l16_bnd_off); lp.bnd_rows = l16_rows;
        lp.queue = ctx->d_queues + 63; lp.one = 1; lp.cflags = ctx->d_cflags;
        lfn<<<l16_redo_grid, l16_redo_nw * 32, 0, ctx->stream>>>(lp);
        CUDA_TRY(ctx, cudaGetLastError());
        ++launches;
    }
    {  // empty-side pairs (only possible for non-uniform batches or a uniform batch of empties)
        bool any_empty = false;
        if (b->uniform) any_empty = b->m[0] == 0 || b->n[0] == 0;
        else for (int64_t p = 0; p < b->n_pairs && !any_empty; ++p) any_empty = b->m[p] == 0 || b->n[p] == 0;
        if (any_empty) {
            // deferred upload (traceback of a large global / semiglobal batch): the metadata this kernel reads travels on
            // the copy stream; piece 0's event is recorded behind all of it
            if (defer_upload && b->n_pieces > 0) CUDA_TRY(ctx, b->wait_piece(ctx->stream, 0));
            const int thr = 256;
            empty_side_kernel<<<(unsigned)((b->n_pairs + thr - 1) / thr), thr, 0, ctx->stream>>>(
                b->d_pq, b->d_ps, b->d_qlen, b->d_slen, b->n_pairs, atype, affine ? 1 : 0, sch->gap_open, beta_eff,
                b->d_score, b->d_i, b->d_j);
            CUDA_TRY(ctx, cudaGetLastError());
            ++launches;
        }
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    if (fetch && fetch->score && !plan_only) {
        const size_t bytes = sizeof(int32_t) * (size_t)b->n_pairs;
        bool refetch = !fetch->done;
        if (fetch->done) {   // pieces went home early; pairs a packed kernel handed back were re-scored after that
            int32_t handed_back = 0;
            static const bool trace = getenv("WSB_TRACE") != nullptr;
            const auto t_a = std::chrono::steady_clock::now();
            if (b->d_redo) CUDA_TRY(ctx, cudaMemcpyAsync(&handed_back, b->d_redo, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
            CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
            const auto t_b = std::chrono::steady_clock::now();
            CUDA_TRY(ctx, cudaStreamSynchronize(ctx->dl_stream));
            if (trace) {
                const auto t_c = std::chrono::steady_clock::now();
                fprintf(stderr, "[wsb] score_fetch: wait for kernels %.2f ms, then for downloads %.2f ms\n",
                        std::chrono::duration<double, std::milli>(t_b - t_a).count(), std::chrono::duration<double, std::milli>(t_c - t_b).count());
            }
            bool any_empty = b->uniform ? (b->m[0] == 0 || b->n[0] == 0) : true;
            refetch = handed_back > 0 || any_empty;
        }
        if (refetch) {
            CUDA_TRY(ctx, cudaMemcpyAsync(fetch->score, b->d_score, bytes, cudaMemcpyDeviceToHost, ctx->stream));
            CUDA_TRY(ctx, cudaMemcpyAsync(fetch->i, b->d_i, bytes, cudaMemcpyDeviceToHost, ctx->stream));
            CUDA_TRY(ctx, cudaMemcpyAsync(fetch->j, b->d_j, bytes, cudaMemcpyDeviceToHost, ctx->stream));
            CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        }
    }
    if (kernel_ms) {
        CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev1));
        CUDA_TRY(ctx, cudaEventElapsedTime(kernel_ms, ctx->ev0, ctx->ev1));
    }
    if (n_launches) *n_launches = launches;
    return WSB_OK;
}

// Score and download in one call: when the batch is still uploading piece by piece, the results of every finished piece
// travel back on a third stream while later pieces upload and run (PCIe is full duplex), so the download of the step hides
// behind its upload instead of following it.  Same results and status contract as wsb_batch_score + wsb_batch_fetch_scores.
extern "C" int wsb_batch_score_fetch(wsb_batch* b, const wsb_scheme* sch, int atype, int variant, float* kernel_ms,
                                     int32_t* n_launches, int32_t* out_score, int32_t* out_i, int32_t* out_j, int32_t* status) {
    if (!b || !out_score || !out_i || !out_j) return WSB_E_ARG;
    std::lock_guard<std::recursive_mutex> lock_(b->ctx->mu);
    FetchDst dst;
    dst.score = out_score; dst.i = out_i; dst.j = out_j;
    {   // early piece downloads need a destination the device can write: page-locked host memory
        cudaPointerAttributes a0 = {}, a1 = {}, a2 = {};
        dst.mapped = cudaPointerGetAttributes(&a0, out_score) == cudaSuccess && a0.type == cudaMemoryTypeHost &&
                     cudaPointerGetAttributes(&a1, out_i) == cudaSuccess && a1.type == cudaMemoryTypeHost &&
                     cudaPointerGetAttributes(&a2, out_j) == cudaSuccess && a2.type == cudaMemoryTypeHost;
        (void)cudaGetLastError();
    }
    const int rc = batch_score_impl(b, sch, atype, variant, kernel_ms, n_launches, false, &dst);
    if (rc) return rc;
    if (status) {
        const size_t bytes = sizeof(int32_t) * (size_t)b->n_pairs;
        if (b->last_plan) std::memcpy(status, b->last_plan->status.data(), bytes);
        else std::memset(status, 0, bytes);
    }
    return WSB_OK;
}

extern "C" int wsb_batch_score(wsb_batch* b, const wsb_scheme* sch, int atype, int variant, float* kernel_ms,
                               int32_t* n_launches) {
    return batch_score_impl(b, sch, atype, variant, kernel_ms, n_launches, false);
}

extern "C" int wsb_batch_fetch_scores(wsb_batch* b, int32_t* out_score, int32_t* out_i, int32_t* out_j, int32_t* status) {
    if (!b || !out_score || !out_i || !out_j) return WSB_E_ARG;
    wsb_ctx* ctx = b->ctx;
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const size_t bytes = sizeof(int32_t) * (size_t)b->n_pairs;
    CUDA_TRY(ctx, cudaMemcpyAsync(out_score, b->d_score, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(out_i, b->d_i, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaMemcpyAsync(out_j, b->d_j, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (status) {
        if (b->last_plan) std::memcpy(status, b->last_plan->status.data(), bytes);
        else std::memset(status, 0, bytes);
    }
    return WSB_OK;
}

extern "C" int wsb_score_batch(wsb_ctx* ctx, const wsb_scheme* scheme, int align_type, int variant,
                               const uint8_t* q_codes, const int64_t* q_off, const int32_t* q_len, int64_t n_q,
                               const uint8_t* s_codes, const int64_t* s_off, const int32_t* s_len, int64_t n_s,
                               const int32_t* pair_q, const int32_t* pair_s, int64_t n_pairs, int32_t* out_score,
                               int32_t* out_i, int32_t* out_j, int32_t* status) {
    if (!ctx) return WSB_E_ARG;
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    wsb_batch* b = nullptr;
    int rc = wsb_batch_create(ctx, q_codes, q_off, q_len, n_q, s_codes, s_off, s_len, n_s, pair_q, pair_s, n_pairs, &b);
    if (rc) return rc;
    rc = wsb_batch_score(b, scheme, align_type, variant, nullptr, nullptr);
    if (!rc) rc = wsb_batch_fetch_scores(b, out_score, out_i, out_j, status);
    wsb_batch_destroy(b);
    return rc;
}

// ------------------------------------------------------------------------------------------------ traceback ABI
#include "traceback_host.inl"
