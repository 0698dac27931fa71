// Host-side 2-bit packing throughput probe: how fast can T threads turn one-byte codes into the 2-bit layout?
// g++ -O3 -march=native -pthread hostpack_bench.cpp -o hostpack_bench -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <thread>
#include <vector>
#include <immintrin.h>
#include <cuda_runtime.h>

__attribute__((target("bmi2"))) static uint64_t pack_pext(const uint8_t* src, uint8_t* dst, int64_t n_out) {
    uint64_t fl = 0;
    const uint64_t* s = reinterpret_cast<const uint64_t*>(src);
    int64_t k = 0;
    for (; k + 8 <= n_out; k += 8) {   // 32 symbols -> 8 bytes
        uint64_t a = s[0], b = s[1], c = s[2], d = s[3];
        s += 4;
        fl |= a | b | c | d;
        uint64_t o = _pext_u64(a, 0x0303030303030303ull) | (_pext_u64(b, 0x0303030303030303ull) << 16) |
                     (_pext_u64(c, 0x0303030303030303ull) << 32) | (_pext_u64(d, 0x0303030303030303ull) << 48);
        memcpy(dst + k, &o, 8);
    }
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(s);
    for (; k < n_out; ++k) {
        dst[k] = (sb[0] & 3) | ((sb[1] & 3) << 2) | ((sb[2] & 3) << 4) | ((sb[3] & 3) << 6);
        fl |= sb[0] | sb[1] | sb[2] | sb[3];
        sb += 4;
    }
    return fl;
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 1200000000ll;
    const int hw = (int)std::thread::hardware_concurrency();
    printf("hardware_concurrency %d bmi2 %d\n", hw, __builtin_cpu_supports("bmi2"));
    uint8_t *src, *dst;
    cudaHostAlloc((void**)&src, n, cudaHostAllocDefault);
    cudaHostAlloc((void**)&dst, n / 4, cudaHostAllocDefault);
    for (int64_t i = 0; i < n; ++i) src[i] = (uint8_t)((i * 2654435761u >> 13) & 3);
    uint8_t* dev; cudaMalloc((void**)&dev, n);
    for (int T : {1, 2, 4, 8, 12, 16, 24, 32}) {
        if (T > hw) break;
        double best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            const int64_t n_out = n / 4;
            for (int t = 0; t < T; ++t) th.emplace_back([=] {
                const int64_t lo = n_out * t / T / 64 * 64, hi = t + 1 == T ? n_out : n_out * (t + 1) / T / 64 * 64;
                volatile uint64_t f = pack_pext(src + lo * 4, dst + lo, hi - lo); (void)f;
            });
            for (auto& x : th) x.join();
            best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        printf("T=%2d pack %.1f ms  %.1f GB/s (input bytes)\n", T, best * 1e3, n / best / 1e9);
    }
    // the same while the copy engine streams the raw bytes of the other half (bus + memory contention)
    {
        cudaStream_t st; cudaStreamCreate(&st);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0, st); cudaMemcpyAsync(dev, src, n, cudaMemcpyHostToDevice, st); cudaEventRecord(e1, st);
        cudaStreamSynchronize(st);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("raw H2D alone: %.1f ms %.1f GB/s\n", ms, n / ms / 1e6);
        const int T = std::min(hw, 16);
        cudaEventRecord(e0, st); cudaMemcpyAsync(dev, src, n, cudaMemcpyHostToDevice, st); cudaEventRecord(e1, st);
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        const int64_t n_out = n / 4;
        for (int t = 0; t < T; ++t) th.emplace_back([=] {
            const int64_t lo = n_out * t / T / 64 * 64, hi = t + 1 == T ? n_out : n_out * (t + 1) / T / 64 * 64;
            volatile uint64_t f = pack_pext(src + lo * 4, dst + lo, hi - lo); (void)f;
        });
        for (auto& x : th) x.join();
        double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        cudaStreamSynchronize(st);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("concurrent: pack(T=%d) %.1f ms, raw H2D %.1f ms\n", T, dt * 1e3, ms);
    }
    return 0;
}
