// hostpack.cpp -- host side of the packed upload: one-byte symbol codes -> the 2-bit layout (four symbols per byte, low
// bits first: the reference's Sequence.data layout, core.py:78-87, here over a whole pool), so that a quarter of the
// bytes cross the PCIe bus (49 GB/s measured on the B200 boxes: a 1.2 GB cfg2 upload takes longer than its kernels).
// Built as plain C++ (the AVX-512 / BMI2 bodies are selected at run time); called by the worker threads of
// batch_create_impl in wsb200.cu.  16 threads pack 86 GB/s of input with the BMI2 body on the bench host
// (tools/probe/hostpack_bench.cpp), more with AVX-512.
#include "hostpack.h"

#include <cstdint>
#include <cstring>
#include <immintrin.h>

namespace wsb {
namespace {

// 64 symbols -> 16 bytes per step: bytes pair up inside 16-bit lanes ((w | w >> 6) & 0xf), nibbles inside 32-bit lanes
// (v | v >> 12), VPMOVDB keeps the low byte of every lane.
__attribute__((target("avx512f,avx512bw"))) uint32_t body_avx512(const uint8_t* src, uint8_t* dst, int64_t n_out) {
    __m512i seen = _mm512_setzero_si512();
    const __m512i m3 = _mm512_set1_epi8(3), m15 = _mm512_set1_epi16(15);
    int64_t k = 0;
    // the staging block is written once and read by the copy engine: streaming stores (no read-for-ownership) where the
    // output is 16-byte aligned, i.e. after at most 15 leading bytes
    const bool stream = n_out >= 64;
    if (stream)
        for (; (reinterpret_cast<uintptr_t>(dst + k) & 15u) != 0; ++k) {
            const uint8_t* s = src + 4 * k;
            dst[k] = (uint8_t)((s[0] & 3) | ((s[1] & 3) << 2) | ((s[2] & 3) << 4) | ((s[3] & 3) << 6));
            seen = _mm512_or_si512(seen, _mm512_set1_epi32((int)(s[0] | s[1] | s[2] | s[3])));
        }
    for (; stream && k + 16 <= n_out; k += 16) {
        const __m512i raw = _mm512_loadu_si512(src + 4 * k);
        seen = _mm512_or_si512(seen, raw);
        const __m512i x = _mm512_and_si512(raw, m3);
        const __m512i t = _mm512_and_si512(_mm512_or_si512(x, _mm512_srli_epi16(x, 6)), m15);
        const __m512i u = _mm512_or_si512(t, _mm512_srli_epi32(t, 12));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k), _mm512_cvtepi32_epi8(u));
    }
    if (stream) _mm_sfence();
    for (; k + 16 <= n_out; k += 16) {
        const __m512i raw = _mm512_loadu_si512(src + 4 * k);
        seen = _mm512_or_si512(seen, raw);
        const __m512i x = _mm512_and_si512(raw, m3);
        const __m512i t = _mm512_and_si512(_mm512_or_si512(x, _mm512_srli_epi16(x, 6)), m15);
        const __m512i u = _mm512_or_si512(t, _mm512_srli_epi32(t, 12));
        _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + k), _mm512_cvtepi32_epi8(u));
    }
    uint32_t fl = _mm512_test_epi8_mask(seen, _mm512_set1_epi8((char)0xfc)) ? 0x80u : 0u;
    for (; k < n_out; ++k) {
        const uint8_t* s = src + 4 * k;
        dst[k] = (uint8_t)((s[0] & 3) | ((s[1] & 3) << 2) | ((s[2] & 3) << 4) | ((s[3] & 3) << 6));
        fl |= s[0] | s[1] | s[2] | s[3];
    }
    return fl;
}

__attribute__((target("bmi2"))) uint32_t body_bmi2(const uint8_t* src, uint8_t* dst, int64_t n_out) {
    const unsigned long long M = 0x0303030303030303ull;
    unsigned long long seen = 0;
    int64_t k = 0;
    for (; k + 8 <= n_out; k += 8) {   // 32 symbols -> 8 bytes
        unsigned long long w[4];
        memcpy(w, src + 4 * k, 32);
        seen |= w[0] | w[1] | w[2] | w[3];
        const unsigned long long o = _pext_u64(w[0], M) | (_pext_u64(w[1], M) << 16) | (_pext_u64(w[2], M) << 32) | (_pext_u64(w[3], M) << 48);
        memcpy(dst + k, &o, 8);
    }
    uint32_t fl = (seen & 0xfcfcfcfcfcfcfcfcull) ? 0x80u : 0u;
    for (; k < n_out; ++k) {
        const uint8_t* s = src + 4 * k;
        dst[k] = (uint8_t)((s[0] & 3) | ((s[1] & 3) << 2) | ((s[2] & 3) << 4) | ((s[3] & 3) << 6));
        fl |= s[0] | s[1] | s[2] | s[3];
    }
    return fl;
}

uint32_t body_plain(const uint8_t* src, uint8_t* dst, int64_t n_out) {
    unsigned long long seen = 0;
    int64_t k = 0;
    for (; k + 2 <= n_out; k += 2) {   // 8 symbols -> 2 bytes, folding inside a 64-bit word
        unsigned long long w;
        memcpy(&w, src + 4 * k, 8);
        seen |= w;
        w &= 0x0303030303030303ull;
        w = (w | (w >> 6)) & 0x000f000f000f000full;
        w = (w | (w >> 12)) & 0x000000ff000000ffull;
        dst[k] = (uint8_t)w;
        dst[k + 1] = (uint8_t)(w >> 32);
    }
    uint32_t fl = (seen & 0xfcfcfcfcfcfcfcfcull) ? 0x80u : 0u;
    for (; k < n_out; ++k) {
        const uint8_t* s = src + 4 * k;
        dst[k] = (uint8_t)((s[0] & 3) | ((s[1] & 3) << 2) | ((s[2] & 3) << 4) | ((s[3] & 3) << 6));
        fl |= s[0] | s[1] | s[2] | s[3];
    }
    return fl;
}

using Body = uint32_t (*)(const uint8_t*, uint8_t*, int64_t);
Body pick_body(const char** name) {
    __builtin_cpu_init();
    if (__builtin_cpu_supports("avx512bw") && __builtin_cpu_supports("avx512f")) { *name = "avx512bw"; return body_avx512; }
    if (__builtin_cpu_supports("bmi2")) { *name = "bmi2"; return body_bmi2; }
    *name = "plain";
    return body_plain;
}
const char* g_name = "";
const Body g_body = pick_body(&g_name);

}  // namespace

const char* hostpack_isa() { return g_name; }

bool hostpack_range(const uint8_t* codes, int64_t total, uint8_t* packed, int64_t b0, int64_t b1) {
    if (b1 <= b0) return false;
    const int64_t whole = total / 4;            // packed bytes whose four symbols all exist
    const int64_t e = b1 < whole ? b1 : whole;
    uint32_t fl = 0;
    if (e > b0) fl |= g_body(codes + 4 * b0, packed + b0, e - b0);
    for (int64_t j = (e > b0 ? e : b0); j < b1; ++j) {   // the pool's last, partial byte: symbols beyond the end read as 0
        unsigned v = 0;
        for (int x = 0; x < 4; ++x) {
            const int64_t s = 4 * j + x;
            if (s < total) { v |= (unsigned)(codes[s] & 3) << (2 * x); fl |= codes[s]; }
        }
        packed[j] = (uint8_t)v;
    }
    return (fl & 0xfcu) != 0;
}

}  // namespace wsb
