// hostpack.h -- host-side 2-bit packing of one-byte symbol codes (hostpack.cpp)
#pragma once
#include <cstdint>

namespace wsb {
// Writes packed bytes [b0, b1) of a pool of `total` one-byte codes: packed byte j = symbols 4j .. 4j+3, two bits each, low
// bits first (symbols beyond the pool's end read as 0).  Returns true when a symbol in that range is not in 0..3 (a
// flagged symbol has no 2-bit encoding: the caller sends that slice as plain bytes instead).
bool hostpack_range(const uint8_t* codes, int64_t total, uint8_t* packed, int64_t b0, int64_t b1);
const char* hostpack_isa();   // "avx512bw", "bmi2" or "plain": the body the running CPU selected
}  // namespace wsb
