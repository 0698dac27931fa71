// wsb200_s16.cu -- the packed int16 kernels (score_short16.cuh: short local reads, score_short16g.cuh: short global reads,
// score_long16.cuh: long reads, two pairs per block) in their own translation unit, compiled with -Xptxas -O1.  Their loops are hand-scheduled straight-line code whose strip state is
// updated in place; ptxas' default optimisation level reorders them and pays with register moves and earlier stalls
// (1 M x 150 bp on a B200: local affine 5.24 -> 5.38 TCUPS, global linear 8.11 -> 8.45 at -O1), while every other kernel
// of the library is faster at the default level (half2 short kernel -13 %, int32 long-read kernel -14 % at -O1).  The packed
// long-read kernel's row loop shrinks from 162 to 151 instructions at -O1.
#include "score_short16.cuh"
#include "score_short16g.cuh"
#include "score_long16.cuh"

namespace wsb {

// alpha / gamma = min(alpha, beta): the schemes of the reference's benchmarks (affine 2/1, linear 1) get instantiations
// with the gap costs as immediates
template <int P, int K, int MINB = 4> static KernelSel pick_local(int gap, int alpha, int gamma) {
    if (gap == GAP_LINEAR) {
        if (alpha == 1) return {s16_local_short_kernel<P, K, GAP_LINEAR, MINB, 1, 1>, short16_smem_bytes<P, K>()};
        return {s16_local_short_kernel<P, K, GAP_LINEAR, MINB>, short16_smem_bytes<P, K>()};
    }
    if (alpha == 2 && gamma == 1) return {s16_local_short_kernel<P, K, GAP_MERGED, MINB, 2, 1>, short16_smem_bytes<P, K>()};
    return {s16_local_short_kernel<P, K, GAP_MERGED, MINB>, short16_smem_bytes<P, K>()};
}

// global alignment; ragged = units of unequal pairs or reads shorter than two lane groups (row m is captured in every trip)
template <int P, int K> static KernelSel pick_global(int gap, int alpha, int gamma, bool ragged) {
    const size_t smem = short16g_smem_bytes<P, K>();
    if (gap == GAP_LINEAR) {
        if (ragged) return {s16_global_short_kernel<P, K, GAP_LINEAR, true>, smem};
        if (alpha == 1) return {s16_global_short_kernel<P, K, GAP_LINEAR, false, 1, 1>, smem};
        return {s16_global_short_kernel<P, K, GAP_LINEAR, false>, smem};
    }
    if (ragged) return {s16_global_short_kernel<P, K, GAP_MERGED, true>, smem};
    if (alpha == 2 && gamma == 1) return {s16_global_short_kernel<P, K, GAP_MERGED, false, 2, 1>, smem};
    return {s16_global_short_kernel<P, K, GAP_MERGED, false>, smem};
}

KernelSel pick_short16_local(int shape, int gap, int alpha, int gamma) {
    return shape == 0 ? pick_local<8, 16>(gap, alpha, gamma) : shape == 1 ? pick_local<8, 19>(gap, alpha, gamma)
                                                                           : pick_local<16, 10>(gap, alpha, gamma);
}
KernelSel pick_short16_global(int shape, int gap, int alpha, int gamma, bool ragged) {
    return shape == 0 ? pick_global<8, 16>(gap, alpha, gamma, ragged) : shape == 1 ? pick_global<8, 19>(gap, alpha, gamma, ragged)
                                                                                   : pick_global<16, 10>(gap, alpha, gamma, ragged);
}

template <int GAP, int AIMM, int GIMM> static LongFn pick_long16_atype(int atype) {
    switch (atype) {
        case AT_GLOBAL: return score_long16_kernel<AT_GLOBAL, GAP, AIMM, GIMM>;
        case AT_LOCAL: return score_long16_kernel<AT_LOCAL, GAP, AIMM, GIMM>;
        default: return score_long16_kernel<AT_SEMI, GAP, AIMM, GIMM>;
    }
}
LongFn pick_long16(int atype, int gap, int alpha, int gamma) {
    if (gap == GAP_LINEAR) return alpha == 1 ? pick_long16_atype<GAP_LINEAR, 1, 1>(atype) : pick_long16_atype<GAP_LINEAR, 0, 0>(atype);
    if (gap == GAP_MERGED) return (alpha == 2 && gamma == 1) ? pick_long16_atype<GAP_MERGED, 2, 1>(atype)
                                                             : pick_long16_atype<GAP_MERGED, 0, 0>(atype);
    return nullptr;
}

}  // namespace wsb
