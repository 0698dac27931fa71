// compile-only harness: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -cubin -o /tmp/s16.cubin tools/probe/short16_probe.cu
#include "../../paper_2205_07610_b200/csrc/score_short16.cuh"
template __global__ void wsb::s16_local_short_kernel<8, 19, wsb::GAP_MERGED>(const wsb::ScoreParams);
template __global__ void wsb::s16_local_short_kernel<8, 19, wsb::GAP_MERGED, 4, 2, 1>(const wsb::ScoreParams);
#ifdef PROBE_ALL
template __global__ void wsb::s16_local_short_kernel<8, 16, wsb::GAP_MERGED>(const wsb::ScoreParams);
template __global__ void wsb::s16_local_short_kernel<8, 19, wsb::GAP_LINEAR>(const wsb::ScoreParams);
template __global__ void wsb::s16_local_short_kernel<8, 19, wsb::GAP_LINEAR, 4, 1, 1>(const wsb::ScoreParams);
#endif
