// Cell-stream microbenchmark for sm_100a: the packed int16 row sweep of score_short16.cuh with everything around it
// removed (no shuffles, no snapshot stores, no shared memory), to find what the bare instruction stream can issue at
// 1..4 warps per scheduler, and which operand forms change that.  Not part of the product path.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o cell_bench cell_bench.cu
#include <cstdint>
#include <cstdio>
#include <vector>

#define ROWS 512

__device__ __forceinline__ unsigned prmt(unsigned a, unsigned b, unsigned s) {
    unsigned d; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s)); return d;
}

// VARIANT 0: constants in registers (kernel params), row max on
// VARIANT 1: constants as immediates
// VARIANT 2: immediates, no row max
// VARIANT 3: immediates, row max, two interleaved independent strips of K/2 columns (ILP 2, same work)
// VARIANT 4: like 0 but h and tn computed with 2-input max pairs (4 ALU per cell instead of 2)
// VARIANT 5: immediates, row max over tn instead of h (h not needed for anything but D)
template <int VARIANT, int K>
__global__ void __launch_bounds__(128) cell_kernel(unsigned* out, const unsigned* in, long long* cyc, int na, int ng) {
    unsigned sel[K], TA[K], TG[K], D[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
        sel[c] = in[c] ^ threadIdx.x; TA[c] = in[32 + c]; TG[c] = in[64 + c]; D[c] = in[96 + c];
    }
    unsigned rw0 = in[128] + threadIdx.x, rw1 = in[129], nw0 = in[130], nw1 = in[131];
    unsigned la = in[132], lg = in[133], hd = in[134], best = 0u;
    const unsigned c_na = VARIANT == 0 || VARIANT == 4 ? (unsigned)na : 0xfffefffeu;
    const unsigned c_ng = VARIANT == 0 || VARIANT == 4 ? (unsigned)ng : 0xffffffffu;
    long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < ROWS; ++r) {
        unsigned rm = 0u, hprev = 0u;
        if (VARIANT != 3) {
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const unsigned d = c == 0 ? __vadd2(hd, prmt(rw0, rw1, sel[0])) : D[c];
                unsigned h, tn;
                if (VARIANT == 4) {
                    h = __vmaxs2(__vmaxs2(TA[c], la), __vmaxs2(d, 0u));
                    tn = __vmaxs2(__vmaxs2(TG[c], lg), __vmaxs2(d, 0u));
                } else {
                    h = __vimax3_s16x2_relu(TA[c], la, d);
                    tn = __vimax3_s16x2_relu(TG[c], lg, d);
                }
                la = __vadd2(tn, c_na);
                lg = __vadd2(tn, c_ng);
                TG[c] = lg; TA[c] = la;
                if (c >= 1) D[c] = __vadd2(hprev, prmt(nw0, nw1, sel[c]));
                if (VARIANT != 2) {
                    const unsigned x = VARIANT == 5 ? tn : h;
                    if (c & 1) rm = __vimax3_s16x2(rm, VARIANT == 5 ? hprev : hprev, x);
                    else if (c == K - 1) rm = __vmaxs2(rm, x);
                }
                hprev = VARIANT == 5 ? h : h;
            }
        } else {
            constexpr int H = K / 2;
            unsigned la2 = la ^ 1u, lg2 = lg ^ 1u, hprev2 = 0u, rm2 = 0u;
#pragma unroll
            for (int c = 0; c < H; ++c) {
                {
                    const unsigned d = c == 0 ? __vadd2(hd, prmt(rw0, rw1, sel[0])) : D[c];
                    const unsigned h = __vimax3_s16x2_relu(TA[c], la, d);
                    const unsigned tn = __vimax3_s16x2_relu(TG[c], lg, d);
                    la = __vadd2(tn, c_na); lg = __vadd2(tn, c_ng);
                    TG[c] = lg; TA[c] = la;
                    if (c >= 1) D[c] = __vadd2(hprev, prmt(nw0, nw1, sel[c]));
                    if (c & 1) rm = __vimax3_s16x2(rm, hprev, h);
                    hprev = h;
                }
                {
                    const int c2 = c + H;
                    const unsigned d = c == 0 ? __vadd2(hd ^ 3u, prmt(rw0, rw1, sel[c2])) : D[c2];
                    const unsigned h = __vimax3_s16x2_relu(TA[c2], la2, d);
                    const unsigned tn = __vimax3_s16x2_relu(TG[c2], lg2, d);
                    la2 = __vadd2(tn, c_na); lg2 = __vadd2(tn, c_ng);
                    TG[c2] = lg2; TA[c2] = la2;
                    if (c >= 1) D[c2] = __vadd2(hprev2, prmt(nw0, nw1, sel[c2]));
                    if (c & 1) rm2 = __vimax3_s16x2(rm2, hprev2, h);
                    hprev2 = h;
                }
            }
            rm = __vmaxs2(rm, rm2); la ^= la2; lg ^= lg2; hprev ^= hprev2;
        }
        best = __vmaxs2(best, rm);
        hd = hprev;
        // next row's words: a cheap rotation keeps the values changing without memory traffic
        const unsigned t = rw0; rw0 = nw0; nw0 = rw1; rw1 = nw1; nw1 = t;
    }
    long long t1 = clock64();
    unsigned acc = best ^ la ^ lg ^ hd;
#pragma unroll
    for (int c = 0; c < K; ++c) acc ^= TA[c] ^ TG[c] ^ D[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int VARIANT, int K>
void run(const char* name, int nsm, unsigned* out, unsigned* in, long long* cyc) {
    for (int wps = 1; wps <= 4; ++wps) {   // warps per scheduler = blocks of 128 threads per SM
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cell_kernel<VARIANT, K>, 128, 0);
        if (per_sm < wps) { printf("%-44s K=%2d wps=%d: only %d blocks fit\n", name, K, wps, per_sm); continue; }
        // shared-memory ballast would be needed to pin blocks per SM exactly; a grid of nsm * wps blocks spreads evenly
        cell_kernel<VARIANT, K><<<nsm * wps, 128>>>(out, in, cyc, 0xfffefffe, 0xffffffff);
        cudaDeviceSynchronize();
        cell_kernel<VARIANT, K><<<nsm * wps, 128>>>(out, in, cyc, 0xfffefffe, 0xffffffff);
        cudaDeviceSynchronize();
        std::vector<long long> h(nsm * wps);
        cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost);
        double avg = 0; for (auto c : h) avg += c; avg /= h.size();
        // cycles the scheduler spends per warp-row = elapsed / rows / (warps on that scheduler)
        printf("%-44s K=%2d wps=%d: %7.1f cycles per row per warp, %6.1f scheduler cycles per warp-row, %5.2f per packed cell\n",
               name, K, wps, avg / ROWS, avg / ROWS / wps, avg / ROWS / wps / K);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    const int nsm = p.multiProcessorCount;
    unsigned *out, *in; long long* cyc;
    cudaMalloc(&out, (size_t)nsm * 4 * 128 * 4); cudaMalloc(&in, 256 * 4); cudaMalloc(&cyc, (size_t)nsm * 4 * 8);
    unsigned hin[256]; for (int i = 0; i < 256; ++i) hin[i] = 0x00030002u * (i + 1);
    cudaMemcpy(in, hin, sizeof(hin), cudaMemcpyHostToDevice);
    printf("device %s, %d SMs\n", p.name, nsm);
    run<0, 19>("constants in registers", nsm, out, in, cyc);
    run<1, 19>("constants as immediates", nsm, out, in, cyc);
    run<2, 19>("immediates, no row max", nsm, out, in, cyc);
    run<3, 18>("immediates, two independent half strips", nsm, out, in, cyc);
    run<4, 19>("2-input max only (4 ALU per cell)", nsm, out, in, cyc);
    run<1, 10>("constants as immediates", nsm, out, in, cyc);
    run<1, 8>("constants as immediates", nsm, out, in, cyc);
    return 0;
}
