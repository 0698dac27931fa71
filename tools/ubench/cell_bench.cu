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


// ---- the loop of score_short16.cuh rebuilt element by element (FEAT bits): 1 = row words from shared memory (2 LDS.64
// per row), 2 = record (VIMNMX with predicates + 10 predicated STS.128 of the T - gamma quads), 4 = hand-over (3 SHFL.UP
// + 3 SEL into the next row), 8 = record predicates true about a quarter of the time (else almost never)
template <int FEAT>
__global__ void __launch_bounds__(128, 4) loop_kernel(unsigned* out, const unsigned* in, long long* cyc) {
    constexpr int K = 19, NW = 20;
    extern __shared__ uint4 sm4[];
    uint2* qb = reinterpret_cast<uint2*>(sm4 + 10 * 128);
    unsigned sel[K], TA[K], TG[NW], D[K];
#pragma unroll
    for (int c = 0; c < K; ++c) { sel[c] = in[c] ^ threadIdx.x; TA[c] = in[32 + c]; TG[c] = in[64 + c]; D[c] = in[96 + c]; }
    TG[K] = 0u;
    for (int x = threadIdx.x; x < 16 * 172; x += 128) qb[x] = make_uint2(in[x & 127] * 3u, in[(x + 7) & 127]);
    __syncthreads();
    const int t = threadIdx.x & 7, gib = threadIdx.x >> 3;
    const unsigned keep = t == 0 ? 0u : 1u;
    unsigned qaddr = (unsigned)__cvta_generic_to_shared(qb + gib * 172 + (8 - t));
    const unsigned snap = (unsigned)__cvta_generic_to_shared(sm4 + threadIdx.x);
    unsigned rw0 = in[128] + threadIdx.x, rw1 = in[129], nw0 = in[130], nw1 = in[131];
    unsigned ta_l = in[132], tg_l = in[133], hd = in[134], hl = 0u, best = 0u, s_la = 0u, s_lg = 0u, s_h = 0u;
    const unsigned c_na = 0xfffefffeu, c_ng = 0xffffffffu;
    long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < ROWS; ++r) {
        if (FEAT & 4) { hd = hl; ta_l = s_la * keep; tg_l = s_lg * keep; hl = s_h * keep; }
        unsigned la = ta_l, lg = tg_l, rm = 0u, hprev = 0u;
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const unsigned d = c == 0 ? __vadd2(hd, prmt(rw0, rw1, sel[0])) : D[c];
            const unsigned h = __vimax3_s16x2_relu(TA[c], la, d);
            const unsigned tn = __vimax3_s16x2_relu(TG[c], lg, d);
            la = __vadd2(tn, c_na); lg = __vadd2(tn, c_ng);
            TG[c] = lg; TA[c] = la;
            if (c >= 1) D[c] = __vadd2(hprev, prmt(nw0, nw1, sel[c]));
            if (c & 1) rm = __vimax3_s16x2(rm, hprev, h);
            else if (c == K - 1) rm = __vmaxs2(rm, h);
            hprev = h;
        }
        if (FEAT & 1) {
            const unsigned qa = qaddr + 8u * (unsigned)(r & 127);
            asm volatile("ld.shared.v2.b32 {%0, %1}, [%2+8];" : "=r"(rw0), "=r"(rw1) : "r"(qa) : "memory");
            asm volatile("ld.shared.v2.b32 {%0, %1}, [%2+16];" : "=r"(nw0), "=r"(nw1) : "r"(qa) : "memory");
        } else { const unsigned x = rw0; rw0 = nw0; nw0 = rw1; rw1 = nw1; nw1 = x; }
        if (FEAT & 2) {
            TG[K] = qaddr;
            if ((FEAT & 8) && (r & 3) == 0) best = 0u;   // records become frequent
            unsigned nb;
            asm volatile("{\n\t.reg .pred p, q;\n\t.reg .s16 r0, r1, a0, a1;\n\t"
                "max.s16x2 %0, %1, %2;\n\tmov.b32 {r0, r1}, %0;\n\tmov.b32 {a0, a1}, %1;\n\t"
                "setp.eq.s16 p, r0, a0;\n\tsetp.eq.s16 q, r1, a1;\n\t"
                "@!p st.shared.v4.b32 [%3+0], {%4, %5, %6, %7};\n\t@!q st.shared.v4.b32 [%3+10240], {%4, %5, %6, %7};\n\t"
                "@!p st.shared.v4.b32 [%3+2048], {%8, %9, %10, %11};\n\t@!q st.shared.v4.b32 [%3+12288], {%8, %9, %10, %11};\n\t"
                "@!p st.shared.v4.b32 [%3+4096], {%12, %13, %14, %15};\n\t@!q st.shared.v4.b32 [%3+14336], {%12, %13, %14, %15};\n\t"
                "@!p st.shared.v4.b32 [%3+6144], {%16, %17, %18, %19};\n\t@!q st.shared.v4.b32 [%3+16384], {%16, %17, %18, %19};\n\t"
                "@!p st.shared.v4.b32 [%3+8192], {%20, %21, %22, %23};\n\t@!q st.shared.v4.b32 [%3+18432], {%20, %21, %22, %23};\n\t}"
                : "=&r"(nb) : "r"(best), "r"(rm), "r"(snap), "r"(TG[0]), "r"(TG[1]), "r"(TG[2]), "r"(TG[3]), "r"(TG[4]), "r"(TG[5]),
                  "r"(TG[6]), "r"(TG[7]), "r"(TG[8]), "r"(TG[9]), "r"(TG[10]), "r"(TG[11]), "r"(TG[12]), "r"(TG[13]), "r"(TG[14]),
                  "r"(TG[15]), "r"(TG[16]), "r"(TG[17]), "r"(TG[18]), "r"(TG[19]) : "memory");
            best = nb;
        } else best = __vmaxs2(best, rm);
        if (FEAT & 4) {
            s_la = __shfl_up_sync(0xffffffffu, la, 1, 8);
            s_lg = __shfl_up_sync(0xffffffffu, lg, 1, 8);
            s_h = __shfl_up_sync(0xffffffffu, hprev, 1, 8);
        } else { ta_l = la; tg_l = lg; hd = hprev; }
    }
    long long t1 = clock64();
    unsigned acc = best ^ ta_l ^ tg_l ^ hd ^ hl;
#pragma unroll
    for (int c = 0; c < K; ++c) acc ^= TA[c] ^ TG[c] ^ D[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int FEAT> void run_loop(const char* name, int nsm, unsigned* out, unsigned* in, long long* cyc) {
    const int smem = 20 * 128 * 16 + 16 * 172 * 8;
    cudaFuncSetAttribute(loop_kernel<FEAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int wps = 1; wps <= 4; ++wps) {
        loop_kernel<FEAT><<<nsm * wps, 128, smem>>>(out, in, cyc); cudaDeviceSynchronize();
        loop_kernel<FEAT><<<nsm * wps, 128, smem>>>(out, in, cyc); cudaDeviceSynchronize();
        std::vector<long long> h(nsm * wps);
        cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost);
        double avg = 0; for (auto c : h) avg += c; avg /= h.size();
        printf("loop %-46s wps=%d: %7.1f cycles per row per warp, %6.1f scheduler cycles per warp-row\n", name, wps, avg / ROWS, avg / ROWS / wps);
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
    run_loop<0>("cells only", nsm, out, in, cyc);
    run_loop<1>("+ row words from shared memory", nsm, out, in, cyc);
    run_loop<3>("+ record, predicates almost never true", nsm, out, in, cyc);
    run_loop<11>("+ record, predicates often true", nsm, out, in, cyc);
    run_loop<5>("+ hand-over (no record)", nsm, out, in, cyc);
    run_loop<7>("+ record (rare) + hand-over", nsm, out, in, cyc);
    run_loop<15>("+ record (often) + hand-over", nsm, out, in, cyc);
    return 0;
}
