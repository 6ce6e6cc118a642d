// Microbenchmark: LOP3 / IMAD / mixed throughput per SM on this GPU (diagnostics only).
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

template <uint32_t L>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(L));
    return d;
}

template <int MODE>
__global__ void k(uint32_t* out, int iters, uint32_t seed) {
    uint32_t x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + i + 1);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 0) x[i] = lop3<0x96>(x[i], x[(i + 1) & 7], x[(i + 3) & 7]);        // 3-reg LOP3
                if (MODE == 1) x[i] = lop3<0xE2>(x[i], 0xFEFEFEFEu, x[(i + 3) & 7]);           // LOP3 with immediate
                if (MODE == 2) x[i] = x[i] * x[(i + 1) & 7] + x[(i + 3) & 7];                  // IMAD
                if (MODE == 3) { x[i] = lop3<0x96>(x[i], x[(i + 1) & 7], x[(i + 3) & 7]); x[(i+5)&7] = x[(i+5)&7] * 3u + x[i]; }  // 1:1 mix
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char* name, int threads, int per_sm_ops) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, sms * 4 * threads * 4);
    const int iters = 2000;
    k<MODE><<<sms, threads>>>(out, 10, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<MODE><<<sms, threads>>>(out, iters, 1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_instr = double(iters) * 16 * 8 * per_sm_ops * (threads / 32);  // per SM
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-22s threads %4d: %.3f ms, %.3f warp-instr/ns/SM -> %.2f warp-instr/clk/SM @%.0f MHz\n", name, threads, ms,
           warp_instr / (ms * 1e6), warp_instr / (ms * 1e-3) / (clk * 1e3), clk / 1e3);
    cudaFree(out);
}

int main() {
    for (int t : {128, 256, 512}) {
        run<0>("LOP3 3-reg", t, 1);
        run<1>("LOP3 imm", t, 1);
        run<2>("IMAD", t, 1);
        run<3>("LOP3+IMAD", t, 2);
    }
    return 0;
}
