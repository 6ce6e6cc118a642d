// Microbenchmark: the lean K3+K1 per-row instruction mix on register-generated
// rows (no shared memory): achievable ALU rate for this mix (diagnostics only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <uint32_t L>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(L));
    return d;
}

template <int CHAINS>
__global__ void k(uint32_t* out, int iters, uint32_t mul2, uint32_t mul17, uint32_t seed) {
    uint32_t x[CHAINS], pa[CHAINS], pb[CHAINS], G2[CHAINS], G3[CHAINS], links[CHAINS], ones[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        x[c] = seed * (threadIdx.x * 7 + c + 1);
        pa[c] = pb[c] = G2[c] = G3[c] = links[c] = ones[c] = 0;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 32; ++r) {
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) {
                x[c] = x[c] * 0x9E3779B1u + 0x7F4A7C15u;   // next row word (FMA pipe)
                const uint32_t a = x[c];
                const uint32_t t1 = a * mul2;
                const uint32_t t3 = (a >> 24) * mul17 + __umulhi(a, mul17);
                const uint32_t b = lop3<0xE2>(t1, 0xFEFEFEFEu, t3);
                const uint32_t P = lop3<0x3A>(a, pa[c], b);
                ones[c] ^= P;
                const uint32_t ab = a & b;
                const uint32_t f = lop3<0x60>(ab, pa[c], pb[c]);
                const uint32_t cont = lop3<0xF8>(a & pa[c], b, pb[c]);
                const uint32_t lk = lop3<0x04>(cont, G2[c], G3[c]);
                const uint32_t g3 = lop3<0xEA>(cont, G3[c], G2[c] & f);
                G2[c] = lop3<0xF8>(ab, cont, G2[c]);
                G3[c] = g3;
                pa[c] = a;
                pb[c] = b;
                if (r & 1) links[c] += __popc(lk);
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) r ^= links[c] ^ ones[c] ^ G2[c] ^ G3[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int CHAINS>
void run(int threads) {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* out;
    cudaMalloc(&out, sms * threads * 4);
    k<CHAINS><<<sms, threads>>>(out, 10, 2, 1 << 17, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 400;
    cudaEventRecord(a);
    k<CHAINS><<<sms, threads>>>(out, iters, 2, 1 << 17, 1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_rows = double(iters) * 32 * CHAINS * (threads / 32);  // per SM
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("chains %d threads %4d: %.3f ms  %.2f cycles per warp-row per SM (ALU-bound ~%.2f)\n", CHAINS, threads, ms,
           cyc / warp_rows, 11.0 / 2.0);
    cudaFree(out);
}

int main() {
    for (int t : {256, 512}) {
        run<1>(t);
        run<2>(t);
        run<4>(t);
    }
    return 0;
}
