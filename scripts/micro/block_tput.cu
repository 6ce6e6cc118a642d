// Microbenchmark: ychg process_block (the real hot loop) on one resident smem stage,
// looped -- measures the hot loop's compute rate without TMA, barriers or merges.
#include "../../paper_1307_2560_b200/csrc/ychg_scan.cu"
#include <cstdio>

using namespace ychg_dev;

template <bool kHead, bool kLinks = true>
__global__ void __launch_bounds__(256) blk(uint32_t* out, int iters, uint32_t mul2, uint32_t mul17) {
    __shared__ __align__(128) uint8_t stage[kStageBytes];
    for (int i = threadIdx.x; i < kStageBytes; i += blockDim.x) stage[i] = static_cast<uint8_t>((i * 2654435761u) >> 13);
    __syncthreads();
    LaneState s{};
    s.mk3 = 0xFFFFFFFFu;
    s.Hd = kHead ? 0xFFFFFFFFu : 0u;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
        asm volatile("" ::: "memory");  // force the smem reloads every iteration (no hoisting)
        process_block<kLinks, kHead, false>(stage, lane, s, Muls{mul2, mul17, mul2 >> 1, 0u - (mul2 >> 1)});
        if ((it & 15) == 15) flush_counts(s);
    }
    uint32_t r = s.links ^ s.G2 ^ s.G3 ^ s.h1;
    for (int i = 0; i < 16; ++i) r ^= s.acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <bool kHead, bool kLinks = true>
void run(int threads, int blocks_per_sm) {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* out;
    cudaMalloc(&out, sms * blocks_per_sm * threads * 4);
    blk<kHead, kLinks><<<sms * blocks_per_sm, threads>>>(out, 4, 2, 1u << 25);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 400;
    cudaEventRecord(a);
    blk<kHead, kLinks><<<sms * blocks_per_sm, threads>>>(out, iters, 2, 1u << 25);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_rows = double(iters) * 32 * (threads / 32) * blocks_per_sm;  // per SM
    printf("links=%d head=%d threads %d x %d CTA/SM: %.3f ms  %.2f cycles per warp-row per SM\n", kLinks, kHead, threads,
           blocks_per_sm, ms, ms * 1e-3 * clk * 1e3 / warp_rows);
    cudaFree(out);
}

int main() {
    run<false>(128, 1);  // the streaming CTA shape (4 warps): 1..3 resident per SM
    run<false>(128, 2);
    run<false>(128, 3);
    run<false>(256, 1);
    run<false>(256, 2);
    run<false>(256, 4);
    run<true>(256, 2);
    run<false, false>(256, 2);
    return 0;
}
