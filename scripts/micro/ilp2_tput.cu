// Microbenchmark: does a lane running TWO independent column words (two K1+K3
// states, rows interleaved) beat one word per lane at the same resident warps?
// (ILP instead of TLP for the fixed-latency dependency stalls of the hot loop.)
#include "../../paper_1307_2560_b200/csrc/ychg_scan.cu"
#include <cstdio>

using namespace ychg_dev;

template <int J>
__device__ __forceinline__ void process_block_ilp(const uint8_t* const* stage, int lane, LaneState* s,
                                                  uint32_t mul2, uint32_t mulnb, uint32_t mul1) {
    uint32_t Pprev[J], tA[J], fA[J], eA[J];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const uint8_t* p = stage[j] + 4 * lane;
            const uint8_t* r0 = p + (2 * q) * kBoxBytes;
            const uint8_t* r1 = r0 + kBoxBytes;
            uint32_t a0 = __byte_perm(*reinterpret_cast<const uint32_t*>(r0), 0u, 0x0123u);
            uint32_t a1 = __byte_perm(*reinterpret_cast<const uint32_t*>(r1), 0u, 0x0123u);
            const uint32_t P = lop3<0x3A>(a0, s[j].pa, a1);
            const uint32_t b0 = right_neighbour_msb(a0, r0[4], mul2, mulnb);
            const uint32_t b1 = right_neighbour_msb(a1, r1[4], mul2, mulnb);
            uint32_t apa0, apa1;
            const uint32_t l0 = k3_step<false>(a0, b0, s[j], apa0);
            const uint32_t l1 = k3_step<false>(a1, b1, s[j], apa1);
            s[j].links = __popc(l0 * mul1 + l1) * mul1 + s[j].links;
            if ((q & 1) == 0) { Pprev[j] = P; continue; }
            const int m = q >> 1;
            uint32_t t;
            csa(t, s[j].ones, s[j].ones, Pprev[j], P);
            if ((m & 1) == 0) { tA[j] = t; continue; }
            uint32_t f;
            csa(f, s[j].twos, s[j].twos, tA[j], t);
            if ((m & 2) == 0) { fA[j] = f; continue; }
            uint32_t e;
            csa(e, s[j].fours, s[j].fours, fA[j], f);
            if ((m & 4) == 0) { eA[j] = e; continue; }
            uint32_t sixteens;
            csa(sixteens, s[j].eights, s[j].eights, eA[j], e);
            const uint32_t c1 = s[j].u16 & sixteens;
            const uint32_t c2 = s[j].u32 & c1;
            const uint32_t c3 = s[j].u64 & c2;
            s[j].u16 ^= sixteens;
            s[j].u32 ^= c1;
            s[j].u64 ^= c2;
            s[j].u128 ^= c3;
        }
    }
}

template <int J>
__global__ void __launch_bounds__(128) blk(uint32_t* out, int iters, uint32_t mul2, uint32_t mulnb) {
    __shared__ __align__(128) uint8_t stage[J][kStageBytes];
    for (int i = threadIdx.x; i < J * kStageBytes; i += blockDim.x)
        (&stage[0][0])[i] = static_cast<uint8_t>((i * 2654435761u) >> 13);
    __syncthreads();
    LaneState s[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        s[j] = LaneState{};
        s[j].mk3 = 0xFFFFFFFFu;
    }
    const uint8_t* st[J];
#pragma unroll
    for (int j = 0; j < J; ++j) st[j] = stage[j];
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
        asm volatile("" ::: "memory");
        process_block_ilp<J>(st, lane, s, mul2, mulnb, mul2 >> 1);
        if ((it & 15) == 15)
#pragma unroll
            for (int j = 0; j < J; ++j) flush_counts(s[j]);
    }
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
        r ^= s[j].links ^ s[j].G2 ^ s[j].G3;
        for (int i = 0; i < 16; ++i) r ^= s[j].acc[i];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int J>
void run(int blocks_per_sm) {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* out;
    cudaMalloc(&out, sms * blocks_per_sm * 128 * 4);
    blk<J><<<sms * blocks_per_sm, 128>>>(out, 4, 2, 1u << 25);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 400;
    cudaEventRecord(a);
    blk<J><<<sms * blocks_per_sm, 128>>>(out, iters, 2, 1u << 25);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_rows = double(iters) * 32 * 4 * blocks_per_sm * J;  // word-rows per SM
    printf("ILP %d: 128 threads x %d CTA/SM (%2d warps): %.3f ms  %.2f cycles per word-row per SM\n", J, blocks_per_sm,
           4 * blocks_per_sm, ms, ms * 1e-3 * clk * 1e3 / warp_rows);
    cudaFree(out);
}

int main() {
    for (int b : {1, 2, 3, 4}) run<1>(b);
    for (int b : {1, 2, 3}) run<2>(b);
    return 0;
}
