// Pipe-rate microbenchmark for the integer instructions of the NTT butterflies on sm_100a.
// Each variant runs V independent chains per thread of one instruction kind (or a fixed mix);
// reports warp-instructions per clock per SM for the measured kind(s).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_pipes micro_pipes.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int V = 16;

template <int MODE>
__global__ void __launch_bounds__(256) kpipe(uint32_t *out, uint32_t c0, uint32_t c1, int iters) {
    uint32_t v[V];
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = threadIdx.x * 7u + i * 13u + c1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < V; ++i) {
            uint32_t x = v[i], r;
            if (MODE == 0) {  // IMAD.HI
                asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(c0));
            } else if (MODE == 1) {  // IMAD (lo)
                asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(c0));
            } else if (MODE == 2) {  // IMAD (mad lo)
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(c0), "r"(c1));
            } else if (MODE == 3) {  // IADD3 (3-input add)
                asm volatile("{.reg .u32 t; add.u32 t, %1, %2; add.u32 %0, t, %3;}" : "=r"(r) : "r"(x), "r"(c0), "r"(v[(i + 1) % V]));
            } else if (MODE == 4) {  // min
                asm volatile("min.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(c0));
                r += 1;
            } else if (MODE == 5) {  // xor (LOP3)
                asm volatile("xor.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(c0));
            } else if (MODE == 6) {  // mul.wide.u32 (IMAD.WIDE)
                uint64_t z;
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(z) : "r"(x), "r"(c0));
                r = (uint32_t)z ^ (uint32_t)(z >> 32);
            } else if (MODE == 7) {  // Shoup product: hi + 2 lo
                const uint32_t q = __umulhi(x, c0);
                r = x * c1 - q * 2147352577u;
            } else if (MODE == 8) {  // hi + xor (fma + alu mix)
                asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(c0));
                r ^= c1;
            } else if (MODE == 9) {  // lo + xor
                asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(c0));
                r ^= c1;
            }
            v[i] = r;
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < V; ++i) s ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t *out;
    cudaMalloc(&out, 1 << 24);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[10] = {"mul.hi", "mul.lo", "mad.lo", "add3", "min+add", "xor", "mul.wide", "shoup(hi+2lo)", "hi+xor", "lo+xor"};
    const int instr_per[10] = {1, 1, 1, 1, 2, 1, 1, 3, 2, 2};
    const int blocks = nsm * 8, iters = 4000;
    for (int mode = 0; mode < 10; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
#define C(M) case M: kpipe<M><<<blocks, 256>>>(out, 0x9e3779b9u, 12345u, iters); break;
                C(0) C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9)
#undef C
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double warp_ops = (double)blocks * 8 * iters * V;  // per "op" of the mode
            const double per_clk_sm = warp_ops / (ms * 1e-3) / nsm / (clk * 1e3);
            if (rep)
                printf("{\"mode\": \"%s\", \"ms\": %.3f, \"warp_ops_per_clk_per_sm\": %.3f, \"warp_instr_per_clk_per_sm\": %.3f}\n",
                       names[mode], ms, per_clk_sm, per_clk_sm * instr_per[mode]);
        }
    }
    printf("{\"sms\": %d, \"clock_khz\": %d}\n", nsm, clk);
    return 0;
}
