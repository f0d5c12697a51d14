// Instruction-mix microbenchmark (sm_100a): cycles per warp-op per SMSP for fixed mixes of
// IMAD.HI / IMAD / IADD3 / VIADDMNMX with V independent chains per thread (z: opaque zero).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
constexpr int V = 16;
template <int MODE>
__global__ void __launch_bounds__(256) k(uint32_t *out, int iters, uint32_t c0, uint32_t c1, uint32_t z) {
    uint32_t v[V];
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = threadIdx.x * 7u + i * 13u + c1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < V; ++i) {
            uint32_t x = v[i], y = v[(i + 5) % V];
            uint32_t r;
            if (MODE == 0) { r = __umulhi(x, c0); r = r + y + z; r = r + c1 + z; r = r + y + z; r = r + c0 + z; }          // hi + 4 iadd3
            else if (MODE == 1) { r = x * c0; r = r * c1; r = r + y + z; r = r + c1 + z; r = r + y + z; r = r + c0 + z; }  // 2 lo + 4 iadd3
            else if (MODE == 2) { uint32_t q = __umulhi(x, c0); r = x * c1 - q * c0; r = r + y + z; r = r + c1 + z; r = r + y + z; r = r + c0 + z; } // shoup + 4 iadd3
            else if (MODE == 3) { uint32_t q = __umulhi(x, c0); r = x * c1 - q * c0; r = min(r, r - c1); r = min(r + y, r - c0); r = min(r, r - c1 + y); r = min(r + c1, r - y); } // shoup + 4 mnmx-ish
            else if (MODE == 4) { r = min(x, x - c1); r = min(r, r - c0); r = min(r, r - c1); r = min(r, r - y); }  // 4 viaddmnmx
            else if (MODE == 5) { uint32_t q = __umulhi(x, c0); r = x * c1 - q * c0; }  // shoup
            else if (MODE == 6) { r = __umulhi(x, c0); r = __umulhi(r, c1); r = r + y + z; r = r + c1 + z; r = r + y + z; r = r + c0 + z; } // 2 hi + 4 iadd3
            else if (MODE == 7) { r = x + y + z; r = r + c1 + z; r = r + y + z; r = r + c0 + z; }  // 4 iadd3
            else if (MODE == 8) { r = __umulhi(x, c0); r = r + y + z; }  // hi + 1 iadd3
            else if (MODE == 9) { r = __umulhi(x, c0); r = r + y + z; r = r + c1 + z; }  // hi + 2 iadd3
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
    uint32_t *out; cudaMalloc(&out, 1 << 24);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char *names[10] = {"hi+4add3", "2lo+4add3", "shoup+4add3", "shoup+4mnmx", "4mnmx", "shoup", "2hi+4add3", "4add3", "hi+1add3", "hi+2add3"};
    const int blocks = nsm * 8, iters = 2000;
    for (int mode = 0; mode < 10; ++mode)
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
#define C(M) case M: k<M><<<blocks, 256>>>(out, iters, 0x9e3779b9u, 2147352577u, 0u); break;
                C(0) C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9)
#undef C
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double warp_ops_per_smsp = (double)blocks * 8 * iters * V / nsm / 4;
            const double cyc = ms * 1e-3 * clk * 1e3;
            if (rep) printf("{\"mix\": \"%s\", \"cycles_per_warp_op_per_smsp\": %.2f}\n", names[mode], cyc / warp_ops_per_smsp);
        }
    return 0;
}
