// Butterfly formulations vs SASS pipe mix (sm_100a).  z is an opaque zero (kernel argument):
// s = a + b + z must be a 3-input IADD3 (ALU pipe) — ptxas cannot turn it into IMAD.IADD, which
// would load the FMA pipe that IMAD.HI (rate 1/4) already binds.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t shoup(uint32_t x, uint32_t w, uint32_t wq, uint32_t p) {
    uint32_t q = __umulhi(x, wq); return x * w - q * p; }
constexpr int V = 16;
template <int MODE>
__global__ void __launch_bounds__(256) k(uint32_t *out, const uint32_t *tw, int iters, uint32_t p, uint32_t z) {
    uint32_t v[V];
    for (int i = 0; i < V; ++i) v[i] = (threadIdx.x * 7 + i * 13) % p;
    uint32_t w[4], wq[4];
    for (int i = 0; i < 4; ++i) { w[i] = tw[(threadIdx.x + i) & 255]; wq[i] = tw[256 + ((threadIdx.x + i) & 255)]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < V / 2; ++i) {
            uint32_t &a = v[i], &b = v[i + V / 2];
            const uint32_t W = w[i & 3], Wq = wq[i & 3];
            if (MODE == 0) {  // GS as in hk_modarith.cuh
                uint32_t d = a - b + p; uint32_t s = a + b; a = min(s, s - p); uint32_t r = shoup(d, W, Wq, p); b = min(r, r - p);
            } else if (MODE == 1) {  // GS, opaque-zero 3-input add
                uint32_t d = a - b + p; uint32_t s = a + b + z; a = min(s, s - p); uint32_t r = shoup(d, W, Wq, p); b = min(r, r - p);
            } else if (MODE == 2) {  // CT as in hk_modarith.cuh
                uint32_t r = shoup(b, W, Wq, p); uint32_t t = min(r, r - p); uint32_t d = a - t; b = min(d, d + p); uint32_t s = a + t; a = min(s, s - p);
            } else if (MODE == 3) {  // CT, opaque zero
                uint32_t r = shoup(b, W, Wq, p); uint32_t t = min(r, r - p); uint32_t d = a - t + z; b = min(d, d + p); uint32_t s = a + t + z; a = min(s, s - p);
            } else if (MODE == 4) {  // CT, t in [0,2p) kept lazy: d = a - r + 2p in (0, 3p)?  no: use a + (2p - r)
                uint32_t r = shoup(b, W, Wq, p); uint32_t t = min(r, r - p); uint32_t d = a - t + p; b = min(d, d - p); uint32_t s = a + t + z; a = min(s, s - p);
            }
        }
#pragma unroll
        for (int i = 0; i < V / 2; ++i) { uint32_t t = v[i]; v[i] = v[i + V / 2]; v[i + V / 2] = t; }
    }
    uint32_t s = 0;
    for (int i = 0; i < V; ++i) s ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const uint32_t p = 2147352577u;
    uint32_t htw[512];
    for (int i = 0; i < 256; ++i) { htw[i] = (uint32_t)((1234567ull * (i + 1)) % p); htw[256 + i] = (uint32_t)(((uint64_t)htw[i] << 32) / p); }
    uint32_t *tw, *out; cudaMalloc(&tw, sizeof(htw)); cudaMalloc(&out, 1 << 24);
    cudaMemcpy(tw, htw, sizeof(htw), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char *names[5] = {"GS", "GS_opaque0", "CT", "CT_opaque0", "CT_alt"};
    const int blocks = nsm * 8, iters = 4000;
    for (int mode = 0; mode < 5; ++mode)
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
#define C(M) case M: k<M><<<blocks, 256>>>(out, tw, iters, p, 0u); break;
                C(0) C(1) C(2) C(3) C(4)
#undef C
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double bf = (double)blocks * 256 * iters * (V / 2);
            if (rep) printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"bfly_per_clk_per_sm\": %.2f}\n", names[mode], ms, bf / (ms * 1e-3) / nsm / (clk * 1e3));
        }
    return 0;
}
