// K7 microbenchmark: register-resident 31-bit butterfly throughput on sm_100a.
// Measures warp-butterflies / clock / SM for the GS (DIF) and CT (DIT) butterflies with
// Shoup (W, W') twiddles and with Montgomery (4-byte) twiddles, plus a plain HBM copy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_bfly micro_bfly.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t red1(uint32_t x, uint32_t p) { return min(x, x - p); }
__device__ __forceinline__ uint32_t addm(uint32_t a, uint32_t b, uint32_t p) { uint32_t s = a + b; return min(s, s - p); }
__device__ __forceinline__ uint32_t subm(uint32_t a, uint32_t b, uint32_t p) { uint32_t d = a - b; return min(d, d + p); }
__device__ __forceinline__ uint32_t shoup(uint32_t x, uint32_t w, uint32_t wq, uint32_t p) {
    uint32_t q = __umulhi(x, wq); return x * w - q * p; }
// ALU-only addition mod p: min(a + b, a + b - p) as IADD3 + VIADDMNMX (no IMAD.IADD)
__device__ __forceinline__ uint32_t addm2(uint32_t a, uint32_t b, uint32_t p) {
    uint32_t t, r;
    asm("add.u32 %0, %1, %2;" : "=r"(t) : "r"(a), "r"(b));
    asm volatile("{.reg .u32 q; sub.u32 q, %1, %2; min.u32 %0, %1, q;}" : "=r"(r) : "r"(t), "r"(p));
    return r;
}
__device__ __forceinline__ uint32_t addm3(uint32_t a, uint32_t b, uint32_t p) {
    const uint32_t t = a + b - p;       // IADD3
    return min(a + b, t);               // VIADDMNMX(a, b, t)?
}
__device__ __forceinline__ uint32_t montr(uint32_t a, uint32_t b, uint32_t p, uint32_t pneg) {
    uint64_t z = (uint64_t)a * b; uint32_t m = (uint32_t)z * pneg; uint64_t t = z + (uint64_t)m * p;
    return (uint32_t)(t >> 32); }

constexpr int V = 16;  // independent values per thread

template <int MODE>
__global__ void __launch_bounds__(256) kbfly(uint32_t *out, const uint32_t *tw, int iters, uint32_t p, uint32_t pneg) {
    uint32_t v[V];
    for (int i = 0; i < V; ++i) v[i] = (threadIdx.x * 7 + i * 13) % p;
    uint32_t w[4], wq[4];
    for (int i = 0; i < 4; ++i) { w[i] = tw[(threadIdx.x + i) & 255]; wq[i] = tw[256 + ((threadIdx.x + i) & 255)]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < V / 2; ++i) {
            uint32_t &a = v[i], &b = v[i + V / 2];
            const uint32_t W = w[i & 3], Wq = wq[i & 3];
            if (MODE == 0) {  // GS Shoup
                uint32_t d = a - b + p; a = addm(a, b, p); b = red1(shoup(d, W, Wq, p), p);
            } else if (MODE == 1) {  // CT Shoup
                uint32_t t = red1(shoup(b, W, Wq, p), p); b = subm(a, t, p); a = addm(a, t, p);
            } else if (MODE == 4) {  // GS Shoup, addm3
                uint32_t d = a - b + p; a = addm3(a, b, p); b = red1(shoup(d, W, Wq, p), p);
            } else if (MODE == 5) {  // CT Shoup, addm3 / subm via min(a - t, a - t + p)
                uint32_t t = red1(shoup(b, W, Wq, p), p); uint32_t d2 = a - t + p; b = min(a - t, d2); a = addm3(a, t, p);
            } else if (MODE == 6) {  // GS Shoup, asm add
                uint32_t d = a - b + p; a = addm2(a, b, p); b = red1(shoup(d, W, Wq, p), p);
            } else if (MODE == 2) {  // GS Montgomery
                uint32_t d = a - b + p; a = addm(a, b, p); b = red1(montr(d, W, p, pneg), p);
            } else {  // CT Montgomery
                uint32_t t = red1(montr(b, W, p, pneg), p); b = subm(a, t, p); a = addm(a, t, p);
            }
        }
#pragma unroll
        for (int i = 0; i < V / 2; ++i) { uint32_t t = v[i]; v[i] = v[i + V / 2]; v[i + V / 2] = t; }
    }
    uint32_t s = 0;
    for (int i = 0; i < V; ++i) s ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void kcopy(const uint4 *__restrict__ a, uint4 *__restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const uint32_t p = 2147352577u;
    uint32_t inv = 1; for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
    const uint32_t pneg = 0u - inv;
    uint32_t htw[512];
    for (int i = 0; i < 256; ++i) { htw[i] = (uint32_t)((1234567ull * (i + 1)) % p); htw[256 + i] = (uint32_t)(((uint64_t)htw[i] << 32) / p); }
    uint32_t *tw, *out; cudaMalloc(&tw, sizeof(htw)); cudaMalloc(&out, 1 << 24);
    cudaMemcpy(tw, htw, sizeof(htw), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char *names[7] = {"GS_shoup", "CT_shoup", "GS_mont", "CT_mont", "GS_addm3", "CT_addm3", "GS_asm"};
    const int blocks = nsm * 8, iters = 4000;
    for (int mode = 0; mode < 7; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
                case 0: kbfly<0><<<blocks, 256>>>(out, tw, iters, p, pneg); break;
                case 1: kbfly<1><<<blocks, 256>>>(out, tw, iters, p, pneg); break;
                case 2: kbfly<2><<<blocks, 256>>>(out, tw, iters, p, pneg); break;
                case 3: kbfly<3><<<blocks, 256>>>(out, tw, iters, p, pneg); break;
                case 4: kbfly<4><<<blocks, 256>>>(out, tw, iters, p, pneg); break;
                case 5: kbfly<5><<<blocks, 256>>>(out, tw, iters, p, pneg); break;
                default: kbfly<6><<<blocks, 256>>>(out, tw, iters, p, pneg); break;
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double bf = (double)blocks * 256 * iters * (V / 2);
            if (rep) printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"Gbfly_per_s\": %.1f, \"bfly_per_clk_per_sm_at_max_clock\": %.2f}\n",
                            names[mode], ms, bf / ms / 1e6, bf / (ms * 1e-3) / nsm / (clk * 1e3));
        }
    }
    size_t n = (size_t)1 << 27;  // 2 GiB per buffer as uint4
    uint4 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16); cudaMemset(a, 1, n * 16);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0); kcopy<<<nsm * 8, 512>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("{\"kernel\": \"copy\", \"GBps\": %.1f}\n", 2.0 * n * 16 / ms / 1e6);
    }
    printf("{\"sms\": %d, \"clock_khz\": %d}\n", nsm, clk);
    return 0;
}
