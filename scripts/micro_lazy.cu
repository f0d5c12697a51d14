// Microbenchmark: register-resident butterflies, fully reduced (p < 2^31, residues in [0, p)) vs
// Harvey's lazy butterflies (p < 2^30: DIF values in [0, 2p), DIT values in [0, 4p), no reduction
// after the Shoup product).  Same harness as micro_bfly.cu (16 values per thread, 4 twiddles).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_lazy micro_lazy.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t red1(uint32_t x, uint32_t p) { return min(x, x - p); }
__device__ __forceinline__ uint32_t addm(uint32_t a, uint32_t b, uint32_t p) { uint32_t s = a + b; return min(s, s - p); }
__device__ __forceinline__ uint32_t subm(uint32_t a, uint32_t b, uint32_t p) { uint32_t d = a - b; return min(d, d + p); }
__device__ __forceinline__ uint32_t shoup(uint32_t x, uint32_t w, uint32_t wq, uint32_t p) {
    uint32_t q = __umulhi(x, wq); return x * w - q * p; }

constexpr int V = 16;

template <int MODE>
__global__ void __launch_bounds__(256) kbfly(uint32_t *out, const uint32_t *tw, int iters, uint32_t p) {
    uint32_t v[V];
    for (int i = 0; i < V; ++i) v[i] = (threadIdx.x * 7 + i * 13) % p;
    uint32_t w[4], wq[4];
    for (int i = 0; i < 4; ++i) { w[i] = tw[(threadIdx.x + i) & 255]; wq[i] = tw[256 + ((threadIdx.x + i) & 255)]; }
    const uint32_t p2 = 2 * p;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < V / 2; ++i) {
            uint32_t &a = v[i], &b = v[i + V / 2];
            const uint32_t W = w[i & 3], Wq = wq[i & 3];
            if (MODE == 0) {  // GS, fully reduced
                uint32_t d = a - b + p; a = addm(a, b, p); b = red1(shoup(d, W, Wq, p), p);
            } else if (MODE == 1) {  // CT, fully reduced
                uint32_t t = red1(shoup(b, W, Wq, p), p); b = subm(a, t, p); a = addm(a, t, p);
            } else if (MODE == 2) {  // GS lazy: [0, 2p) -> [0, 2p)
                uint32_t d = a - b + p2; a = addm(a, b, p2); b = shoup(d, W, Wq, p);
            } else {  // CT lazy: [0, 4p) -> [0, 4p)
                uint32_t a0 = red1(a, p2); uint32_t t = shoup(b, W, Wq, p); b = a0 - t + p2; a = a0 + t;
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
    int dev = 0, nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const uint32_t pbig = 2147352577u, plazy = 1073479681u;
    uint32_t *tw, *out; cudaMalloc(&tw, 2048 * 4); cudaMalloc(&out, 1 << 24);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char *names[4] = {"GS_full", "CT_full", "GS_lazy", "CT_lazy"};
    for (int mode = 0; mode < 4; ++mode) {
        const uint32_t p = mode < 2 ? pbig : plazy;
        uint32_t htw[512];
        for (int i = 0; i < 256; ++i) { htw[i] = (uint32_t)((1234567ull * (i + 1)) % p); htw[256 + i] = (uint32_t)(((uint64_t)htw[i] << 32) / p); }
        cudaMemcpy(tw, htw, sizeof(htw), cudaMemcpyHostToDevice);
        for (int bpsm : {8, 4, 2}) {
            const int blocks = nsm * bpsm, iters = 4000;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                switch (mode) {
                    case 0: kbfly<0><<<blocks, 256>>>(out, tw, iters, p); break;
                    case 1: kbfly<1><<<blocks, 256>>>(out, tw, iters, p); break;
                    case 2: kbfly<2><<<blocks, 256>>>(out, tw, iters, p); break;
                    default: kbfly<3><<<blocks, 256>>>(out, tw, iters, p); break;
                }
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                double bf = (double)blocks * 256 * iters * (V / 2);
                if (rep) printf("{\"kernel\": \"%s\", \"warps_per_sm\": %d, \"ms\": %.3f, \"bfly_per_clk_per_sm\": %.2f}\n",
                                names[mode], bpsm * 8, ms, bf / (ms * 1e-3) / nsm / (clk * 1e3));
            }
        }
    }
    return 0;
}
