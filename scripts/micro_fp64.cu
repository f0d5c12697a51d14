// FP64-pipe microbenchmark on sm_100a: is the double-precision pipe a second modular-multiply
// unit beside the integer FMA pipe ("next")?  Each variant runs V
// independent chains per thread; reports warp-operations per clock per SM.
//   dfma, dmul            raw FP64 pipe rate
//   dfma+imad.hi          one of each per element: co-issue if the rate stays at the slower one
//   f64 modmul            a*b mod p for a 50-bit prime with FMA error-free product + rint quotient
//   i32 shoup             the integer Shoup product the NTT kernels use (IMAD.HI + 2 IMAD)
//   f64 modmul + i32 shoup  both on disjoint chains in the same loop (combined modmuls / clk)
//   cvt                   I2F.F64 + F2I round trip
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_fp64 micro_fp64.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int V = 16;

__device__ __forceinline__ double modmul_f64(double a, double b, double p, double pinv) {
    const double h = a * b;
    const double l = fma(a, b, -h);        // a b = h + l exactly
    const double q = rint(h * pinv);
    double r = fma(-q, p, h) + l;          // |r| < p (a, b < p < 2^50)
    r = r < 0.0 ? r + p : r;
    return r >= p ? r - p : r;
}

template <int MODE>
__global__ void __launch_bounds__(256) kf(double *outd, uint32_t *outu, double c0, double c1, uint32_t u0,
                                          uint32_t u1, int iters) {
    double d[V];
    uint32_t v[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
        d[i] = (double)(threadIdx.x * 7 + i * 13 + 1);
        v[i] = threadIdx.x * 7u + i * 13u + u1;
    }
    const double p = 1125899906826241.0, pinv = 1.0 / p;  // 2^50 - 2^14 + 1 (any odd < 2^50)
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < V; ++i) {
            if (MODE == 0) {
                d[i] = fma(d[i], c0, c1);
            } else if (MODE == 1) {
                d[i] = d[i] * c0;
            } else if (MODE == 2) {
                d[i] = fma(d[i], c0, c1);
                v[i] = __umulhi(v[i], u0) ^ u1;
            } else if (MODE == 3) {
                d[i] = modmul_f64(d[i], c0, p, pinv);
            } else if (MODE == 4) {
                const uint32_t q = __umulhi(v[i], u0);
                v[i] = v[i] * u1 - q * 2147352577u;
            } else if (MODE == 5) {
                if (i & 1) {
                    d[i] = modmul_f64(d[i], c0, p, pinv);
                } else {
                    const uint32_t q = __umulhi(v[i], u0);
                    v[i] = v[i] * u1 - q * 2147352577u;
                }
            } else if (MODE == 6) {
                d[i] = (double)(uint32_t)(d[i] * c0) + c1;
            }
        }
    }
    double s = 0;
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        s += d[i];
        t ^= v[i];
    }
    outd[blockIdx.x * blockDim.x + threadIdx.x] = s;
    outu[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *od;
    uint32_t *ou;
    cudaMalloc(&od, 1 << 25);
    cudaMalloc(&ou, 1 << 24);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[7] = {"dfma", "dmul", "dfma+imad.hi", "f64 modmul (50-bit p)", "i32 shoup (31-bit p)",
                            "f64 modmul + i32 shoup (half each)", "cvt f64->u32->f64 + dadd"};
    const int blocks = nsm * 8, iters = 2000;
    for (int mode = 0; mode < 7; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
#define C(M) case M: kf<M><<<blocks, 256>>>(od, ou, 1.0000001, 0.5, 0x9e3779b9u, 12345u, iters); break;
                C(0) C(1) C(2) C(3) C(4) C(5) C(6)
#undef C
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double warp_ops = (double)blocks * 8 * iters * V;  // per element-operation of the mode
            const double per_clk_sm = warp_ops / (ms * 1e-3) / nsm / (clk * 1e3);
            if (rep)
                printf("{\"mode\": \"%s\", \"ms\": %.3f, \"warp_ops_per_clk_per_sm\": %.3f, \"lane_ops_per_clk_per_sm\": %.1f}\n",
                       names[mode], ms, per_clk_sm, per_clk_sm * 32);
        }
    }
    printf("{\"sms\": %d, \"clock_khz\": %d}\n", nsm, clk);
    return 0;
}
