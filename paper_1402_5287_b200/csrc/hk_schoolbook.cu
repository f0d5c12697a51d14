// hk_schoolbook.cu -- companion A6: the direct schoolbook matvec on limbs,
// y_i = sum_j a_{idx(i,j)} x_j, without any transform.
//
// One CTA per output row.  For every j the CTA stages the two operands' 32-bit limbs in shared
// memory; thread t owns output columns t, t + T, ... and product-scans
// sum_u A32[u] X32[col - u] into a 128-bit two's-complement column accumulator (adding for a
// positive sign product, subtracting for a negative one).  |column| < n L32 2^64, far below
// 2^127.  A final carry pass converts the columns (bit weight 2^(32 col)) into Ly 64-bit limbs
// mod 2^(64 Ly) and then to sign-magnitude.
#include <cuda_runtime.h>

#include <cstdio>

#include "hk_internal.h"

namespace hk {

constexpr int kSbThreads = 512;
constexpr int kSbMaxCols = 8;  // 2 L32 <= 4096 -> L <= 1024

__global__ void __launch_bounds__(kSbThreads)
k6_schoolbook(int kind, int64_t m, int64_t n, int L, const uint64_t *__restrict__ a_mag,
              const int8_t *__restrict__ a_sign, const uint64_t *__restrict__ x_mag,
              const int8_t *__restrict__ x_sign, uint64_t *__restrict__ y_mag,
              int8_t *__restrict__ y_sign) {
    extern __shared__ uint32_t sm[];
    const int L32 = 2 * L;
    uint32_t *A = sm;          // [L32]
    uint32_t *X = sm + L32;    // [L32]
    const int tid = threadIdx.x;
    const int64_t i = blockIdx.x;
    const int ncol = 2 * L32 - 1;
    unsigned __int128 acc[kSbMaxCols];
#pragma unroll
    for (int c = 0; c < kSbMaxCols; ++c) acc[c] = 0;

    for (int64_t j = 0; j < n; ++j) {
        int64_t k;
        if (kind == HK_HANKEL) k = i + j;
        else if (kind == HK_TOEPLITZ) k = (n - 1) - i + j;
        else k = ((i - j) % n + n) % n;
        const int s = (int)a_sign[k] * (int)x_sign[j];
        if (s == 0) continue;  // uniform across the CTA
        __syncthreads();
        const uint32_t *a32 = (const uint32_t *)(a_mag + k * L);
        const uint32_t *x32 = (const uint32_t *)(x_mag + j * L);
        for (int u = tid; u < L32; u += kSbThreads) {
            A[u] = a32[u];
            X[u] = x32[u];
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < kSbMaxCols; ++c) {
            const int col = tid + c * kSbThreads;
            if (col >= ncol) break;
            const int ulo = col - L32 + 1 > 0 ? col - L32 + 1 : 0;
            const int uhi = col < L32 - 1 ? col : L32 - 1;
            unsigned __int128 sum = 0;
            for (int u = ulo; u <= uhi; ++u) sum += (uint64_t)A[u] * X[col - u];
            if (s > 0) acc[c] += sum; else acc[c] -= sum;
        }
    }
    __syncthreads();
    // columns -> shared (reuse the staging area; 16 bytes per column)
    unsigned __int128 *cols = (unsigned __int128 *)sm;
#pragma unroll
    for (int c = 0; c < kSbMaxCols; ++c) {
        const int col = tid + c * kSbThreads;
        if (col < ncol) cols[col] = acc[c];
    }
    __syncthreads();
    if (tid == 0) {
        const int Ly = 2 * L + 1;
        uint64_t *y = y_mag + i * Ly;
        __int128 carry = 0;
        // 32-bit output words; word w gets column w plus the carry
        uint64_t lo_word = 0;
        for (int wd = 0; wd < 2 * Ly; ++wd) {
            __int128 v = carry;
            if (wd < ncol) v += (__int128)cols[wd];
            const uint32_t word = (uint32_t)(uint64_t)v;
            carry = v >> 32;  // arithmetic shift: exact floor division
            if (wd & 1) y[wd >> 1] = lo_word | ((uint64_t)word << 32);
            else lo_word = word;
        }
        const bool neg = (int64_t)y[Ly - 1] < 0;
        int z = Ly;
        for (int l = 0; l < Ly; ++l)
            if (y[l]) { z = l; break; }
        if (neg) {
            for (int l = z; l < Ly; ++l) y[l] = (l == z) ? (0ull - y[l]) : ~y[l];
        }
        y_sign[i] = neg ? (int8_t)-1 : (z < Ly ? (int8_t)1 : (int8_t)0);
    }
}

int launch_schoolbook(int kind, int64_t m, int64_t n, int32_t P, const uint64_t *a_mag,
                      const int8_t *a_sign, const uint64_t *x_mag, const int8_t *x_sign,
                      uint64_t *y_mag, int8_t *y_sign, void *stream) {
    const int L = (P + 63) / 64;
    if (2 * (2 * L) - 1 > kSbThreads * kSbMaxCols) return HK_EUNSUPPORTED;
    size_t smem = (size_t)(2 * (2 * L)) * sizeof(uint32_t);
    const size_t csmem = (size_t)(4 * L) * 16;
    if (csmem > smem) smem = csmem;
    if (cudaFuncSetAttribute(k6_schoolbook, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return HK_ECUDA;
    k6_schoolbook<<<(unsigned)m, kSbThreads, smem, (cudaStream_t)stream>>>(
        kind, m, n, L, a_mag, a_sign, x_mag, x_sign, y_mag, y_sign);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "hk: schoolbook launch error: %s\n", cudaGetErrorString(e));
        return HK_ECUDA;
    }
    return HK_OK;
}

}  // namespace hk
