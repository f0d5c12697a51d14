// hk_karatsuba.cu -- companion A5: the paper's Algorithm 1,
// the Karatsuba-like half-size recursion, executed level by level on the GPU.
//
// Level d holds 3^d Hankel subproblems of one uniform size s_d (s_0 = n, s_{d+1} = m1(s_d) =
// ceil((s_d + 1)/2)); the children of size m = floor((s+1)/2) are zero-padded to m1, which is
// exact (the padded x entry is zero, so the extra a entries never meet a non-zero x and the first
// m outputs are unchanged).  Per level:
//   split  (steps 3-6)   c_i = a_{2i-1} + a_{2i}, d_i = a_{2i}, e_i = a_{2i-1},
//                        h_i = x_{2i-1}, f_i = x_{2i-1} - x_{2i}, g_i = x_{2i-2} - x_{2i-1}
//                        children (c, h), (d, f), (e, g)  (step 7)
//   leaves (s <= cutoff) direct products sum_j a_{i+j-1} x_j (step 1's explicit formula for s = 2)
//   merge  (step 8)      y_{2i-1} = p_i - q_i, y_{2i} = p_i + r_i
// Entries are two's-complement big integers: W = L + 1 limbs for a and x (the entries grow by at
// most one bit per level), WY = 2W + 1 limbs for products and sums.  Adds/subtracts run one warp
// per entry with a ballot-based carry-lookahead across lanes.
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>

#include "hk_internal.h"

namespace hk {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxLevels = 40;

struct KLevels {
    int D = 0;                    // leaves live at level D
    int64_t s[kMaxLevels]{};      // subproblem size at level d
    int64_t cnt[kMaxLevels]{};    // 3^d
    size_t offA[kMaxLevels]{}, offX[kMaxLevels]{}, offY[kMaxLevels]{};
    int L = 0, W = 0, WY = 0, Ly = 0;
    size_t total = 0;
};

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

int kplan(int64_t n, int32_t P, int32_t cutoff, KLevels *k) {
    if (n < 1 || P < 1 || cutoff < 2) return HK_EINVAL;
    k->L = (P + 63) / 64;
    k->W = k->L + 1;
    k->WY = 2 * k->W + 1;
    k->Ly = 2 * k->L + 1;
    int64_t s = n, cnt = 1;
    int d = 0;
    k->s[0] = s;
    k->cnt[0] = 1;
    while (s > cutoff) {
        s = (s + 2) / 2;
        cnt *= 3;
        ++d;
        if (d >= kMaxLevels - 1 || cnt > (int64_t(1) << 31)) return HK_EUNSUPPORTED;
        k->s[d] = s;
        k->cnt[d] = cnt;
    }
    k->D = d;
    size_t off = 0;
    for (int l = 0; l <= d; ++l) {
        k->offA[l] = off;
        off = al256(off + (size_t)k->cnt[l] * (2 * k->s[l] - 1) * k->W * 8);
        k->offX[l] = off;
        off = al256(off + (size_t)k->cnt[l] * k->s[l] * k->W * 8);
        k->offY[l] = off;
        off = al256(off + (size_t)k->cnt[l] * k->s[l] * k->WY * 8);
    }
    k->total = off;
    return HK_OK;
}

// lowest index l in [0, nl) with v[l] != 0 (nl if none), warp-cooperative
__device__ int warp_lowest_nonzero(const uint64_t *v, int nl) {
    const int lane = threadIdx.x & 31;
    int z = INT_MAX;
    for (int l = lane; l < nl; l += 32)
        if (v[l]) { z = l; break; }
    z = __reduce_min_sync(kFull, (unsigned)z);
    return z == INT_MAX ? nl : z;
}

// r = a + b or a - b over nl limbs (two's complement); a, b may be null (= 0).  One warp.
__device__ void warp_addsub(uint64_t *r, const uint64_t *a, const uint64_t *b, int nl, bool sub) {
    const int lane = threadIdx.x & 31;
    const int K = (nl + 31) / 32;
    const int l0 = lane * K, l1 = min(nl, l0 + K);
    unsigned c = 0;
    bool ones = true;
    for (int l = l0; l < l1; ++l) {
        const uint64_t x = a ? a[l] : 0ull;
        const uint64_t y = b ? (sub ? ~b[l] : b[l]) : (sub ? ~0ull : 0ull);
        const uint64_t s = x + y;
        const uint64_t s2 = s + c;
        c = (s < x) | (s2 < s);
        ones = ones && (s2 == ~0ull);
    }
    const unsigned G = __ballot_sync(kFull, c != 0);
    const unsigned X = G | __ballot_sync(kFull, ones);
    const unsigned S = X + G + (sub ? 1u : 0u);
    c = ((S ^ X ^ G) >> lane) & 1u;  // carry into this lane's chunk
    for (int l = l0; l < l1; ++l) {
        const uint64_t x = a ? a[l] : 0ull;
        const uint64_t y = b ? (sub ? ~b[l] : b[l]) : (sub ? ~0ull : 0ull);
        const uint64_t s = x + y;
        const uint64_t s2 = s + c;
        c = (s < x) | (s2 < s);
        r[l] = s2;
    }
}

// sign-magnitude (L limbs) -> two's complement (W limbs); one warp per entry
__global__ void k5_to_twos(const uint64_t *__restrict__ mag, const int8_t *__restrict__ sign,
                           int64_t count, int L, int W, uint64_t *__restrict__ dst) {
    const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (e >= count) return;
    const int lane = threadIdx.x & 31;
    const uint64_t *m = mag + e * L;
    const int z = warp_lowest_nonzero(m, L);
    const bool neg = sign[e] < 0;
    for (int l = lane; l < W; l += 32) {
        uint64_t v = l < L ? m[l] : 0ull;
        if (neg) v = l < z ? 0ull : (l == z ? (0ull - v) : ~v);
        dst[e * W + l] = v;
    }
}

// steps 3-6: one warp per child entry.  Parent level: size s, cnt problems; child size s2.
__global__ void k5_split(const uint64_t *__restrict__ A, const uint64_t *__restrict__ X,
                         uint64_t *__restrict__ A2, uint64_t *__restrict__ X2, int64_t cnt,
                         int64_t s, int64_t s2, int W) {
    const int64_t na2 = 2 * s2 - 1;
    const int64_t per = 3 * na2 + 3 * s2;  // child entries per parent
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (wid >= cnt * per) return;
    const int64_t pr = wid / per;
    int64_t k = wid % per;
    const uint64_t *pa = A + pr * (2 * s - 1) * W;
    const uint64_t *px = X + pr * s * W;
    auto Aent = [&](int64_t i) -> const uint64_t * {  // a_i, 1-based, null outside 1..2s-1
        return (i >= 1 && i <= 2 * s - 1) ? pa + (i - 1) * W : nullptr;
    };
    auto Xent = [&](int64_t i) -> const uint64_t * {  // x_i, 1-based, null outside 1..s
        return (i >= 1 && i <= s) ? px + (i - 1) * W : nullptr;
    };
    if (k < 3 * na2) {
        const int c = (int)(k / na2);
        const int64_t i = k % na2 + 1;
        uint64_t *out = A2 + ((3 * pr + c) * na2 + (i - 1)) * W;
        if (c == 0) warp_addsub(out, Aent(2 * i - 1), Aent(2 * i), W, false);       // c_i
        else if (c == 1) warp_addsub(out, Aent(2 * i), nullptr, W, false);         // d_i
        else warp_addsub(out, Aent(2 * i - 1), nullptr, W, false);                 // e_i
    } else {
        k -= 3 * na2;
        const int c = (int)(k / s2);
        const int64_t i = k % s2 + 1;
        uint64_t *out = X2 + ((3 * pr + c) * s2 + (i - 1)) * W;
        if (c == 0) warp_addsub(out, Xent(2 * i - 1), nullptr, W, false);          // h_i
        else if (c == 1) warp_addsub(out, Xent(2 * i - 1), Xent(2 * i), W, true);  // f_i
        else warp_addsub(out, Xent(2 * i - 2), Xent(2 * i - 1), W, true);          // g_i
    }
}

// leaves: one CTA per (problem, output row): y_i = sum_j a_{i+j-1} x_j on two's-complement
// operands (sign + 32-bit magnitude words in smem, 128-bit column sums), result in WY limbs.
constexpr int kLeafThreads = 256;
constexpr int kLeafCols = 16;  // columns per thread: 4W - 1 <= 4096 -> W <= 1024

__device__ void load_signmag(const uint64_t *v, int W, uint32_t *mag32, int *s_z, int *sgn) {
    // block-cooperative: magnitude of the two's-complement value v[0..W)
    const bool neg = (int64_t)v[W - 1] < 0;
    if (threadIdx.x == 0) *s_z = W;
    __syncthreads();
    if (neg) {
        for (int l = threadIdx.x; l < W; l += blockDim.x)
            if (v[l]) { atomicMin(s_z, l); break; }
    }
    __syncthreads();
    const int z = *s_z;
    for (int l = threadIdx.x; l < W; l += blockDim.x) {
        uint64_t x = v[l];
        if (neg) x = l < z ? 0ull : (l == z ? (0ull - x) : ~x);
        mag32[2 * l] = (uint32_t)x;
        mag32[2 * l + 1] = (uint32_t)(x >> 32);
    }
    if (threadIdx.x == 0) *sgn = neg ? -1 : 1;
}

__global__ void __launch_bounds__(kLeafThreads)
k5_leaf(const uint64_t *__restrict__ A, const uint64_t *__restrict__ X, uint64_t *__restrict__ Y,
        int64_t s, int W, int WY) {
    extern __shared__ uint32_t sm[];
    uint32_t *am = sm, *xm = sm + 2 * W;
    __shared__ int s_za, s_zx, s_sa, s_sx;
    const int64_t pr = blockIdx.x / s, i = blockIdx.x % s;  // 0-based row
    const int W32 = 2 * W, ncol = 2 * W32 - 1;
    unsigned __int128 acc[kLeafCols];
#pragma unroll
    for (int c = 0; c < kLeafCols; ++c) acc[c] = 0;
    for (int64_t j = 0; j < s; ++j) {
        __syncthreads();
        load_signmag(A + (pr * (2 * s - 1) + i + j) * W, W, am, &s_za, &s_sa);
        load_signmag(X + (pr * s + j) * W, W, xm, &s_zx, &s_sx);
        __syncthreads();
        const bool neg = s_sa * s_sx < 0;
#pragma unroll
        for (int c = 0; c < kLeafCols; ++c) {
            const int col = threadIdx.x + c * kLeafThreads;
            if (col >= ncol) break;
            const int ulo = col - W32 + 1 > 0 ? col - W32 + 1 : 0;
            const int uhi = col < W32 - 1 ? col : W32 - 1;
            unsigned __int128 sum = 0;
            for (int u = ulo; u <= uhi; ++u) sum += (uint64_t)am[u] * xm[col - u];
            if (neg) acc[c] -= sum; else acc[c] += sum;
        }
    }
    __syncthreads();
    unsigned __int128 *cols = reinterpret_cast<unsigned __int128 *>(sm);
#pragma unroll
    for (int c = 0; c < kLeafCols; ++c) {
        const int col = threadIdx.x + c * kLeafThreads;
        if (col < ncol) cols[col] = acc[c];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t *y = Y + (pr * s + i) * WY;
        __int128 carry = 0;
        uint64_t lo_word = 0;
        for (int wd = 0; wd < 2 * WY; ++wd) {
            __int128 v = carry;
            if (wd < ncol) v += (__int128)cols[wd];
            const uint32_t word = (uint32_t)(uint64_t)v;
            carry = v >> 32;
            if (wd & 1) y[wd >> 1] = lo_word | ((uint64_t)word << 32);
            else lo_word = word;
        }
    }
}

// step 8: one warp per output entry of the parent level
__global__ void k5_merge(const uint64_t *__restrict__ Yc, uint64_t *__restrict__ Yp, int64_t cnt,
                         int64_t s, int64_t s2, int WY) {
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (wid >= cnt * s) return;
    const int64_t pr = wid / s, i = wid % s + 1;  // 1-based output index
    const int64_t k = (i + 1) / 2;               // p_k with y_{2k-1} = p_k - q_k, y_{2k} = p_k + r_k
    const uint64_t *pk = Yc + ((3 * pr + 0) * s2 + (k - 1)) * WY;
    const bool odd = i & 1;
    const uint64_t *other = Yc + ((3 * pr + (odd ? 1 : 2)) * s2 + (k - 1)) * WY;
    warp_addsub(Yp + (pr * s + (i - 1)) * WY, pk, other, WY, odd);
}

// two's complement (WY limbs) -> sign-magnitude (Ly limbs); one warp per row
__global__ void k5_final(const uint64_t *__restrict__ Y, int64_t n, int WY, int Ly,
                         uint64_t *__restrict__ y_mag, int8_t *__restrict__ y_sign) {
    const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (e >= n) return;
    const int lane = threadIdx.x & 31;
    const uint64_t *v = Y + e * WY;
    const bool neg = (int64_t)v[WY - 1] < 0;
    const int z = warp_lowest_nonzero(v, WY);
    for (int l = lane; l < Ly; l += 32) {
        uint64_t x = v[l];
        if (neg) x = l < z ? 0ull : (l == z ? (0ull - x) : ~x);
        y_mag[e * Ly + l] = x;
    }
    if (lane == 0) y_sign[e] = neg ? (int8_t)-1 : (z < WY ? (int8_t)1 : (int8_t)0);
}

int check(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "hk: %s launch error: %s\n", what, cudaGetErrorString(e));
        return HK_ECUDA;
    }
    return HK_OK;
}

unsigned warp_blocks(int64_t warps, int threads) {
    return (unsigned)((warps * 32 + threads - 1) / threads);
}

}  // namespace

int karatsuba_workspace_size(int64_t n, int32_t P, int32_t cutoff, size_t *bytes) {
    KLevels k;
    const int rc = kplan(n, P, cutoff, &k);
    if (rc) return rc;
    *bytes = k.total;
    return HK_OK;
}

int launch_karatsuba(int64_t n, int32_t P, int32_t cutoff, const uint64_t *a_mag,
                     const int8_t *a_sign, const uint64_t *x_mag, const int8_t *x_sign,
                     uint64_t *y_mag, int8_t *y_sign, void *ws, size_t ws_bytes, void *stream) {
    KLevels k;
    int rc = kplan(n, P, cutoff, &k);
    if (rc) return rc;
    if (ws_bytes < k.total) return HK_ENOMEM;
    if (4 * k.W - 1 > kLeafThreads * kLeafCols) return HK_EUNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    char *base = (char *)ws;
    auto Ap = [&](int d) { return (uint64_t *)(base + k.offA[d]); };
    auto Xp = [&](int d) { return (uint64_t *)(base + k.offX[d]); };
    auto Yp = [&](int d) { return (uint64_t *)(base + k.offY[d]); };
    const int T = 256;
    k5_to_twos<<<warp_blocks(2 * n - 1, T), T, 0, st>>>(a_mag, a_sign, 2 * n - 1, k.L, k.W, Ap(0));
    k5_to_twos<<<warp_blocks(n, T), T, 0, st>>>(x_mag, x_sign, n, k.L, k.W, Xp(0));
    if ((rc = check("k5_to_twos"))) return rc;
    for (int d = 0; d < k.D; ++d) {
        const int64_t per = 3 * (2 * k.s[d + 1] - 1) + 3 * k.s[d + 1];
        k5_split<<<warp_blocks(k.cnt[d] * per, T), T, 0, st>>>(Ap(d), Xp(d), Ap(d + 1), Xp(d + 1),
                                                            k.cnt[d], k.s[d], k.s[d + 1], k.W);
        if ((rc = check("k5_split"))) return rc;
    }
    const size_t leaf_smem = (size_t)(4 * k.W - 1) * 16 > (size_t)4 * k.W * 4
                                 ? (size_t)(4 * k.W - 1) * 16
                                 : (size_t)4 * k.W * 4;
    if (cudaFuncSetAttribute(k5_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)leaf_smem) != cudaSuccess)
        return HK_ECUDA;
    const int D = k.D;
    k5_leaf<<<(unsigned)(k.cnt[D] * k.s[D]), kLeafThreads, leaf_smem, st>>>(Ap(D), Xp(D), Yp(D),
                                                                            k.s[D], k.W, k.WY);
    if ((rc = check("k5_leaf"))) return rc;
    for (int d = D - 1; d >= 0; --d) {
        k5_merge<<<warp_blocks(k.cnt[d] * k.s[d], T), T, 0, st>>>(Yp(d + 1), Yp(d), k.cnt[d],
                                                                 k.s[d], k.s[d + 1], k.WY);
        if ((rc = check("k5_merge"))) return rc;
    }
    k5_final<<<warp_blocks(n, T), T, 0, st>>>(Yp(0), n, k.WY, k.Ly, y_mag, y_sign);
    return check("k5_final");
}

}  // namespace hk
