// hk_schoolbook.cu -- companion A6: the direct schoolbook matvec on limbs,
// y_i = sum_j a_{idx(i,j)} x_j, without any transform.
//
// Row i is one thread-block cluster of Q CTAs (Q = 1..8, chosen so the grid covers the SMs
// even for few rows); inside a CTA, S warp groups ("slices") take different j, and inside a
// slice thread t owns kCpt = 5 consecutive output columns c of the 32-bit-word product
// sum_u A32[u] X32[c - u].  Per j the slice stages a_{idx(i,j)} and x_j (zero-padded on both
// sides, so the column window needs no bounds checks) in shared memory; the thread slides a
// 5-word register window over X32 (one new shared load per u, A32[u] read once per u: two
// loads per five 32x32 products) and accumulates each product with a mad.lo.cc / madc.hi.cc /
// addc chain into a 96-bit column sum (|sum_u| < L32 2^64), which is then added to or
// subtracted from a 128-bit two's-complement column total with the sign product of the pair.
// Odd kCpt keeps the stride-5 window loads free of bank conflicts.
// Reduction: the slices' totals are summed in shared memory, then the cluster's CTAs add
// theirs into CTA 0 over distributed shared memory.  CTA 0's first warp resolves the carries:
// output word k gets s_k = sum_t word_t(col k - t) (t = 0..3, word 3 signed), split into
// lo + 2^32 hi and re-associated as t_k = lo_k + hi_(k-1) in [-1, 2^32 + 2], so every
// carry is in {-1, 0, 1}; a warp scan of the ternary carry-transfer functions gives each
// lane's carry-in.  Then two's complement -> sign-magnitude (lowest nonzero word by a warp
// min-reduction), canonical zero.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>

#include "hk_internal.h"

namespace hk {

namespace cg = cooperative_groups;

constexpr int kCpt = 5;         // output columns per thread (odd: conflict-free window loads)
constexpr int kXPad = 8;        // zero words in front of X32 (>= kCpt - 1)
constexpr int kSbMaxT = 512;    // threads per CTA (upper bound)

// (c2 : c01) += a x: one IMAD.WIDE with carry out and one IMAD.X (c01 is a 64-bit pair)
__device__ __forceinline__ void sb_mac(uint64_t &c01, uint32_t &c2, uint32_t a, uint32_t x) {
    asm("{\n\t.reg .u32 lo, hi;\n\tmov.b64 {lo, hi}, %0;\n\t"
        "mad.lo.cc.u32 lo, %2, %3, lo;\n\tmadc.hi.cc.u32 hi, %2, %3, hi;\n\taddc.u32 %1, %1, 0;\n\t"
        "mov.b64 %0, {lo, hi};\n\t}"
        : "+l"(c01), "+r"(c2) : "r"(a), "r"(x));
}
__device__ __forceinline__ void sb_add128(uint32_t (&t)[4], uint32_t c0, uint32_t c1, uint32_t c2,
                                          uint32_t c3) {
    asm("add.cc.u32 %0, %0, %4;\n\taddc.cc.u32 %1, %1, %5;\n\taddc.cc.u32 %2, %2, %6;\n\t"
        "addc.u32 %3, %3, %7;"
        : "+r"(t[0]), "+r"(t[1]), "+r"(t[2]), "+r"(t[3]) : "r"(c0), "r"(c1), "r"(c2), "r"(c3));
}
__device__ __forceinline__ void sb_sub128(uint32_t (&t)[4], uint32_t c0, uint32_t c1, uint32_t c2) {
    asm("sub.cc.u32 %0, %0, %4;\n\tsubc.cc.u32 %1, %1, %5;\n\tsubc.cc.u32 %2, %2, %6;\n\t"
        "subc.u32 %3, %3, 0;"
        : "+r"(t[0]), "+r"(t[1]), "+r"(t[2]), "+r"(t[3]) : "r"(c0), "r"(c1), "r"(c2));
}
// ternary carry-transfer functions {-1,0,1} -> {-1,0,1}, 2 bits per input (value + 1)
__device__ __forceinline__ int sb_tf_apply(int f, int c) { return ((f >> (2 * (c + 1))) & 3) - 1; }
__device__ __forceinline__ int sb_tf_compose(int g, int f) {  // g o f
    int h = 0;
#pragma unroll
    for (int c = -1; c <= 1; ++c) h |= (sb_tf_apply(g, sb_tf_apply(f, c)) + 1) << (2 * (c + 1));
    return h;
}
constexpr int kSbTfId = 0 | (1 << 2) | (2 << 4);

__device__ __forceinline__ int64_t sb_entry_index(int kind, int64_t i, int64_t j, int64_t n) {
    if (kind == HK_HANKEL) return i + j;
    if (kind == HK_TOEPLITZ) return (n - 1) - i + j;
    int64_t k = (i - j) % n;
    return k < 0 ? k + n : k;
}

// signed 64-bit sum of the output word k: word t of column k - t (t = 0..3; word 3 signed)
__device__ __forceinline__ int64_t sb_word_sum(const uint32_t *red, int k, int ncol) {
    int64_t s = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int c = k - t;
        if (c >= 0 && c < ncol) {
            const uint32_t w = red[4 * c + t];
            s += t == 3 ? (int64_t)(int32_t)w : (int64_t)w;
        }
    }
    return s;
}

// One j for the column group c0 .. c0 + kCpt - 1: its 96-bit column sums, added to or subtracted
// from the group's 128-bit totals.  Rounds of kCpt consecutive u keep the X window in registers:
// at u = u0 + r, column c0 + k needs X32[c0 + k - u0 - r] = xw[k - r + kCpt - 1] with
// xw[d] = X32[c0 - u0 - (kCpt - 1) + d].
__device__ __forceinline__ void sb_group(const uint32_t *A, const uint32_t *Xp, int c0, int L32, int s,
                                         uint32_t (&tot)[kCpt][4]) {
    const int ulo = c0 - (L32 - 1) > 0 ? c0 - (L32 - 1) : 0;
    const int uhi = c0 + kCpt - 1 < L32 - 1 ? c0 + kCpt - 1 : L32 - 1;
    uint64_t acc[kCpt];
    uint32_t top[kCpt];
#pragma unroll
    for (int k = 0; k < kCpt; ++k) acc[k] = 0ull, top[k] = 0u;
    constexpr int NW = 2 * kCpt - 1;
    uint32_t xw[NW];
    const uint32_t *xb = Xp + kXPad + c0;
    int u0 = ulo;
#pragma unroll
    for (int d = kCpt - 1; d < NW; ++d) xw[d] = xb[-u0 - (kCpt - 1) + d];
    for (; u0 + kCpt - 1 <= uhi; u0 += kCpt) {
#pragma unroll
        for (int d = 0; d < kCpt - 1; ++d) xw[d] = xb[-u0 - (kCpt - 1) + d];
#pragma unroll
        for (int r = 0; r < kCpt; ++r) {
            const uint32_t a = A[u0 + r];
#pragma unroll
            for (int k = 0; k < kCpt; ++k) sb_mac(acc[k], top[k], a, xw[k - r + kCpt - 1]);
        }
#pragma unroll
        for (int d = kCpt; d < NW; ++d) xw[d] = xw[d - kCpt];  // next round's upper part
        xw[kCpt - 1] = xb[-(u0 + kCpt)];
    }
    for (int u = u0; u <= uhi; ++u) {  // remainder: single steps, window from smem
        const uint32_t a = A[u];
#pragma unroll
        for (int k = 0; k < kCpt; ++k) sb_mac(acc[k], top[k], a, xb[k - u]);
    }
#pragma unroll
    for (int k = 0; k < kCpt; ++k) {
        const uint32_t l0 = (uint32_t)acc[k], l1 = (uint32_t)(acc[k] >> 32);
        if (s > 0) sb_add128(tot[k], l0, l1, top[k], 0u);
        else sb_sub128(tot[k], l0, l1, top[k]);
    }
}

// Threads of a slice (MIRROR, few columns): TC = ceil(NG / 2) for NG = ceil(ncol / kCpt) column
// groups; thread ct takes group ct and its mirror NG - 1 - ct, whose u ranges add up to ~L32 + kCpt
// for every thread (the column sums of a product are a tent over the columns), so no lane idles
// in a warp.  With many columns (!MIRROR) a warp's 32 consecutive groups have nearly equal u
// ranges and thread ct takes group ct only (TC = NG), which keeps the registers of the second
// group's totals free.
template <bool MIRROR>
__global__ void __launch_bounds__(kSbMaxT)
k6_schoolbook(int kind, int64_t m, int64_t n, int L, int Q, int S, int TC,
              const uint64_t *__restrict__ a_mag, const int8_t *__restrict__ a_sign,
              const uint64_t *__restrict__ x_mag, const int8_t *__restrict__ x_sign,
              uint64_t *__restrict__ y_mag, int8_t *__restrict__ y_sign) {
    extern __shared__ __align__(16) uint32_t sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int L32 = 2 * L, ncol = 2 * L32 - 1, XW = 2 * L32 + 2 * kXPad;
    const int NG = (ncol + kCpt - 1) / kCpt;
    const int tid = threadIdx.x, T = blockDim.x;
    const int js = tid / TC, ct = tid % TC;
    const bool act = js < S;
    const int q = (int)cluster.block_rank();
    const int64_t i = blockIdx.x / Q;
    uint32_t *A = sm + js * (L32 + XW);  // this slice's a entry ...
    uint32_t *Xp = A + L32;              // ... and zero-padded x entry (X32[t] at Xp[kXPad + t])
    for (int e = tid; e < S * (L32 + XW); e += T) sm[e] = 0u;
    __syncthreads();

    const int g1 = ct, g2 = MIRROR ? NG - 1 - ct : ct;  // g2 == g1: no second group
    const bool grp = g1 < NG;
    uint32_t tot1[kCpt][4], tot2[kCpt][MIRROR ? 4 : 1];
#pragma unroll
    for (int k = 0; k < kCpt; ++k) {
#pragma unroll
        for (int w = 0; w < 4; ++w) tot1[k][w] = 0u;
#pragma unroll
        for (int w = 0; w < (MIRROR ? 4 : 1); ++w) tot2[k][w] = 0u;
    }

    const int64_t step = (int64_t)Q * S;
    for (int64_t jb = 0; jb < n; jb += step) {
        const int64_t j = jb + (int64_t)q * S + js;
        int s = 0;
        if (act && j < n) {
            const int64_t kidx = sb_entry_index(kind, i, j, n);
            s = (int)a_sign[kidx] * (int)x_sign[j];
            if (s != 0) {
                const uint32_t *a32 = reinterpret_cast<const uint32_t *>(a_mag + kidx * L);
                const uint32_t *x32 = reinterpret_cast<const uint32_t *>(x_mag + j * L);
                for (int u = ct; u < L32; u += TC) {
                    A[u] = __ldg(a32 + u);
                    Xp[kXPad + u] = __ldg(x32 + u);
                }
            }
        }
        __syncthreads();
        if (s != 0 && grp) {
            sb_group(A, Xp, g1 * kCpt, L32, s, tot1);
            if constexpr (MIRROR)
                if (g2 > g1) sb_group(A, Xp, g2 * kCpt, L32, s, tot2);
        }
        __syncthreads();  // the staging area is rewritten next round
    }

    // ---- every slice's totals to its own region part[js][ncol][4] (reuses the staging area), then
    // all threads sum the slices column by column into red[ncol][4] (after the S regions)
    uint32_t *part = sm, *red = sm + (size_t)S * ncol * 4;
    if (act && grp) {
#pragma unroll
        for (int k = 0; k < kCpt; ++k) {
            int c = g1 * kCpt + k;
            if (c < ncol) {
                uint32_t *d = part + ((size_t)js * ncol + c) * 4;
                d[0] = tot1[k][0]; d[1] = tot1[k][1]; d[2] = tot1[k][2]; d[3] = tot1[k][3];
            }
            if constexpr (MIRROR) {
                c = g2 * kCpt + k;
                if (g2 > g1 && c < ncol) {
                    uint32_t *d = part + ((size_t)js * ncol + c) * 4;
                    d[0] = tot2[k][0]; d[1] = tot2[k][1]; d[2] = tot2[k][2]; d[3] = tot2[k][3];
                }
            }
        }
    }
    __syncthreads();
    for (int c = tid; c < ncol; c += T) {
        uint32_t v[4] = {0u, 0u, 0u, 0u};
        for (int r = 0; r < S; ++r) {
            const uint32_t *d = part + ((size_t)r * ncol + c) * 4;
            sb_add128(v, d[0], d[1], d[2], d[3]);
        }
        red[4 * c] = v[0]; red[4 * c + 1] = v[1]; red[4 * c + 2] = v[2]; red[4 * c + 3] = v[3];
    }
    // ---- CTA 0 of the cluster pulls the other CTAs' column sums (distributed shared memory);
    // the second cluster barrier keeps them resident until it has read them
    if (Q > 1) {
        cluster.sync();
        if (q == 0) {
            for (int c = tid; c < ncol; c += T) {
                uint32_t v[4] = {red[4 * c], red[4 * c + 1], red[4 * c + 2], red[4 * c + 3]};
                for (int r = 1; r < Q; ++r) {
                    const uint32_t *o = cluster.map_shared_rank(red, r) + 4 * c;
                    sb_add128(v, o[0], o[1], o[2], o[3]);
                }
                red[4 * c] = v[0]; red[4 * c + 1] = v[1]; red[4 * c + 2] = v[2]; red[4 * c + 3] = v[3];
            }
        }
        cluster.sync();
        if (q != 0) return;
    } else {
        __syncthreads();
    }
    if (tid >= 32) return;

    // ---- carries (one warp): output words k in [0, K), K = 2 Ly; lane owns [lane W, lane W + W)
    const int Ly = 2 * L + 1, K = 2 * Ly, lane = tid;
    const int W = (K + 31) / 32, k0 = lane * W, k1 = k0 + W < K ? k0 + W : K;
    int F = kSbTfId;
    int64_t hprev = k0 > 0 ? (sb_word_sum(red, k0 - 1, ncol) >> 32) : 0;
    for (int k = k0; k < k1; ++k) {
        const int64_t sk = sb_word_sum(red, k, ncol);
        const int64_t tk = (int64_t)(uint32_t)sk + hprev;  // in [-1, 2^32 + 2]
        hprev = sk >> 32;
        int f = 0;
#pragma unroll
        for (int c = -1; c <= 1; ++c) {
            const int64_t v = tk + c;
            const int co = v < 0 ? -1 : (v >= (int64_t(1) << 32) ? 1 : 0);
            f |= (co + 1) << (2 * (c + 1));
        }
        F = sb_tf_compose(f, F);
    }
    int incl = F;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl = sb_tf_compose(incl, o);
    }
    const int prev = __shfl_up_sync(0xffffffffu, incl, 1);
    int carry = lane > 0 ? sb_tf_apply(prev, 0) : 0;
    uint32_t *yw = reinterpret_cast<uint32_t *>(y_mag + i * Ly);
    hprev = k0 > 0 ? (sb_word_sum(red, k0 - 1, ncol) >> 32) : 0;
    int zloc = INT_MAX;
    for (int k = k0; k < k1; ++k) {
        const int64_t sk = sb_word_sum(red, k, ncol);
        const int64_t v = (int64_t)(uint32_t)sk + hprev + carry;
        hprev = sk >> 32;
        carry = v < 0 ? -1 : (v >= (int64_t(1) << 32) ? 1 : 0);
        const uint32_t wv = (uint32_t)v;
        yw[k] = wv;
        if (wv != 0u && zloc == INT_MAX) zloc = k;
    }
    // two's complement -> sign-magnitude: -Y = ~Y + 1, the + 1 stopping at the lowest nonzero word
    const int zmin = __reduce_min_sync(0xffffffffu, zloc);
    const bool neg = (int)__shfl_sync(0xffffffffu, (K - 1 >= k0 && K - 1 < k1) ? (yw[K - 1] >> 31) : 0u,
                                      (K - 1) / W) != 0;
    __syncwarp();
    if (neg) {
        for (int k = k0; k < k1; ++k) {
            if (k == zmin) yw[k] = 0u - yw[k];
            else if (k > zmin) yw[k] = ~yw[k];
        }
    }
    if (lane == 0) y_sign[i] = neg ? (int8_t)-1 : (zmin < K ? (int8_t)1 : (int8_t)0);
}

int launch_schoolbook(int kind, int64_t m, int64_t n, int32_t P, const uint64_t *a_mag,
                      const int8_t *a_sign, const uint64_t *x_mag, const int8_t *x_sign,
                      uint64_t *y_mag, int8_t *y_sign, void *stream) {
    const int L = (P + 63) / 64, L32 = 2 * L, ncol = 2 * L32 - 1;
    const int NG = (ncol + kCpt - 1) / kCpt;
    const bool mirror = NG <= 128;  // the tent's imbalance within a warp matters for few groups
    const int TC = mirror ? (NG + 1) / 2 : ((NG + 31) / 32) * 32;
    if (TC > kSbMaxT) return HK_EUNSUPPORTED;  // > 2560 columns: P > 40,960 bits
    static int nsm = 0;  // SM count of the device (queried once; one device per process)
    if (nsm == 0) {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            nsm = v;
        else
            return HK_ECUDA;
    }
    const int XW = 2 * L32 + 2 * kXPad;
    auto smem_of = [&](int s) {
        const size_t st = (size_t)s * (L32 + XW) * 4, rd = (size_t)(s + 1) * ncol * 16;
        return st > rd ? st : rd;
    };
    // slices S (j per CTA round) and cluster size Q (CTAs per row): the fewest j rounds x CTA
    // waves, with the CTAs resident at once counted from the thread count (1 or 2 per SM)
    int bestS = 1, bestQ = 1;
    double best = 1e300;
    const int smax = kSbMaxT / TC;
    for (int Q = 1; Q <= 8; Q *= 2) {
        for (int S = 1; S <= smax; ++S) {
            if ((int64_t)Q * S > n && !(Q == 1 && S == 1)) continue;
            if (smem_of(S) > 200 * 1024) continue;
            const int64_t rounds = (n + (int64_t)Q * S - 1) / ((int64_t)Q * S);
            const int thr = S * TC < 32 ? 32 : S * TC;
            // resident CTAs per SM from the register file (ptxas: 120 / 82 registers per thread)
            int per_sm = 65536 / ((mirror ? 120 : 82) * ((thr + 31) / 32 * 32));
            per_sm = per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm);
            const int64_t waves = (m * Q + (int64_t)nsm * per_sm - 1) / ((int64_t)nsm * per_sm);
            // a round's duration grows with the threads sharing an SM once they fill its issue slots
            const double fill = (double)(thr * per_sm) / 512.0;
            const double cost = (double)rounds * (double)waves * (fill > 1.0 ? fill : 1.0) + 0.02 * Q;
            if (cost < best - 1e-9) best = cost, bestS = S, bestQ = Q;
        }
    }
    const int S = bestS, Q = bestQ;
    if (smem_of(S) > 200 * 1024) return HK_EUNSUPPORTED;
    const size_t smem = smem_of(S);
    static size_t smem_set = 0;  // the kernel's dynamic-smem limit only ever grows
    if (smem > 48 * 1024 && smem > smem_set) {
        if (cudaFuncSetAttribute(k6_schoolbook<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024) != cudaSuccess ||
            cudaFuncSetAttribute(k6_schoolbook<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024) != cudaSuccess)
            return HK_ECUDA;
        smem_set = 200 * 1024;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(m * Q));
    cfg.blockDim = dim3((unsigned)(TC * S < 32 ? 32 : TC * S));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)Q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = mirror ? cudaLaunchKernelEx(&cfg, k6_schoolbook<true>, kind, m, n, L, Q, S, TC, a_mag,
                                                a_sign, x_mag, x_sign, y_mag, y_sign)
                           : cudaLaunchKernelEx(&cfg, k6_schoolbook<false>, kind, m, n, L, Q, S, TC, a_mag,
                                                a_sign, x_mag, x_sign, y_mag, y_sign);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "hk: schoolbook launch error: %s\n", cudaGetErrorString(e));
        return HK_ECUDA;
    }
    return HK_OK;
}

}  // namespace hk
