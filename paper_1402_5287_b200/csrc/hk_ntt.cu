// hk_ntt.cu -- the hot path: exact multiprecision Hankel/Toeplitz/circulant matvec as a 2-D
// multi-prime NTT convolution.
//
//   K0 k0_init           twiddle tables + workspace header (once per plan)
//   K1 k1_slice_rowntt   A1 limb slicing + validation, A2 slice-dimension forward NTT (N2),
//                        a and x tiles in one launch
//   K2 k2_column         A2 matrix-index forward NTTs (N1) of X^ and A^ columns, A3 pointwise
//                        Montgomery product, inverse matrix-index NTT, keep the n needed rows
//   K3a k3a_row_intt     A3 inverse slice-dimension NTT per output row
//   K3b k3b_carry    A3 Garner CRT -> signed coefficients, A4 carry propagation and
//                        sign-magnitude output
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <cstdlib>

#include "hk_internal.h"
#include "hk_modarith.cuh"
#include "hk_k2.cuh"

namespace hk {

// ------------------------------------------------------------------------------------------
// K0: twiddle tables.  Per prime: [N2 table | N1 table]; entry h + j of a table of length N
// holds omega_{2h}^j and its Shoup quotient floor(W 2^32 / p) (forward roots only).
__device__ uint32_t mulmod_slow(uint32_t a, uint32_t b, uint32_t p) {
    return (uint32_t)(((uint64_t)a * b) % p);
}
__device__ uint32_t powmod_slow(uint32_t g, uint64_t e, uint32_t p) {
    uint32_t r = 1 % p, b = g % p;
    while (e) {
        if (e & 1) r = mulmod_slow(r, b, p);
        b = mulmod_slow(b, b, p);
        e >>= 1;
    }
    return r;
}

__global__ void k0_init(Params prm, uint2 *tw, uint32_t g0, uint32_t g1, uint32_t g2, uint32_t g3,
                        uint32_t g4) {
    const uint32_t gens[kNumPrimes] = {g0, g1, g2, g3, g4};
    const int N2 = prm.N2, N1 = prm.N1;
    const int per = N2 + N1;
    const int64_t total = (int64_t)kNumPrimes * per;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int kp = (int)(idx / per);
        int e = (int)(idx % per);
        if (e >= N2) e -= N2;  // [N2 table | N1 table], both forward
        const uint32_t p = prm.pc[kp].p;
        uint32_t W = 1;
        if (e > 0) {
            const int h = 1 << (31 - __clz(e));
            const int j = e - h;
            const uint32_t root = powmod_slow(gens[kp], (uint64_t)(p - 1) / (uint64_t)(2 * h), p);
            W = powmod_slow(root, (uint64_t)j, p);
        }
        tw[idx] = make_uint2(W, (uint32_t)(((uint64_t)W << 32) / p));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        prm.hdr->magic = kWsMagic;
        prm.hdr->hash = prm.hash;
        prm.hdr->status = HK_OK;
        prm.hdr->a_ready = 0;
    }
}

// ------------------------------------------------------------------------------------------
// K1: slice + residues + slice-dimension forward NTT.  One CTA = 16 entries (rows) of a or x.
template <int LOGN2>
constexpr int k1_row_stride() {  // = 4 (mod 32): transposed [row][sigma] tiles are conflict-free
    return (padded_len(1 << LOGN2) + 31) / 32 * 32 + 4;
}

// K1 v2: a CTA owns kK1Rows entries (a and x tiles in one launch).  Each thread extracts the
// w-bit digits of its top-pass group once (registers), then for every prime: residues -> top
// DIF pass (radix 2^5, upper half zero) in registers -> smem -> remaining passes -> transposed
// write of [prime][sigma][row] (kK1Rows consecutive rows per sigma = one 32-byte sector).
constexpr int kK1Rows = 8;
template <int LOGN2>
constexpr int k1_threads() {
    return kK1Rows * ((1 << LOGN2) / 32 > 8 ? (1 << LOGN2) / 32 : 8);
}

template <int LOGN2>
__global__ void __launch_bounds__(k1_threads<LOGN2>(), 3) k1_slice_rowntt(Params prm, int tiles_a) {
    constexpr int N2 = 1 << LOGN2;
    constexpr int RS = k1_row_stride<LOGN2>();
    constexpr int T = k1_threads<LOGN2>();
    constexpr int R1 = 5, G1 = 32, H1 = 16;  // top pass: 32 points, upper 16 are zero padding
    constexpr int S1 = N2 / G1;              // top-pass groups per row
    constexpr int TPR = T / kK1Rows;         // threads per row (>= S1)
    static_assert(LOGN2 >= 5 && TPR >= S1, "K1 tiling");
    extern __shared__ uint32_t sm[];
    __shared__ int8_t s_sign[kK1Rows];
    __shared__ int s_nz[kK1Rows];

    const int tid = threadIdx.x;
    if (prm.hdr->magic != kWsMagic || prm.hdr->hash != prm.hash) {
        if (tid == 0 && blockIdx.x == 0) atomicMin(&prm.hdr->status, (int)HK_EINVAL);
        return;
    }
    const int bt = (int)blockIdx.x + prm.tile0;
    const bool is_x = bt >= tiles_a;
    if (prm.need_a_ready && prm.hdr->a_ready != 1) {
        if (tid == 0) atomicMin(&prm.hdr->status, (int)HK_EINVAL);
        return;
    }
    const int tile = is_x ? bt - tiles_a : bt;
    const uint64_t *mag = is_x ? prm.x_mag : prm.a_mag;
    const int8_t *sgn = is_x ? prm.x_sign : prm.a_sign;
    const int64_t count = is_x ? prm.n : prm.a_count;
    uint32_t *out = is_x ? prm.Xhat : prm.Ahat;
    const int64_t ld = is_x ? prm.ldX : prm.ldA;
    const bool rev = is_x && prm.x_reversed;
    const int64_t r0 = (int64_t)tile * kK1Rows;
    const int L = prm.L, w = prm.w, Ls = prm.Ls;

    // ---- stage the tile's limbs (kK1Rows consecutive entries = one contiguous block) in smem
    uint64_t *slimb = reinterpret_cast<uint64_t *>(sm + kK1Rows * RS);
    {
        const int64_t nrows = count - r0 < kK1Rows ? count - r0 : kK1Rows;
        const int64_t bytes = nrows * L * 8;
        const char *g = reinterpret_cast<const char *>(mag + r0 * L);
        char *d = reinterpret_cast<char *>(slimb);
        for (int64_t c = tid; c < bytes / 16; c += T) cp_async16(d + 16 * c, g + 16 * c);
        if ((bytes & 15) && tid == 0) cp_async8(d + (bytes & ~int64_t(15)), g + (bytes & ~int64_t(15)));
        cp_async_wait_all();
    }
    // ---- validation (A1): bits >= P zero, sign in {-1,0,1}, sign == 0 <=> magnitude == 0
    const int rem = prm.P - 64 * (L - 1);
    const uint64_t topmask = rem >= 64 ? ~0ull : ((1ull << rem) - 1);
    if (tid < kK1Rows) s_nz[tid] = 0;
    __syncthreads();
    bool bad = false;
    for (int idx = tid; idx < kK1Rows * L; idx += T) {
        const int r = idx / L, u = idx - (idx / L) * L;
        const int64_t row = r0 + r;
        if (row >= count) continue;
        const uint64_t v = slimb[idx];
        if (v) s_nz[r] = 1;
        if (u == L - 1 && (v & ~topmask)) bad = true;
    }
    __syncthreads();
    if (tid < kK1Rows) {
        const int64_t row = r0 + tid;
        int sg = 0;
        if (row < count) {
            sg = sgn[row];
            if (sg < -1 || sg > 1 || ((sg == 0) != (s_nz[tid] == 0))) bad = true;
        }
        s_sign[tid] = (int8_t)sg;
    }
    if (bad) atomicMin(&prm.hdr->status, (int)HK_ERANGE);
    __syncthreads();

    // ---- A1: this thread's digits t = j0 + m S1 (m < 16), extracted once for all primes
    const int r = tid / TPR, j0 = tid % TPR;
    const int sg = s_sign[r];
    const bool act = j0 < S1;
    uint32_t dlo[H1], dhi[H1], dtop = 0;
#pragma unroll
    for (int m = 0; m < H1; ++m) {
        const int t = j0 + m * S1;
        uint64_t lo = 0;
        if (act && sg != 0 && t < Ls) {
            const int o = w * t, q = o >> 6, sh = o & 63;
            const uint64_t *rp = slimb + r * L;
            const uint64_t l0 = rp[q];
            const uint64_t l1 = (q + 1 < L) ? rp[q + 1] : 0ull;
            lo = sh ? ((l0 >> sh) | (l1 << (64 - sh))) : l0;
            if (w < 64) lo &= (1ull << w) - 1;
            else if (w == 65) dtop |= (uint32_t)((l1 >> sh) & 1ull) << m;
        }
        dlo[m] = (uint32_t)lo;
        dhi[m] = (uint32_t)(lo >> 32);
    }

    for (int kp = 0; kp < kNumPrimes; ++kp) {
        const uint32_t p = prm.pc[kp].p;
        const uint32_t *F = is_x ? prm.pc[kp].fx : prm.pc[kp].fa;
        const uint32_t *Fq = is_x ? prm.pc[kp].fx_q : prm.pc[kp].fa_q;
        // this prime's N2 twiddle table -> smem (the limb staging area is free after extraction)
        uint2 *tw = reinterpret_cast<uint2 *>(slimb);
        __syncthreads();
        {
            const uint4 *src = reinterpret_cast<const uint4 *>(prm.tw + (size_t)kp * (prm.N2 + prm.N1));
            for (int i = tid; i < N2 / 2; i += T) reinterpret_cast<uint4 *>(tw)[i] = src[i];
        }
        __syncthreads();
        if (act) {
            uint32_t v[G1];
#pragma unroll
            for (int m = 0; m < H1; ++m) {
                // residue of the signed digit: (lo32 F0 + hi32 F1 + top F2) mod p, negated if sign < 0
                uint32_t x0 = red1(shoup(dlo[m], F[0], Fq[0], p), p);
                uint32_t x1 = red1(shoup(dhi[m], F[1], Fq[1], p), p);
                uint32_t res = addm(x0, x1, p);
                if ((dtop >> m) & 1u) res = addm(res, F[2], p);
                if (sg < 0) res = subm(0u, res, p);
                v[m] = res;
            }
            // top stage (h = N2/2) with a zero upper half: (u, 0) -> (u, u W)
#pragma unroll
            for (int m = 0; m < H1; ++m) {
                const uint2 wv = TwShared::ld(tw, S1 * H1 + j0 + S1 * m);
                v[m + H1] = red1(shoup(v[m], wv.x, wv.y, p), p);
            }
#pragma unroll
            for (int l = R1 - 2; l >= 0; --l) {
                const int half = 1 << l;
#pragma unroll
                for (int m = 0; m < G1; ++m) {
                    if (m & half) continue;
                    const uint2 wv = TwShared::ld(tw, S1 * half + j0 + S1 * (m & (half - 1)));
                    gs_bfly(v[m], v[m + half], wv, p);
                }
            }
#pragma unroll
            for (int m = 0; m < G1; ++m) sm[r * RS + pad(j0 + m * S1)] = v[m];
        }
        __syncthreads();
        constexpr int REM = LOGN2 - R1;          // stages left after the top pass
        constexpr int RB = REM < 5 ? REM : 5;    // bottom pass (S = 1) radix
        if constexpr (REM > RB)
            dif_pass<TwShared, LOGN2, REM - RB, (1 << RB), false>(sm, kK1Rows, RS, tw, p, tid, T);
        // ---- bottom pass in registers, stored straight to [prime][sigma][row]; lanes cover
        // 8 rows x 4 groups so every store instruction writes full 32-byte row segments
        // (x rows reversed: matrix index n-1-row)
        constexpr int GB = 1 << RB, NGR = N2 / GB;
        for (int gi = tid; gi < kK1Rows * NGR; gi += T) {
            const int rr = gi % kK1Rows, g = gi / kK1Rows;
            uint32_t v[GB];
#pragma unroll
            for (int m = 0; m < GB; ++m) v[m] = sm[rr * RS + pad(g * GB + m)];
            dif_bottom_regs<TwShared, RB>(v, tw, p);
            const int64_t orow = r0 + rr;
            if (orow < count) {
                const int64_t pos = rev ? (count - 1 - orow) : orow;
                uint32_t *o = out + ((int64_t)kp * N2 + (int64_t)g * GB) * ld + pos;
#pragma unroll
                for (int m = 0; m < GB; ++m) o[(int64_t)m * ld] = v[m];
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// K3a: for a tile of k3_rows() output rows and all 5 primes: inverse slice-dimension NTT (DIT with
// forward roots, slice index negated), then Garner CRT (balanced mixed radix) of every
// coefficient C_s, |C_s| < M/2 < 2^155, written as five 32-bit two's-complement words
// Ycoef[(row * 5 + word) * ldS + s] (word planes: coalesced stores here and loads in K3b).
template <int LOGN2>
constexpr int k3_rows() { return LOGN2 >= 11 ? 2 : 4; }  // 5 x rows x N2 words in smem
constexpr int kK3aThreads = 320;  // 5 primes x 4 rows x 32 groups = 2 groups per thread

// Garner CRT with standard mixed-radix digits u_k in [0, p_k):
//   C' = u0 + p0 (u1 + p1 (u2 + p2 (u3 + p3 u4)))  in [0, M),  M = p0 p1 p2 p3 p4 < 2^155,
// evaluated in 32-bit words; the symmetric value is C' - M when C' > (M-1)/2, which holds iff the
// digit vector (u4..u0) exceeds ((p4-1)/2 .. (p0-1)/2) lexicographically.  Output: C as five
// 32-bit two's-complement words (bit 159 = sign; |C| < M/2 < 2^154).
HK_DEV void garner(const uint32_t r[kNumPrimes], const Params &prm, uint32_t (&cw)[kNumPrimes]) {
    uint32_t u[kNumPrimes];
#pragma unroll
    for (int k = 0; k < kNumPrimes; ++k) {
        const uint32_t p = prm.pc[k].p;
        uint32_t t = r[k];
#pragma unroll
        for (int j = 0; j < k; ++j) {
            t = subm(t, red1(u[j], p), p);  // u_j < p_j < 2 p_k
            t = red1(shoup(t, prm.gc.inv[j][k], prm.gc.inv_q[j][k], p), p);
        }
        u[k] = t;
    }
    uint32_t a0, a1, a2, a3, a4;
    uint64_t t = (uint64_t)u[4] * prm.pc[3].p + u[3];
    a0 = (uint32_t)t; a1 = (uint32_t)(t >> 32);
    t = (uint64_t)a0 * prm.pc[2].p + u[2]; a0 = (uint32_t)t;
    t = (uint64_t)a1 * prm.pc[2].p + (t >> 32); a1 = (uint32_t)t; a2 = (uint32_t)(t >> 32);
    t = (uint64_t)a0 * prm.pc[1].p + u[1]; a0 = (uint32_t)t;
    t = (uint64_t)a1 * prm.pc[1].p + (t >> 32); a1 = (uint32_t)t;
    t = (uint64_t)a2 * prm.pc[1].p + (t >> 32); a2 = (uint32_t)t; a3 = (uint32_t)(t >> 32);
    t = (uint64_t)a0 * prm.pc[0].p + u[0]; a0 = (uint32_t)t;
    t = (uint64_t)a1 * prm.pc[0].p + (t >> 32); a1 = (uint32_t)t;
    t = (uint64_t)a2 * prm.pc[0].p + (t >> 32); a2 = (uint32_t)t;
    t = (uint64_t)a3 * prm.pc[0].p + (t >> 32); a3 = (uint32_t)t; a4 = (uint32_t)(t >> 32);
    // sign: lexicographic (u4, u3, u2, u1, u0) > (h4, h3, h2, h1, h0)
    bool neg = false, eq = true;
#pragma unroll
    for (int k = kNumPrimes - 1; k >= 0; --k) {
        const uint32_t h = prm.gc.half[k];
        neg = neg || (eq && u[k] > h);
        eq = eq && u[k] == h;
    }
    if (neg) {  // C = C' - M (160-bit)
        const uint64_t lo = ((uint64_t)a1 << 32 | a0), mlo = ((uint64_t)prm.gc.M[1] << 32 | prm.gc.M[0]);
        const uint64_t mid = ((uint64_t)a3 << 32 | a2), mmid = ((uint64_t)prm.gc.M[3] << 32 | prm.gc.M[2]);
        const uint64_t rlo = lo - mlo;
        const uint64_t b1 = lo < mlo;
        const uint64_t rmid = mid - mmid - b1;
        const uint32_t b2 = (mid < mmid) | ((mid == mmid) & (uint32_t)b1);
        a4 = a4 - prm.gc.M[4] - b2;
        a0 = (uint32_t)rlo; a1 = (uint32_t)(rlo >> 32);
        a2 = (uint32_t)rmid; a3 = (uint32_t)(rmid >> 32);
    }
    cw[0] = a0; cw[1] = a1; cw[2] = a2; cw[3] = a3; cw[4] = a4;
}

template <int LOGN2, int R, int S>
HK_DEV void k3_dit_pass_all(uint32_t *sm, const Params &prm) {
    constexpr int N = 1 << LOGN2, G = 1 << R, NG = N / G;
    constexpr int RS = k1_row_stride<LOGN2>();
    constexpr int total = kNumPrimes * k3_rows<LOGN2>() * NG;
    for (int gi = threadIdx.x; gi < total; gi += kK3aThreads) {
        const int b = gi / NG, g = gi % NG;  // b = kp * k3_rows<LOGN2>() + row
        const int kp = b / k3_rows<LOGN2>();
        const uint32_t p = prm.pc[kp].p;
        const uint2 *tw = prm.tw + (size_t)kp * (prm.N2 + prm.N1);
        const int j0 = g % S;
        const int B = (g / S) * (S * G);
        uint32_t *base = sm + b * RS;
        uint32_t v[G];
#pragma unroll
        for (int m = 0; m < G; ++m) v[m] = base[pad(B + j0 + m * S)];
#pragma unroll
        for (int l = 0; l < R; ++l) {
            const int half = 1 << l;
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & half) continue;
                if (S == 1 && (m & (half - 1)) == 0) bfly1(v[m], v[m + half], p);  // twiddle 1
                else ct_bfly(v[m], v[m + half], TwGlobal::ld(tw, S * half + j0 + S * (m & (half - 1))), p);
            }
        }
#pragma unroll
        for (int m = 0; m < G; ++m) base[pad(B + j0 + m * S)] = v[m];
    }
    __syncthreads();
}
template <int LOGN2, int LO>
struct K3DitPasses {
    static HK_DEV void run(uint32_t *sm, const Params &prm) {
        if constexpr (LO < LOGN2) {
            constexpr int R = (LOGN2 - LO) < 5 ? (LOGN2 - LO) : 5;
            k3_dit_pass_all<LOGN2, R, (1 << LO)>(sm, prm);
            K3DitPasses<LOGN2, LO + R>::run(sm, prm);
        }
    }
};

template <int LOGN2>
__global__ void __launch_bounds__(kK3aThreads, 2) k3a_row_intt_crt(Params prm) {
    constexpr int N2 = 1 << LOGN2;
    constexpr int RS = k1_row_stride<LOGN2>();
    extern __shared__ uint32_t sm[];  // [prime][row][RS]
    const int tid = threadIdx.x;
    const int64_t r0 = prm.row0 + (int64_t)blockIdx.x * k3_rows<LOGN2>();
    const int64_t m = prm.m;
    for (int idx = tid; idx < kNumPrimes * N2 * k3_rows<LOGN2>(); idx += kK3aThreads) {
        const int r = idx % k3_rows<LOGN2>(), cs = idx / k3_rows<LOGN2>();  // cs = kp * N2 + sigma
        const int64_t row = r0 + r;
        const int kp = cs / N2, sigma = cs % N2;
        uint32_t *dst = sm + (kp * k3_rows<LOGN2>() + r) * RS + pad(sigma);
        if (row < m) cp_async4(dst, prm.Yhat + (int64_t)cs * prm.ldY + row);
        else *dst = 0u;
    }
    cp_async_wait_all();
    __syncthreads();
    K3DitPasses<LOGN2, 0>::run(sm, prm);
    const int S2 = prm.S2;
    for (int idx = tid; idx < k3_rows<LOGN2>() * S2; idx += kK3aThreads) {
        const int r = idx / S2, t = idx - (idx / S2) * S2;
        const int64_t row = r0 + r;
        if (row >= m) continue;
        uint32_t res[kNumPrimes];
        const int pos = pad((N2 - t) & (N2 - 1));  // slice index negated (forward-root DIT)
#pragma unroll
        for (int kp = 0; kp < kNumPrimes; ++kp) res[kp] = sm[(kp * k3_rows<LOGN2>() + r) * RS + pos];
        uint32_t cw[kNumPrimes];
        garner(res, prm, cw);
        uint32_t *dst = prm.Yres + row * kNumPrimes * prm.ldS + t;
#pragma unroll
        for (int k = 0; k < kNumPrimes; ++k) dst[k * prm.ldS] = cw[k];  // bit 159 = sign
    }
}

// ------------------------------------------------------------------------------------------
// K3b: Y = sum_s C_s 2^(w s) mod 2^(64 Ly), carry propagation by a block scan of
// carry-transfer functions, two's complement -> sign-magnitude.
// carry-transfer function {-1,0,1} -> {-1,0,1}, packed 2 bits per input (value + 1)
HK_DEV int tf_apply(int f, int c) { return ((f >> (2 * (c + 1))) & 3) - 1; }
HK_DEV int tf_compose(int g, int f) {  // g o f
    int h = 0;
#pragma unroll
    for (int c = -1; c <= 1; ++c) h |= (tf_apply(g, tf_apply(f, c)) + 1) << (2 * (c + 1));
    return h;
}
constexpr int kTfId = (0) | (1 << 2) | (2 << 4);

// One CTA per output row.  Coefficient s (160-bit two's complement C_s, w in {64, 65}) sits at
// limb q(s) = floor(w s / 64), bit sh = w s mod 64; its shifted value C_s 2^sh spans the four
// words S_0..S_3 (sign-extended to 256 bits) plus a -1 borrow into limb q + 4 when C_s < 0.
// Because q is injective for w >= 64, word d of every coefficient lands in its own slot
// P_d[q(s) + d]; limb l's sum is P_0[l] + P_1[l] + P_2[l] + P_3[l] - borrow[l].
template <int CHUNK>  // limbs per thread = ceil(Ly / kK3Threads)
__global__ void __launch_bounds__(kK3Threads) k3b_carry(Params prm) {
    extern __shared__ uint64_t sP[];  // [4][Ly] words, then borrow bytes [Ly]
    __shared__ uint8_t s_ecarry[kK3Threads];
    __shared__ int s_wtot[kK3Threads / 32];
    __shared__ int s_wcarry[kK3Threads / 32];
    __shared__ int s_neg, s_zmin;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t row = prm.row0 + blockIdx.x;
    const int S2 = prm.S2, Ly = prm.Ly, w = prm.w;
    uint8_t *sB = reinterpret_cast<uint8_t *>(sP + 4 * Ly);
    {  // zero the slot arrays (positions without a coefficient stay 0)
        uint4 *z = reinterpret_cast<uint4 *>(sP);
        const int n16 = (4 * Ly * 8 + Ly + 15) / 16;
        for (int i = tid; i < n16; i += kK3Threads) z[i] = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) { s_neg = 0; s_zmin = INT_MAX; }
    __syncthreads();
    const uint32_t *src = prm.Yres + row * kNumPrimes * prm.ldS;
    const int64_t ldS = prm.ldS;
    for (int s = tid; s < S2; s += kK3Threads) {
        const uint32_t w0 = __ldcs(src + s), w1 = __ldcs(src + ldS + s), w2 = __ldcs(src + 2 * ldS + s),
                       w3 = __ldcs(src + 3 * ldS + s), w4 = __ldcs(src + 4 * ldS + s);
        const uint64_t C0 = (uint64_t)w0 | ((uint64_t)w1 << 32);
        const uint64_t C1 = (uint64_t)w2 | ((uint64_t)w3 << 32);
        const uint64_t C2 = (uint64_t)(int64_t)(int32_t)w4;  // sign-extend bit 159
        const uint64_t C3 = (uint64_t)((int64_t)C2 >> 63);
        const int o = w * s, q = o >> 6, sh = o & 63;
        uint64_t S0 = C0, S1 = C1, S2w = C2, S3 = C3;
        if (sh) {
            S3 = (C3 << sh) | (C2 >> (64 - sh));
            S2w = (C2 << sh) | (C1 >> (64 - sh));
            S1 = (C1 << sh) | (C0 >> (64 - sh));
            S0 = C0 << sh;
        }
        if (q < Ly) sP[q] = S0;
        if (q + 1 < Ly) sP[Ly + q + 1] = S1;
        if (q + 2 < Ly) sP[2 * Ly + q + 2] = S2w;
        if (q + 3 < Ly) sP[3 * Ly + q + 3] = S3;
        if (C3 && q + 4 < Ly) sB[q + 4] = 1;
    }
    __syncthreads();

    const int l0 = tid * CHUNK;
    uint64_t u[CHUNK];
    int e[CHUNK];
#pragma unroll
    for (int c = 0; c < CHUNK; ++c) {
        const int l = l0 + c;
        uint64_t acc = 0;
        int hi = 0;
        if (l < Ly) {
            acc = sP[l];
            uint64_t t = sP[Ly + l];
            acc += t; hi += acc < t;
            t = sP[2 * Ly + l];
            acc += t; hi += acc < t;
            t = sP[3 * Ly + l];
            acc += t; hi += acc < t;
            const int bw = sB[l];
            hi -= bw & (acc == 0);
            acc -= bw;
        }
        u[c] = acc;
        e[c] = hi;  // carry into limb l+1, in [-1, 3]
    }
    s_ecarry[tid] = (uint8_t)(e[CHUNK - 1] + 1);
    __syncthreads();
    // u_l = w_l + e_{l-1} -> g_l in {-1,0,1}; transfer f_l(c) = g_l + [c=1, u_l=MAX] - [c=-1, u_l=0]
    // packed 2 bits per input c in {-1,0,1}: (f(-1)+1) | (f(0)+1) << 2 | (f(1)+1) << 4
    int F = kTfId;
    int fl[CHUNK];
    int ein = tid > 0 ? (int)s_ecarry[tid - 1] - 1 : 0;
#pragma unroll
    for (int c = 0; c < CHUNK; ++c) {
        const uint64_t wv = u[c];
        const uint64_t uv = wv + (uint64_t)(int64_t)ein;
        const int g = (ein > 0 && uv < wv) ? 1 : ((ein < 0 && uv > wv) ? -1 : 0);
        u[c] = uv;
        const int g1 = g + 1;
        const int f = (g1 - (uv == 0)) | (g1 << 2) | ((g1 + (uv == ~0ull)) << 4);
        fl[c] = f;
        F = tf_compose(f, F);
        ein = e[c];
    }
    // block scan of transfer functions (low limbs first)
    int incl = F;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int other = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl = tf_compose(incl, other);
    }
    if (lane == 31) s_wtot[warp] = incl;
    __syncthreads();
    if (tid == 0) {
        int c = 0;
        for (int wi = 0; wi < kK3Threads / 32; ++wi) {
            s_wcarry[wi] = c;
            c = tf_apply(s_wtot[wi], c);
        }
    }
    __syncthreads();
    const int prev = __shfl_up_sync(0xffffffffu, incl, 1);
    int carry = s_wcarry[warp];
    if (lane > 0) carry = tf_apply(prev, carry);
    int zloc = INT_MAX;
#pragma unroll
    for (int c = 0; c < CHUNK; ++c) {  // final limbs (mod 2^(64 Ly))
        const uint64_t v = u[c] + (uint64_t)(int64_t)carry;
        carry = tf_apply(fl[c], carry);
        u[c] = v;
        if (l0 + c < Ly && v && zloc == INT_MAX) zloc = l0 + c;
        if (l0 + c == Ly - 1) s_neg = (int)(v >> 63);
    }
    if (zloc != INT_MAX) atomicMin(&s_zmin, zloc);
    __syncthreads();
    const bool neg = s_neg != 0;
    const int zmin = s_zmin;
    const int64_t orow = prm.reverse_out ? (prm.m - 1 - row) : row;
    uint64_t *yo = prm.y_mag + orow * Ly;
#pragma unroll
    for (int c = 0; c < CHUNK; ++c) {
        const int l = l0 + c;
        if (l < Ly) {
            uint64_t v = u[c];
            if (neg) v = l < zmin ? 0ull : (l == zmin ? (0ull - v) : ~v);
            yo[l] = v;
        }
    }
    if (tid == 0) prm.y_sign[orow] = neg ? (int8_t)-1 : (zmin < Ly ? (int8_t)1 : (int8_t)0);
}

// ------------------------------------------------------------------------------------------
// launchers
static int check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "hk: CUDA launch error: %s\n", cudaGetErrorString(e));
        return HK_ECUDA;
    }
    return HK_OK;
}

int launch_init(const Params &prm, const uint32_t *gens, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t total = (int64_t)kNumPrimes * (prm.N2 + prm.N1);
    const int threads = 256;
    const int blocks = (int)((total + threads - 1) / threads);
    k0_init<<<blocks, threads, 0, st>>>(prm, const_cast<uint2 *>(prm.tw), gens[0], gens[1],
                                        gens[2], gens[3], gens[4]);
    return check_launch();
}

template <int LOGN2>
static int launch_rows(const Params &prm0, cudaStream_t st, int tile0 = 0, int ntiles = -1) {
    const int ga = (int)((prm0.a_count + kK1Rows - 1) / kK1Rows);
    const int gx = (int)((prm0.n + kK1Rows - 1) / kK1Rows);
    if (ntiles < 0) ntiles = ga + gx - tile0;
    if (ntiles <= 0) return HK_OK;
    Params prm = prm0;
    prm.tile0 = tile0;
    const size_t limb_bytes = (size_t)kK1Rows * prm.L * sizeof(uint64_t);
    const size_t tab_bytes = (size_t)(1 << LOGN2) * sizeof(uint2);  // reuses the limb area
    const size_t smem1 = (size_t)kK1Rows * k1_row_stride<LOGN2>() * sizeof(uint32_t) +
                         (limb_bytes > tab_bytes ? limb_bytes : tab_bytes);
    if (cudaFuncSetAttribute(k1_slice_rowntt<LOGN2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem1) != cudaSuccess)
        return HK_ECUDA;
    k1_slice_rowntt<LOGN2><<<ntiles, k1_threads<LOGN2>(), smem1, st>>>(prm, ga);
    return check_launch();
}

template <int LOGN2>
static int launch_rows_inverse(const Params &prm0, cudaStream_t st, int64_t row0 = 0,
                               int64_t nrows = -1) {
    if (nrows < 0) nrows = prm0.m - row0;
    if (nrows <= 0) return HK_OK;
    Params prm = prm0;
    prm.row0 = row0;
    const size_t smem =
        (size_t)kNumPrimes * k3_rows<LOGN2>() * k1_row_stride<LOGN2>() * sizeof(uint32_t);
    if (cudaFuncSetAttribute(k3a_row_intt_crt<LOGN2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return HK_ECUDA;
    const unsigned grid = (unsigned)((nrows + k3_rows<LOGN2>() - 1) / k3_rows<LOGN2>());
    k3a_row_intt_crt<LOGN2><<<grid, kK3aThreads, smem, st>>>(prm);
    return check_launch();
}

template <int LOGN1>
static int launch_cols(const Params &prm, cudaStream_t st) {
    const int ncols = kNumPrimes * prm.N2;
    const size_t smem = k2_smem_bytes<LOGN1>();
    if (cudaFuncSetAttribute(k2_column<LOGN1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return HK_ECUDA;
    // one CTA per SM: keep the carveout minimal so the N1 twiddle table stays L1-resident
    const int pct = (int)((smem + 2048) * 100 / (228 * 1024)) + 1;
    if (getenv("HK_K2_CARVEOUT"))
        cudaFuncSetAttribute(k2_column<LOGN1>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             atoi(getenv("HK_K2_CARVEOUT")));
    (void)pct;
    const int diag = getenv("HK_K2_DIAG") ? atoi(getenv("HK_K2_DIAG")) : 0;  // diagnostics only
    Params p2 = prm;
    p2.diag = diag;
    if (diag & 1) {
        cudaFuncSetAttribute(k2_column<LOGN1, TwConst>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        k2_column<LOGN1, TwConst><<<ncols, k2_threads<LOGN1>(), smem, st>>>(p2);
    } else {
        k2_column<LOGN1><<<ncols, k2_threads<LOGN1>(), smem, st>>>(p2);
    }
    return check_launch();
}

int launch_ntt_path(const Params &prm, void *stream, uint32_t stages) {
    cudaStream_t st = (cudaStream_t)stream;
    int rc = HK_OK;
    if (stages & HK_STAGE_SLICE_ROWS) switch (prm.log_n2) {
#define HK_CASE(LG) case LG: rc = launch_rows<LG>(prm, st); break;
        HK_CASE(5) HK_CASE(6) HK_CASE(7) HK_CASE(8) HK_CASE(9) HK_CASE(10) HK_CASE(11)
#undef HK_CASE
        default: return HK_EUNSUPPORTED;
    }
    if (rc) return rc;
    if (stages & HK_STAGE_COLUMNS) switch (prm.log_n1) {
#define HK_CASE(LG) case LG: rc = launch_cols<LG>(prm, st); break;
        HK_CASE(6) HK_CASE(7) HK_CASE(8) HK_CASE(9) HK_CASE(10) HK_CASE(11) HK_CASE(12)
        HK_CASE(13) HK_CASE(14) HK_CASE(15)
#undef HK_CASE
        default: return HK_EUNSUPPORTED;
    }
    if (rc) return rc;
    if (!(stages & HK_STAGE_FINISH)) return HK_OK;
    return launch_k3_range(prm, stream, 0, prm.m);
}

template <int LOGN1, int MODE>
static int launch_cols_mode(const Params &prm, cudaStream_t st) {
    const int ncols = kNumPrimes * prm.N2;
    const size_t smem = (size_t)padded_len(1 << LOGN1) * sizeof(uint32_t);
    if (cudaFuncSetAttribute(k2_column<LOGN1, TwGlobal, MODE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return HK_ECUDA;
    k2_column<LOGN1, TwGlobal, MODE><<<ncols, k2_threads<LOGN1>(), smem, st>>>(prm);
    return check_launch();
}

int launch_k2_mode(const Params &prm, void *stream, int mode) {
    cudaStream_t st = (cudaStream_t)stream;
    if (mode == 0) return launch_ntt_path(prm, stream, HK_STAGE_COLUMNS);
    switch (prm.log_n1) {
#define HK_CASE(LG)                                                                   \
    case LG:                                                                          \
        return mode == 1 ? launch_cols_mode<LG, 1>(prm, st) : launch_cols_mode<LG, 2>(prm, st);
        HK_CASE(6) HK_CASE(7) HK_CASE(8) HK_CASE(9) HK_CASE(10) HK_CASE(11) HK_CASE(12)
        HK_CASE(13) HK_CASE(14) HK_CASE(15)
#undef HK_CASE
        default: return HK_EUNSUPPORTED;
    }
}

int k1_tiles_a(const Params &prm) { return (int)((prm.a_count + kK1Rows - 1) / kK1Rows); }
int k1_tiles_x(const Params &prm) { return (int)((prm.n + kK1Rows - 1) / kK1Rows); }

int launch_k1_range(const Params &prm, void *stream, int tile0, int ntiles) {
    cudaStream_t st = (cudaStream_t)stream;
    switch (prm.log_n2) {
#define HK_CASE(LG) case LG: return launch_rows<LG>(prm, st, tile0, ntiles);
        HK_CASE(5) HK_CASE(6) HK_CASE(7) HK_CASE(8) HK_CASE(9) HK_CASE(10) HK_CASE(11)
#undef HK_CASE
        default: return HK_EUNSUPPORTED;
    }
}

int launch_k3_range(const Params &prm0, void *stream, int64_t row0, int64_t nrows) {
    cudaStream_t st = (cudaStream_t)stream;
    int rc = HK_OK;
    switch (prm0.log_n2) {
#define HK_CASE(LG) case LG: rc = launch_rows_inverse<LG>(prm0, st, row0, nrows); break;
        HK_CASE(5) HK_CASE(6) HK_CASE(7) HK_CASE(8) HK_CASE(9) HK_CASE(10) HK_CASE(11)
#undef HK_CASE
        default: return HK_EUNSUPPORTED;
    }
    if (rc) return rc;
    if (nrows <= 0) return HK_OK;
    Params prm = prm0;
    prm.row0 = row0;
    const size_t smem3 = ((size_t)4 * prm.Ly * 8 + prm.Ly + 15) / 16 * 16;
    const int chunk = (prm.Ly + kK3Threads - 1) / kK3Threads;
    switch (chunk) {
#define HK_CASE(C)                                                                             \
    case C:                                                                                    \
        if (cudaFuncSetAttribute(k3b_carry<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                 (int)smem3) != cudaSuccess)                                   \
            return HK_ECUDA;                                                                   \
        k3b_carry<C><<<(unsigned)nrows, kK3Threads, smem3, st>>>(prm);                         \
        break;
        HK_CASE(1) HK_CASE(2) HK_CASE(3) HK_CASE(4) HK_CASE(5) HK_CASE(6) HK_CASE(7) HK_CASE(8)
        HK_CASE(9) HK_CASE(10) HK_CASE(11) HK_CASE(12) HK_CASE(13) HK_CASE(14) HK_CASE(15)
        HK_CASE(16) HK_CASE(17)
#undef HK_CASE
        default: return HK_EUNSUPPORTED;
    }
    return check_launch();
}

}  // namespace hk
