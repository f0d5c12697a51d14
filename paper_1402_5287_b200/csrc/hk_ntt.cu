// hk_ntt.cu -- the hot path: exact multiprecision Hankel/Toeplitz/circulant matvec as a 2-D
// multi-prime NTT convolution.
//
//   K0 k0_init           twiddle tables + workspace header (once per plan)
//   K1 k1_slice_rowntt   A1 limb slicing + validation, A2 slice-dimension forward NTT (N2),
//                        a and x tiles in one launch
//   K2 k2_column         A2 matrix-index forward NTTs (N1) of X^ and A^ columns, A3 pointwise
//                        Montgomery product, inverse matrix-index NTT, keep the n needed rows
//   K3 k3_finish         A3 inverse slice-dimension NTT, Garner CRT -> signed coefficients,
//                        A4 carry propagation and sign-magnitude output (one launch, rows tiled)
#include <cuda_runtime.h>

#include <mutex>
#include <unordered_map>

#include <climits>
#include <cstdio>
#include <cstdlib>

#include "hk_internal.h"
#include "hk_modarith.cuh"
#include "hk_k2.cuh"

namespace hk {

// Raise a kernel's dynamic shared-memory limit once per (kernel, size) instead of on every launch
// (the attribute call is host time that small problems feel; one device per process).
// The default limit covers static + dynamic <= 48 KB; beyond that the attribute must be raised.
static int ensure_smem(const void *kern, size_t smem) {
    if (smem <= 32 * 1024) return HK_OK;  // every kernel here has < 16 KB of static shared memory
    static std::mutex mu;
    static std::unordered_map<const void *, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t &cur = done[kern];
    if (smem <= cur) return HK_OK;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return HK_ECUDA;
    cur = smem;
    return HK_OK;
}

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
#ifndef HK_K1_ROWS
#define HK_K1_ROWS 8
#endif
#ifndef HK_K1_MINB
#define HK_K1_MINB 3
#endif
constexpr int kK1Rows = HK_K1_ROWS;
#ifndef HK_K1_MINB_SMALL
#define HK_K1_MINB_SMALL 5  // resident CTAs per SM for N2 <= 512 (128-thread CTAs; 3 -> 5: C5 K1 -4%)
#endif
template <int LOGN2>
constexpr int k1_minb() { return LOGN2 <= 9 ? HK_K1_MINB_SMALL : HK_K1_MINB; }
#ifndef HK_K1_TMA
#define HK_K1_TMA 1  // stage the limb tile with one TMA bulk copy (else per-thread cp.async)
#endif
#ifndef HK_K1_L2PF
#define HK_K1_L2PF 148  // tiles ahead whose limbs are bulk-prefetched into L2 (0: off)
#endif
// words of K1's transform area: the kK1Rows padded rows, or the tile's limbs if larger (16-byte
// multiple, so the twiddle tables after it stay 16-byte aligned)
__host__ __device__ inline int k1_transform_words(int rs, int L) {
    const int t = kK1Rows * rs, l = kK1Rows * L * 2;
    return ((t > l ? t : l) + 3) & ~3;
}
template <int LOGN2>
constexpr int k1_threads() {
    return kK1Rows * ((1 << LOGN2) / 32 > 8 ? (1 << LOGN2) / 32 : 8);
}

// GAMMA > 0 (sigma-coset shards): only block b = prm.k1_block of the 2^GAMMA
// blocks of N2 / 2^GAMMA consecutive outputs is produced.  After the first GAMMA DIF stages the
// array splits into independent blocks; block b only needs, at stage h, the "sum" (bit 0) or the
// "difference x twiddle" (bit 1) half selected by b's bits from the top -- i.e. the coset fold.
// Block b holds the transform outputs at bit-reversed positions [b N2 / G, (b + 1) N2 / G), the
// frequencies congruent to bitrev(b) mod G.
template <int LOGN2, int GSEL>  // GSEL = gamma (coset shards keep N2 / 2^gamma outputs), -1: sliced shards
__global__ void __launch_bounds__(k1_threads<LOGN2>(), k1_minb<LOGN2>()) k1_slice_rowntt(Params prm, int tiles_a) {
    constexpr int GAMMA = GSEL < 0 ? 0 : GSEL;
    constexpr bool SLICED = GSEL < 0;
    constexpr int N2 = 1 << LOGN2;
    constexpr int BL = N2 >> GAMMA;          // outputs kept per row and prime
    constexpr int GK = 32 >> GAMMA;          // top-pass points kept per group
    static_assert(BL >= 32, "shard blocks must hold >= 32 outputs");
    constexpr int RS = k1_row_stride<LOGN2>();
    constexpr int T = k1_threads<LOGN2>();
    constexpr int R1 = 5, G1 = 32, H1 = 16;  // top pass: 32 points, upper 16 are zero padding
    constexpr int S1 = N2 / G1;              // top-pass groups per row
    constexpr int TPR = T / kK1Rows;         // threads per row (>= S1)
    static_assert(LOGN2 >= 5 && TPR >= S1, "K1 tiling");
    extern __shared__ uint32_t sm[];
    __shared__ int8_t s_sign[kK1Rows];

    const int tid = threadIdx.x;
    if (prm.hdr->magic != kWsMagic || prm.hdr->hash != prm.hash) {
        if (tid == 0 && blockIdx.x == 0) atomicMin(&prm.hdr->status, (int)HK_EINVAL);
        return;
    }
    const int bt = (int)blockIdx.x + prm.tile0 + ((int)blockIdx.x >= prm.tile_split ? prm.tile_skip : 0);
    const bool is_x = bt >= tiles_a;
    if (prm.need_a_ready && prm.hdr->a_ready != 1) {
        if (tid == 0) atomicMin(&prm.hdr->status, (int)HK_EINVAL);
        return;
    }
    const int tile = is_x ? bt - tiles_a : bt;
    const int64_t vb = (int64_t)blockIdx.y;  // batch vector (x tiles only; 0 otherwise)
    const uint64_t *mag = is_x ? prm.x_mag + vb * prm.x_vstride * prm.L : prm.a_mag;
    const int8_t *sgn = is_x ? prm.x_sign + vb * prm.x_vstride : prm.a_sign;
    const int64_t count = is_x ? prm.n : prm.a_count;
    uint32_t *out = is_x ? prm.Xhat + vb * (int64_t)kNumPrimes * prm.n2loc * prm.ldX : prm.Ahat;
    const int64_t ld = is_x ? prm.ldX : prm.ldA;
    const bool rev = is_x && prm.x_reversed;
    const int64_t r0 = (int64_t)tile * kK1Rows;
    const int L = prm.L, w = prm.w, Ls = prm.Ls;

    // ---- stage the tile's limbs (kK1Rows consecutive entries = one contiguous block) in smem: in
    // the transform area, dead until the first prime's top pass (the limbs fit: L <= N2 / 2 + 1
    // for w >= 64); the two N2 twiddle tables live after it
    uint64_t *slimb = reinterpret_cast<uint64_t *>(sm);
    const int ta_words = k1_transform_words(RS, L);
    uint2 *stw = reinterpret_cast<uint2 *>(sm + ta_words);
    {
        const int64_t nrows = count - r0 < kK1Rows ? count - r0 : kK1Rows;
        const int64_t bytes = nrows * L * 8;
        const char *g = reinterpret_cast<const char *>(mag + r0 * L);
        char *d = reinterpret_cast<char *>(slimb);
#if HK_K1_TMA
        // one TMA bulk copy of the tile's contiguous limb block (its 16-byte-aligned part)
        __shared__ __align__(8) uint64_t s_mbar;
        if (tid == 0) mbar_init(&s_mbar, 1);
        __syncthreads();
        if (tid == 0) bulk_copy_g2s(d, g, (unsigned)(bytes & ~int64_t(15)), &s_mbar);
#else
        for (int64_t c = tid; c < bytes / 16; c += T) cp_async16(d + 16 * c, g + 16 * c);
#endif
        if ((bytes & 15) && tid == 0) cp_async8(d + (bytes & ~int64_t(15)), g + (bytes & ~int64_t(15)));
        if (HK_K1_L2PF && tid == 0) {  // bring the limbs of the tile one wave ahead into L2
            const int bt2 = bt + HK_K1_L2PF;
            const bool x2 = bt2 >= tiles_a;
            const int64_t cnt2 = x2 ? prm.n : prm.a_count;
            const int64_t q0 = (int64_t)(x2 ? bt2 - tiles_a : bt2) * kK1Rows;
            if (q0 < cnt2) {
                const int64_t nr2 = cnt2 - q0 < kK1Rows ? cnt2 - q0 : kK1Rows;
                const uint64_t *g2 = (x2 ? prm.x_mag + vb * prm.x_vstride * L : prm.a_mag) + q0 * L;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(g2),
                             "r"((unsigned)(nr2 * L * 8) & ~15u) : "memory");
            }
        }
        cp_async_wait_all();
#if HK_K1_TMA
        mbar_wait_parity(&s_mbar, 0);
#endif
        __syncthreads();
    }
    // ---- validation (A1): bits >= P zero, sign in {-1,0,1}, sign == 0 <=> magnitude == 0;
    // one warp per row (no division by L, one vote per row)
    {
        const int rem = prm.P - 64 * (L - 1);
        const uint64_t topmask = rem >= 64 ? ~0ull : ((1ull << rem) - 1);
        const int lane = tid & 31;
        for (int r = tid >> 5; r < kK1Rows; r += T / 32) {
            const int64_t row = r0 + r;
            int sg = 0;
            if (row < count) {
                const uint64_t *rp = slimb + r * L;
                uint64_t orv = 0;
                for (int u = lane; u < L; u += 32) orv |= rp[u];
                const bool nz = __any_sync(0xffffffffu, orv != 0);
                if (lane == 0) {
                    sg = sgn[row];
                    if ((rp[L - 1] & ~topmask) || sg < -1 || sg > 1 || ((sg == 0) == nz))
                        atomicMin(&prm.hdr->status, (int)HK_ERANGE);
                }
            }
            if (lane == 0) s_sign[r] = (int8_t)sg;
        }
        __syncthreads();
    }

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

    // N2 twiddle tables -> smem, double-buffered in the (now free) limb staging area: the table
    // of prime kp + 2 streams in by cp.async while prime kp is transformed
    auto fetch_tw = [&](int kp) {
        uint4 *dst = reinterpret_cast<uint4 *>(stw) + (kp & 1) * (N2 / 2);
        const uint4 *src = reinterpret_cast<const uint4 *>(prm.tw + (size_t)kp * (prm.N2 + prm.N1));
        for (int i = tid; i < N2 / 2; i += T) cp_async16(dst + i, src + i);
        cp_async_commit();
    };
    __syncthreads();  // every thread is done with the limbs
    // primes [kb, ke): all five, or (launches under one wave, prm.k1_prime_split) blockIdx.z's
    const int kb = prm.k1_prime_split ? (int)blockIdx.z : 0;
    const int ke = prm.k1_prime_split ? kb + 1 : kNumPrimes;
    fetch_tw(kb);
    if (kb + 1 < ke) fetch_tw(kb + 1);
    for (int kp = kb; kp < ke; ++kp) {
        const uint32_t p = prm.pc[kp].p;
        const uint32_t *F = is_x ? prm.pc[kp].fx : prm.pc[kp].fa;
        const uint32_t *Fq = is_x ? prm.pc[kp].fx_q : prm.pc[kp].fa_q;
        const uint2 *tw = stw + (kp & 1) * N2;
        if (kp + 1 < ke) cp_async_wait_group<1>();
        else cp_async_wait_group<0>();
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
            if constexpr (GAMMA == 0) {
#pragma unroll
                for (int m = 0; m < H1; ++m) {
                    const uint2 wv = TwShared::ld(tw, S1 * H1 + j0 + S1 * m);
                    v[m + H1] = red1(shoup(v[m], wv.x, wv.y, p), p);
                }
            } else {  // keep the half selected by the top bit of b (in v[0 .. 16))
                if ((prm.k1_block >> (GAMMA - 1)) & 1) {
#pragma unroll
                    for (int m = 0; m < H1; ++m) {
                        const uint2 wv = TwShared::ld(tw, S1 * H1 + j0 + S1 * m);
                        v[m] = red1(shoup(v[m], wv.x, wv.y, p), p);
                    }
                }
#pragma unroll
                for (int l = 1; l < GAMMA; ++l) {  // stages h = N2/4 .. : keep one half each
                    const int half = H1 >> l;
                    const bool hi = (prm.k1_block >> (GAMMA - 1 - l)) & 1;
#pragma unroll
                    for (int m = 0; m < half; ++m) {
                        const uint32_t u = v[m], w = v[m + half];
                        if (hi) {
                            const uint2 wv = TwShared::ld(tw, S1 * half + j0 + S1 * m);
                            v[m] = red1(shoup(u - w + p, wv.x, wv.y, p), p);
                        } else {
                            v[m] = addm(u, w, p);
                        }
                    }
                }
            }
#pragma unroll
            for (int l = R1 - 2 - (GAMMA > 0 ? GAMMA - 1 : 0); l >= 0; --l) {
                const int half = 1 << l;
#pragma unroll
                for (int m = 0; m < GK; ++m) {
                    if (m & half) continue;
                    const uint2 wv = TwShared::ld(tw, S1 * half + j0 + S1 * (m & (half - 1)));
                    gs_bfly(v[m], v[m + half], wv, p);
                }
            }
#pragma unroll
            for (int m = 0; m < GK; ++m) sm[r * RS + pad(j0) + padded_len(m * S1)] = v[m];
        }
        __syncthreads();
        constexpr int REM = LOGN2 - R1;          // stages left after the top pass
        constexpr int RB = REM < 5 ? REM : 5;    // bottom pass (S = 1) radix
        if constexpr (REM > RB)  // block-local (positions relative to the block start)
            dif_pass<TwShared, LOGN2 - GAMMA, REM - RB, (1 << RB), false>(sm, kK1Rows, RS, tw, p, tid, T);
        // ---- bottom pass in registers, stored straight to [prime][sigma][row]; lanes cover
        // 8 rows x 4 groups so every store instruction writes full 32-byte row segments
        // (x rows reversed: matrix index n-1-row)
        constexpr int GB = 1 << RB, NGR = BL / GB;
        for (int gi = tid; gi < kK1Rows * NGR; gi += T) {
            const int rr = gi % kK1Rows, g = gi / kK1Rows;
            uint32_t v[GB];
#pragma unroll
            for (int m = 0; m < GB; ++m) v[m] = sm[rr * RS + pad(g * GB) + m];
            dif_bottom_regs<TwShared, RB>(v, tw, p);
            const int64_t orow = r0 + rr;
            if (orow < count) {
                const int64_t pos = rev ? (count - 1 - orow) : orow;
                if constexpr (SLICED) {
                    // sliced shards: positions [src Rs, (src+1) Rs) of this rank only; sigma-block
                    // d = (g GB) / n2loc goes to chunk d of the send buffer (or, over peer memory,
                    // to chunk src of rank d's receive buffer)
                    const int lg = is_x ? prm.lg_rs_x : prm.lg_rs_a;
                    const int64_t lo = (int64_t)prm.k1_block << lg;
                    if (pos >= lo && pos < lo + (int64_t(1) << lg)) {
                        const int sg0 = g * GB, dst = sg0 >> prm.log_n2loc, sl = sg0 & (prm.n2loc - 1);
                        uint32_t *base = prm.p2p ? prm.peer_slice[dst] + (int64_t)prm.k1_block * prm.slice_chunk
                                                 : prm.slice_out + (int64_t)dst * prm.slice_chunk;
                        uint32_t *o = base + (is_x ? prm.slice_xoff : 0) + (((int64_t)kp * prm.n2loc + sl) << lg) +
                                      (pos - lo);
#pragma unroll
                        for (int m = 0; m < GB; ++m) o[(int64_t)m << lg] = v[m];
                    }
                } else {
                    uint32_t *o = out + ((int64_t)kp * BL + (int64_t)g * GB) * ld + pos;
#pragma unroll
                    for (int m = 0; m < GB; ++m) o[(int64_t)m * ld] = v[m];
                }
            }
        }
        __syncthreads();
        if (kp + 2 < ke) fetch_tw(kp + 2);
    }
    if constexpr (SLICED) if (prm.p2p) __threadfence_system();  // peer slice stores visible
}

// ------------------------------------------------------------------------------------------
// K3 (fused): for R = k3_rows() output rows and all 5 primes in shared memory
//   (a) inverse slice-dimension NTT (DIT with forward roots: slice index negated),
//   (b) Garner CRT of every coefficient C_s, |C_s| < M/2 < 2^155, as five 32-bit
//       two's-complement words written in place over the residues,
//   (c) per row: Y = sum_s C_s 2^(w s) mod 2^(64 Ly) gathered limb by limb (w in {64, 65}
//       makes the limb index q(s) = floor(w s / 64) injective), carries resolved by a block
//       scan of carry-transfer functions, two's complement -> sign-magnitude, coalesced store.
// Shared layout: word (prime kp, slice sigma, row r) at kp PS + pad(sigma) R + r with
// pad(sigma) = sigma + sigma / 32: rows interleaved so one 16-byte cp.async brings the R rows of a
// (prime, sigma) column segment; the pad keeps the contiguous (S = 1, radix 32: lanes 32 sigma
// apart) and the strided (S >= 32 / R) passes and the Garner pairs bank-conflict-free, and it is
// separable (pad(B + j0 + m S) = pad(B + j0) + pad(m S)) so per-point offsets are immediates.
#ifndef HK_K3_ROWS
#define HK_K3_ROWS 4   // output rows per K3 tile (N2 <= 1024)
#endif
#ifndef HK_K3_BLOCK
#define HK_K3_BLOCK 384  // 96 threads per row, 80 registers, 2 CTAs/SM (320: 96 registers, C3 K3 +5%)
#endif
#ifndef HK_K3_GARNER_SLOT
#define HK_K3_GARNER_SLOT 1  // Garner slot by slot (CRT words at the residue slot) instead of in pairs
#endif
#ifndef HK_K3_FLAT_STORE
#define HK_K3_FLAT_STORE 1  // y rows of a tile stored as one flat range
#endif
#ifndef HK_K3_MINB
#define HK_K3_MINB 2
#endif
#ifndef HK_K3_GARNER_X2
#define HK_K3_GARNER_X2 0  // two Garner slots per thread per round
#endif
#ifndef HK_K3_WSCAN
#define HK_K3_WSCAN 1  // each thread folds the earlier warps' carry totals itself (one barrier fewer; C3 K3 -0.6%)
#endif
#ifndef HK_K3_FUSED
#define HK_K3_FUSED 1  // Garner fused into the carry gather (no separate CRT phase, no lookbehind): C3 K3 -1.5%
#endif
#ifndef HK_K3_SKIP
#define HK_K3_SKIP 0  // dev timing only (wrong results): 1 skips the inverse NTTs, 2 Garner, 4 the
                      // gather, 8 the Y^ load, 16 the y store
#endif
template <int LOGN2>
constexpr int k3_rows() { return LOGN2 >= 11 ? 2 : HK_K3_ROWS; }
// threads per K3 CTA and CTAs per SM: HK_K3_BLOCK (320 for the 2-row tiles of N2 = 2048)
template <int LOGN2>
constexpr int k3_threads() { return LOGN2 >= 11 ? 320 : HK_K3_BLOCK; }
template <int LOGN2>
constexpr int k3_minb() { return LOGN2 >= 11 ? 2 : HK_K3_MINB; }

template <int LOGN2>
struct K3Layout {
    static constexpr int N2 = 1 << LOGN2, R = k3_rows<LOGN2>(), PS = padded_len(N2) * R;
    static HK_DEV int idx(int kp, int s, int r) { return kp * PS + pad(s) * R + r; }
    static constexpr size_t res_words() { return (size_t)kNumPrimes * PS; }
};

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

#ifndef HK_K3_V2
#define HK_K3_V2 1  // unsigned CRT (ascending Garner over C + H) + unsigned carry gather
#endif
// K3 v2 CRT: digits of C'' = C + H (H = (M-1)/2, so C'' is in [0, M) with no sign test) with the
// primes in ascending order p'_0 < ... < p'_4: every earlier digit u_j < p'_j < p'_g, so
// x = t + p'_g - u_j lies in (0, 2 p'_g) and is = t - u_j (mod p'_g) with no reduction first.
//   u_g = ((((r_g + h_g) - u_0) c_0g - u_1) c_1g - ...) mod p'_g,   c_jg = p'_j^-1 mod p'_g
//   C'' = u_0 + p'_0 (u_1 + p'_1 (u_2 + p'_2 (u_3 + p'_3 u_4)))  as five 32-bit words.
HK_DEV void garner2(const uint32_t r[kNumPrimes], const Params &prm, uint32_t (&cw)[kNumPrimes]) {
    const Garner2Consts &G = prm.g2;
    uint32_t u[kNumPrimes];
#pragma unroll
    for (int g = 0; g < kNumPrimes; ++g) {
        const uint32_t p = G.p[g];
        uint32_t t = addm(r[kNumPrimes - 1 - g], G.h[g], p);  // residues are in descending order
#pragma unroll
        for (int j = 0; j < g; ++j) t = red1(shoup(t + p - u[j], G.c[j][g], G.cq[j][g], p), p);
        u[g] = t;
    }
    uint64_t v = (uint64_t)u[4] * G.p[3] + u[3];
    uint32_t a0 = (uint32_t)v, a1 = (uint32_t)(v >> 32), a2, a3, a4;
    v = (uint64_t)a0 * G.p[2] + u[2]; a0 = (uint32_t)v;
    v = (uint64_t)a1 * G.p[2] + (v >> 32); a1 = (uint32_t)v; a2 = (uint32_t)(v >> 32);
    v = (uint64_t)a0 * G.p[1] + u[1]; a0 = (uint32_t)v;
    v = (uint64_t)a1 * G.p[1] + (v >> 32); a1 = (uint32_t)v;
    v = (uint64_t)a2 * G.p[1] + (v >> 32); a2 = (uint32_t)v; a3 = (uint32_t)(v >> 32);
    v = (uint64_t)a0 * G.p[0] + u[0]; a0 = (uint32_t)v;
    v = (uint64_t)a1 * G.p[0] + (v >> 32); a1 = (uint32_t)v;
    v = (uint64_t)a2 * G.p[0] + (v >> 32); a2 = (uint32_t)v;
    v = (uint64_t)a3 * G.p[0] + (v >> 32); a3 = (uint32_t)v; a4 = (uint32_t)(v >> 32);
    cw[0] = a0; cw[1] = a1; cw[2] = a2; cw[3] = a3; cw[4] = a4;
}

// K3 v2 carry helpers: (hi:lo) += (vh:vl) with the carry out counted (add.cc chain), and a
// branch-free 32-bit select
HK_DEV void add64_count(uint32_t &lo, uint32_t &hi, int &cnt, uint32_t vl, uint32_t vh) {
    asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, 0;"
        : "+r"(lo), "+r"(hi), "+r"(cnt) : "r"(vl), "r"(vh));
}
HK_DEV uint32_t sel32(bool c, uint32_t a, uint32_t b) {  // c ? a : b
    uint32_t d;
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\tselp.b32 %0, %2, %3, p;\n\t}"
        : "=r"(d) : "r"((uint32_t)c), "r"(a), "r"(b));
    return d;
}


// Inverse DIT pass of radix 2^RR at stride S over all (prime, row) transforms of the tile.
template <int LOGN2, int RR, int S>
HK_DEV void k3_dit_pass(uint32_t *sm, const Params &prm) {
    using LY = K3Layout<LOGN2>;
    constexpr int N = 1 << LOGN2, G = 1 << RR, NG = N / G, R = LY::R;
    constexpr int total = kNumPrimes * R * NG;
    for (int gi = threadIdx.x; gi < total; gi += k3_threads<LOGN2>()) {
        const int r = gi % R, rest = gi / R;
        const int g = rest % NG, kp = rest / NG;
        const uint32_t p = prm.pc[kp].p;
        const uint2 *tw = prm.tw + (size_t)kp * (prm.N2 + prm.N1);
        const int j0 = g % S, B = (g / S) * (S * G);
        uint32_t *b0 = sm + LY::idx(kp, B + j0, r);
        uint32_t v[G];
#pragma unroll
        for (int m = 0; m < G; ++m) v[m] = b0[padded_len(m * S) * R];
#pragma unroll
        for (int l = 0; l < RR; ++l) {
            const int half = 1 << l;
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & half) continue;
                if (S == 1 && (m & (half - 1)) == 0) bfly1(v[m], v[m + half], p);  // twiddle 1
                else ct_bfly(v[m], v[m + half], TwGlobal::ld(tw, S * half + j0 + S * (m & (half - 1))), p);
            }
        }
#pragma unroll
        for (int m = 0; m < G; ++m) b0[padded_len(m * S) * R] = v[m];
    }
    __syncthreads();
}
template <int LOGN2, int LO>
struct K3Dit {  // radix-32 bottom pass (S = 1) first, then passes of radix <= 32 at S >= 32
    static HK_DEV void run(uint32_t *sm, const Params &prm) {
        if constexpr (LO < LOGN2) {
            constexpr int RR = (LOGN2 - LO) < 5 ? (LOGN2 - LO) : 5;
            k3_dit_pass<LOGN2, RR, (1 << LO)>(sm, prm);
            K3Dit<LOGN2, LO + RR>::run(sm, prm);
        }
    }
};

// carry-transfer function {-1,0,1} -> {-1,0,1}, packed 2 bits per input (value + 1)
HK_DEV int tf_apply(int f, int c) { return ((f >> (2 * (c + 1))) & 3) - 1; }
HK_DEV int tf_compose(int g, int f) {  // g o f
    int h = 0;
#pragma unroll
    for (int c = -1; c <= 1; ++c) h |= (tf_apply(g, tf_apply(f, c)) + 1) << (2 * (c + 1));
    return h;
}
constexpr int kTfId = (0) | (1 << 2) | (2 << 4);

// coefficient index s with limb index q(s) = floor(w s / 64) == qq (w in {64, 65}), else -1;
// *sh = w s mod 64.  w = 65: s = 64 a + b, q = 65 a + b (b < 64).
HK_DEV int k3_coef_of_limb(int qq, int w, int *sh) {
    if (w == 64) { *sh = 0; return qq; }
    const int a = qq / 65, b = qq - 65 * a;
    *sh = b;
    return b < 64 ? 64 * a + b : -1;
}

// F4: y rounded to the input format, m = round_half_even(|Y| / 2^P) with the sign
// of Y (y = m 2^-P; canonical: sign 0 iff m = 0), Lr = L + 1 output limbs (|Y| / 2^P < n 2^P).
// M: |Y| in Ly limbs (shared).  Block-wide: sticky bits, the first q limb that is not all ones
// (where a rounding increment stops), and whether q is nonzero.
HK_DEV void k3_store_rounded(const Params &prm, const uint64_t *M, bool neg, int64_t orow,
                             uint64_t *y_mag, int8_t *y_sign) {
    __shared__ int s_first;
    const int tid = threadIdx.x, T = blockDim.x, Ly = prm.Ly, Lr = prm.L + 1, P = prm.P;
    const int qs = P >> 6, qb = P & 63, hl = (P - 1) >> 6, hb = (P - 1) & 63;
    if (tid == 0) s_first = INT_MAX;
    __syncthreads();
    int sticky = 0, nz = 0;
    for (int l = tid; l <= hl; l += T) {  // bits [0, P - 1)
        const uint64_t v = M[l];
        sticky |= (l < hl ? v : (v & ((1ull << hb) - 1))) != 0;
    }
    for (int j = tid; j < Lr; j += T) {
        const uint64_t lo = qs + j < Ly ? M[qs + j] : 0, hi = qs + j + 1 < Ly ? M[qs + j + 1] : 0;
        const uint64_t q = qb ? ((lo >> qb) | (hi << (64 - qb))) : lo;
        nz |= q != 0;
        if (q != ~0ull) atomicMin(&s_first, j);
    }
    sticky = __syncthreads_or(sticky);
    nz = __syncthreads_or(nz);
    const bool half = (M[hl] >> hb) & 1;
    const bool lsb = (M[qs] >> qb) & 1;
    const bool inc = half && (sticky || lsb);
    const int first = s_first;
    uint64_t *yo = y_mag + orow * Lr;
    for (int j = tid; j < Lr; j += T) {
        const uint64_t lo = qs + j < Ly ? M[qs + j] : 0, hi = qs + j + 1 < Ly ? M[qs + j + 1] : 0;
        uint64_t q = qb ? ((lo >> qb) | (hi << (64 - qb))) : lo;
        if (inc) q = j < first ? 0ull : (j == first ? q + 1 : q);
        yo[j] = q;
    }
    if (tid == 0) y_sign[orow] = (nz || inc) ? (neg ? (int8_t)-1 : (int8_t)1) : (int8_t)0;
    __syncthreads();  // s_first reuse
}

template <int LOGN2, int CH>  // CH = limbs per thread = ceil(Ly / (k3_threads / R))
__global__ void __launch_bounds__(k3_threads<LOGN2>(), k3_minb<LOGN2>()) k3_finish(Params prm) {
    using LY = K3Layout<LOGN2>;
    constexpr int N2 = 1 << LOGN2, R = LY::R, T = k3_threads<LOGN2>();
    extern __shared__ uint32_t sm[];  // residues -> CRT words [5][N2][R] (swizzled) -> y rows [R][Ly]
    __shared__ int s_wtot[T / 32 * R], s_wcarry[T / 32 * R];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = prm.row0 + (int64_t)blockIdx.x * R;
    const int64_t m = prm.m;
    if (HK_K3_SKIP & 32) return;
    const int64_t vb = (int64_t)blockIdx.y;  // batch vector (0 unless hk_matvec_prepared_batch)
    const uint32_t *Yhat = prm.Yhat + vb * (int64_t)kNumPrimes * N2 * prm.ldY;
    uint64_t *y_mag = prm.y_mag + vb * prm.y_vstride * (prm.round_out ? prm.L + 1 : prm.Ly);
    int8_t *y_sign = prm.y_sign + vb * prm.y_vstride;

    // (0) Y^ columns of the R rows, all primes -> smem
    {
        const bool vec = r0 + R <= m && ((r0 & (R - 1)) == 0);
        for (int e = tid; e < kNumPrimes * N2; e += T) {
            const int kp = e >> LOGN2, sg = e & (N2 - 1);
            const uint32_t *g;
            if (prm.shard_gamma == 0) {
                g = Yhat + (int64_t)(kp * N2 + sg) * prm.ldY + r0;
            } else {  // all-to-all receive buffer [source rank][prime][sigma-block column][rpr]
                const int src = sg >> prm.log_n2loc, q = sg & (prm.n2loc - 1);  // rank src held block src
                g = prm.Yhat + ((int64_t)(src * kNumPrimes + kp) * prm.n2loc + q) * prm.shard_rpr +
                    (r0 - prm.shard_row0);
            }
            uint32_t *d = sm + LY::idx(kp, sg, 0);
            if (HK_K3_SKIP & 8) {
                d[0] = e;
            } else if (vec) {
                if constexpr (R == 8) { cp_async16(d, g); cp_async16(d + 4, g + 4); }
                else if constexpr (R == 4) cp_async16(d, g);
                else cp_async8(d, g);
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) d[r] = r0 + r < m ? g[r] : 0u;
            }
        }
        cp_async_wait_all();
        __syncthreads();
    }
    // (a) inverse slice NTTs
#if !(HK_K3_SKIP & 1)
    K3Dit<LOGN2, 0>::run(sm, prm);
#endif
    // fused (HK_K3_FUSED, chunks of >= 3 limbs): each coefficient is converted inside the carry
    // gather (c) below instead
    constexpr bool kFused = HK_K3_FUSED && HK_K3_V2 && CH >= 3;
#if HK_K3_SKIP & 2
#elif HK_K3_GARNER_X2 && HK_K3_V2
    // (b) Garner CRT in place, two slots per thread per round (independent chains interleave)
    for (int it = tid; it < R * N2; it += 2 * T) {
        const int itb = it + T < R * N2 ? it + T : it;
        const int r = it % R, sg = it / R, rb = itb % R, sgb = itb / R;
        uint32_t ra[kNumPrimes], rbv[kNumPrimes], ca[kNumPrimes], cb[kNumPrimes];
#pragma unroll
        for (int kp = 0; kp < kNumPrimes; ++kp) {
            ra[kp] = sm[LY::idx(kp, sg, r)];
            rbv[kp] = sm[LY::idx(kp, sgb, rb)];
        }
        garner2(ra, prm, ca);
        garner2(rbv, prm, cb);
        if (sg == 1) {
#pragma unroll
            for (int k = 0; k < kNumPrimes; ++k) ca[k] = 0;
        }
        if (sgb == 1) {
#pragma unroll
            for (int k = 0; k < kNumPrimes; ++k) cb[k] = 0;
        }
#pragma unroll
        for (int k = 0; k < kNumPrimes; ++k) sm[LY::idx(k, sg, r)] = ca[k];
        if (itb != it) {
#pragma unroll
            for (int k = 0; k < kNumPrimes; ++k) sm[LY::idx(k, sgb, rb)] = cb[k];
        }
    }
#elif HK_K3_GARNER_SLOT
    // (b) Garner CRT in place, slot by slot: coefficient s lives at sigma = (N2 - s) mod N2 and its
    // CRT words overwrite its own residues there, so any thread may take any slot (R N2 slots over
    // the block: no pairing, no remainder round of pairs)
    for (int it = tid; it < (kFused ? 0 : R * N2); it += T) {
        const int r = it % R, sg = it / R;
        uint32_t ra[kNumPrimes], ca[kNumPrimes];
#pragma unroll
        for (int kp = 0; kp < kNumPrimes; ++kp) ra[kp] = sm[LY::idx(kp, sg, r)];
#if HK_K3_V2
        garner2(ra, prm, ca);
        if (sg == 1) {  // s = N2 - 1 >= S2 is never a coefficient: a zero slot for the gather
#pragma unroll
            for (int k = 0; k < kNumPrimes; ++k) ca[k] = 0;
        }
#else
        garner(ra, prm, ca);
#endif
#pragma unroll
        for (int k = 0; k < kNumPrimes; ++k) sm[LY::idx(k, sg, r)] = ca[k];
    }
#else
    // (b) Garner CRT in place: coefficient s lives at sigma = (N2 - s) mod N2 and its CRT words
    // go to sigma = s, so the pair {s, N2 - s} is read and written by one thread.
    for (int it = tid; it < R * (N2 / 2 + 1); it += T) {
        const int r = it % R, s1 = it / R, s2 = (N2 - s1) & (N2 - 1);
        uint32_t ra[kNumPrimes], rb[kNumPrimes], ca[kNumPrimes], cb[kNumPrimes];
#pragma unroll
        for (int kp = 0; kp < kNumPrimes; ++kp) {
            ra[kp] = sm[LY::idx(kp, s2, r)];
            rb[kp] = sm[LY::idx(kp, s1, r)];
        }
        garner(ra, prm, ca);
#pragma unroll
        for (int k = 0; k < kNumPrimes; ++k) sm[LY::idx(k, s1, r)] = ca[k];
        if (s2 != s1) {
            garner(rb, prm, cb);
#pragma unroll
            for (int k = 0; k < kNumPrimes; ++k) sm[LY::idx(k, s2, r)] = cb[k];
        }
    }
#endif
    if constexpr (!kFused) __syncthreads();

#if HK_K3_V2
    const int Ly = prm.Ly;
    const int r = tid % R, k = tid / R, lane_r = lane / R;  // lane_r: position among the row's lanes
    const int l0 = k * CH;
    const uint32_t *smr = sm + r;
    uint64_t u[CH];                  // limb values of the chunk
    uint32_t gbits = 0, pbits = 0;   // per-limb generate / propagate bits
    uint32_t Gt = 0, Pt = 1;         // the chunk's composed (G, P)
    __shared__ int s_neg[R], s_zmin[R];
    if constexpr (kFused) {
        // (c) v3, Garner fused into the gather: thread t owns limbs [k CH, k CH + CH) of row r = t % R
        // (k = t / R) and converts exactly the coefficients that sit at those limbs (the residues of
        // coefficient s at its slot -> garner2 -> five words C'' < M), shifting each into the partial
        // sums of limbs q .. q + 3 (w = 65: q = 65 a + b for s = 64 a + b, shift b; w = 64: q = s).
        // Limb l0 + c is complete after position l0 + c except for the spill-over of the previous
        // chunk's last three coefficients into limbs l0 .. l0 + 2: that arrives through shared memory
        // (the previous thread's pending partial sums and carry counts) instead of being recomputed.
        const uint32_t *qmap = prm.qmap + l0 + 3;  // entry c: position l0 + c (padded past Ly)
        const uint64_t *negk = prm.negK + l0;      // zero-padded past Ly
        constexpr uint32_t kZeroSlot = (uint32_t)R;  // LY::idx(0, 1, 0) = pad(1) R: s = N2 - 1, never a coefficient
        static_assert(CH <= 16, "4-bit carry counts for at most 16 limbs per thread");
        uint32_t a0l = 0, a0h = 0, a1l = 0, a1h = 0, a2l = 0, a2h = 0;
        int n0 = 0, n1 = 0, n2 = 0;
        uint64_t ecnt = 0;              // e_c: carries out of those sums, 4 bits per limb
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const uint32_t qm = __ldg(qmap + c);
            const uint32_t o = qm >> 6, sh = qm & 63u;
            uint32_t ra[kNumPrimes], cw[kNumPrimes];
#pragma unroll
            for (int kp = 0; kp < kNumPrimes; ++kp) ra[kp] = smr[kp * LY::PS + o];
            garner2(ra, prm, cw);
            const bool zs = o == kZeroSlot;
            const uint32_t w0 = zs ? 0u : cw[0], w1 = zs ? 0u : cw[1], w2 = zs ? 0u : cw[2],
                           w3 = zs ? 0u : cw[3], w4 = zs ? 0u : cw[4];
            const uint32_t bs = sh & 31u;
            const uint32_t h0 = w0 << bs, h1 = __funnelshift_l(w0, w1, bs), h2 = __funnelshift_l(w1, w2, bs),
                           h3 = __funnelshift_l(w2, w3, bs), h4 = __funnelshift_l(w3, w4, bs),
                           h5 = __funnelshift_l(w4, 0u, bs);
            const bool up = sh >= 32u;  // the image starts one 32-bit word higher
            const uint32_t s0 = sel32(up, 0u, h0), s1 = sel32(up, h0, h1), s2 = sel32(up, h1, h2),
                           s3 = sel32(up, h2, h3), s4 = sel32(up, h3, h4), s5 = sel32(up, h4, h5),
                           s6 = sel32(up, h5, 0u);
            add64_count(a0l, a0h, n0, s0, s1);  // limb l0 + c
            add64_count(a1l, a1h, n1, s2, s3);  // limb l0 + c + 1
            add64_count(a2l, a2h, n2, s4, s5);  // limb l0 + c + 2 (s6 -> limb l0 + c + 3, below)
            const uint64_t nk = __ldg(negk + c);
            add64_count(a0l, a0h, n0, (uint32_t)nk, (uint32_t)(nk >> 32));
            u[c] = (uint64_t)a0h << 32 | a0l;
            ecnt |= (uint64_t)n0 << (4 * c);
            a0l = a1l; a0h = a1h; n0 = n1;
            a1l = a2l; a1h = a2h; n1 = n2;
            a2l = s6; a2h = 0; n2 = 0;
        }
        // spill-over into the next chunk: partial sums of limbs l0 + CH, + 1 (64-bit), + 2 (32-bit),
        // their carry counts and the carry count of this chunk's last limb
        __shared__ uint32_t s_pend[6][T];
        s_pend[0][tid] = a0l; s_pend[1][tid] = a0h; s_pend[2][tid] = a1l; s_pend[3][tid] = a1h;
        s_pend[4][tid] = a2l;
        s_pend[5][tid] = (uint32_t)n0 | ((uint32_t)n1 << 8) | ((uint32_t)((ecnt >> (4 * (CH - 1))) & 15u) << 16);
        if (tid < R) { s_neg[tid] = 0; s_zmin[tid] = INT_MAX; }
        __syncthreads();
        int e_prev = 0;  // carries into limb l0 from the previous chunk's last limb sum
        if (k > 0) {
            const int tp = tid - R;
            const uint32_t cn = s_pend[5][tp];
            const uint32_t pl[3] = {s_pend[0][tp], s_pend[2][tp], s_pend[4][tp]};
            const uint32_t ph[3] = {s_pend[1][tp], s_pend[3][tp], 0u};
            const int pn[3] = {(int)(cn & 255u), (int)((cn >> 8) & 255u), 0};
#pragma unroll
            for (int c = 0; c < 3 && c < CH; ++c) {
                uint32_t lo = (uint32_t)u[c], hi = (uint32_t)(u[c] >> 32);
                int cnt = (int)((ecnt >> (4 * c)) & 15u) + pn[c];
                add64_count(lo, hi, cnt, pl[c], ph[c]);
                u[c] = (uint64_t)hi << 32 | lo;
                ecnt = (ecnt & ~(15ull << (4 * c))) | ((uint64_t)cnt << (4 * c));
            }
            e_prev = (int)(cn >> 16);
        }
        // binary lookahead on w_c = v_c + e_(c-1): generate g_c (carry out) / propagate p_c
        // (w_c = 2^64 - 1); the chunk's (G, P) composes limbs 0 .. CH-1
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            uint32_t lo = (uint32_t)u[c], hi = (uint32_t)(u[c] >> 32);
            int g = 0;
            add64_count(lo, hi, g, (uint32_t)e_prev, 0u);
            const uint32_t pr = (lo & hi) == 0xffffffffu;
            u[c] = (uint64_t)hi << 32 | lo;
            gbits |= (uint32_t)g << c;
            pbits |= pr << c;
            Gt = (uint32_t)g | (pr & Gt);
            Pt &= pr;
            e_prev = (int)((ecnt >> (4 * c)) & 15u);
        }
    } else {
        // (c) v2: thread t owns limbs [k CH, k CH + CH) of row r = t % R (k = t / R).  Coefficient s
        // (unsigned C'' < M < 2^155, five words at its residue slot) sits at limb q(s) = floor(w s / 64)
        // shifted by w s mod 64 (w = 65: s = 64 a + b -> q = 65 a + b, shift b; w = 64: q = s).  The
        // thread walks positions q = l0 - 3 .. l0 + CH - 1 once, keeping the partial sums of the next
        // three limbs in registers: limb q is complete after the coefficient at q, and then gets -K's
        // limb.  u = limb value mod 2^64, e = carries out of those additions (<= 4, added to limb q + 1
        // below).
        const uint32_t *qmap = prm.qmap + l0;  // entry j: position qq = l0 - 3 + j (padded past Ly)
        const uint64_t *negk = prm.negK + l0;  // zero-padded past Ly
        // pending partial sums of limbs q, q + 1, q + 2 as 32-bit halves, and their carry counts
        uint32_t a0l = 0, a0h = 0, a1l = 0, a1h = 0, a2l = 0, a2h = 0;
        int n0 = 0, n1 = 0, n2 = 0;
        // Limb c of the chunk: v_c = its sum mod 2^64, e_c = carries out of that sum (<= 4).  Binary
        // lookahead on w_c = v_c + e_(c-1): w_c generates g_c (carry out) or propagates p_c
        // (w_c = 2^64 - 1); carry into c + 1 = g_c | (p_c & carry into c).  For c >= 1 e_(c-1) is this
        // thread's, so w_c, g_c, p_c are formed here; limb 0 waits for the previous chunk's e.
        uint32_t v0l = 0, v0h = 0;       // limb 0 before e_in
        int e_prev = 0;
#if HK_K3_SKIP & 4
#pragma unroll
        for (int c = 0; c < CH; ++c) u[c] = smr[c * R];
#pragma unroll
        for (int j = 0; j < 0; ++j) {
#else
#pragma unroll
        for (int j = 0; j < CH + 3; ++j) {
#endif
            const uint32_t qm = __ldg(qmap + j);
            const uint32_t o = qm >> 6, sh = qm & 63u;
            const uint32_t w0 = smr[o], w1 = smr[LY::PS + o], w2 = smr[2 * LY::PS + o],
                           w3 = smr[3 * LY::PS + o], w4 = smr[4 * LY::PS + o];
            const uint32_t bs = sh & 31u;
            const uint32_t h0 = w0 << bs, h1 = __funnelshift_l(w0, w1, bs), h2 = __funnelshift_l(w1, w2, bs),
                           h3 = __funnelshift_l(w2, w3, bs), h4 = __funnelshift_l(w3, w4, bs),
                           h5 = __funnelshift_l(w4, 0u, bs);
            const bool up = sh >= 32u;  // the image starts one 32-bit word higher
            const uint32_t s0 = sel32(up, 0u, h0), s1 = sel32(up, h0, h1), s2 = sel32(up, h1, h2),
                           s3 = sel32(up, h2, h3), s4 = sel32(up, h3, h4), s5 = sel32(up, h4, h5),
                           s6 = sel32(up, h5, 0u);
            add64_count(a0l, a0h, n0, s0, s1);  // limb q
            add64_count(a1l, a1h, n1, s2, s3);  // limb q + 1
            add64_count(a2l, a2h, n2, s4, s5);  // limb q + 2 (s6 -> limb q + 3, below)
            if (j >= 3) {  // limb l = qq is complete: add -K's limb
                const int c = j - 3;
                const uint64_t nk = __ldg(negk + c);
                add64_count(a0l, a0h, n0, (uint32_t)nk, (uint32_t)(nk >> 32));
                if (c == 0) {
                    v0l = a0l; v0h = a0h;
                } else {
                    int g = 0;
                    add64_count(a0l, a0h, g, (uint32_t)e_prev, 0u);
                    const uint32_t pr = (a0l & a0h) == 0xffffffffu;
                    u[c] = (uint64_t)a0h << 32 | a0l;
                    gbits |= (uint32_t)g << c;
                    pbits |= pr << c;
                    Gt = (uint32_t)g | (pr & Gt);
                    Pt &= pr;
                }
                e_prev = n0;
            }
            a0l = a1l; a0h = a1h; n0 = n1;
            a1l = a2l; a1h = a2h; n1 = n2;
            a2l = s6; a2h = 0; n2 = 0;
        }
        // the local carry count of the previous chunk's last limb (thread t - R) comes via smem
        __shared__ int8_t s_ecarry[T];
        s_ecarry[tid] = (int8_t)e_prev;
        if (tid < R) { s_neg[tid] = 0; s_zmin[tid] = INT_MAX; }
        __syncthreads();
        {  // limb 0 with the previous chunk's local carry; chunk (G, P) = (limbs 1..) o (limb 0)
            int g0 = 0;
            add64_count(v0l, v0h, g0, k > 0 ? (uint32_t)s_ecarry[tid - R] : 0u, 0u);
            const uint32_t p0 = (v0l & v0h) == 0xffffffffu;
            u[0] = (uint64_t)v0h << 32 | v0l;
            gbits |= (uint32_t)g0;
            pbits |= p0;
            Gt = Gt | (Pt & (uint32_t)g0);
            Pt &= p0;
        }
    }
    const int gp = (int)(Gt | (Pt << 1));  // (G, P) packed as bit 0 / 1
    // segmented scan over the chunks of each row (lanes r, r + R, ...): compose(later, earlier)
    auto gp_compose = [](int later, int earlier) {
        return ((later | ((later >> 1) & earlier)) & 1) | ((later & earlier) & 2);
    };
    int incl = gp;
#pragma unroll
    for (int off = R; off < 32; off <<= 1) {
        const int other = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl = gp_compose(incl, other);
    }
    if (lane >= 32 - R) s_wtot[warp * R + (lane - (32 - R))] = incl;  // per (warp, row) total
    __syncthreads();
#if HK_K3_WSCAN
    // carry into this warp's first chunk of row r: every thread folds the earlier warps' totals
    // itself (at most T / 32 - 1 of them) -- no serial pass by R threads and no second barrier
    int carry = 0;
    for (int wi = 0; wi < warp; ++wi) {
        const int t = s_wtot[wi * R + r];
        carry = (t & 1) | ((t >> 1) & carry);
    }
    const int prev = __shfl_up_sync(0xffffffffu, incl, R);
#else
    if (tid < R) {  // carry into each warp's first chunk of row tid
        int c = 0;
        for (int wi = 0; wi < T / 32; ++wi) {
            s_wcarry[wi * R + tid] = c;
            const int t = s_wtot[wi * R + tid];
            c = (t & 1) | ((t >> 1) & c);
        }
    }
    __syncthreads();
    const int prev = __shfl_up_sync(0xffffffffu, incl, R);
    int carry = s_wcarry[warp * R + r];
#endif
    if (lane_r > 0) carry = (prev & 1) | ((prev >> 1) & carry);
#pragma unroll
    for (int c = 0; c < CH; ++c) {  // final limbs (mod 2^(64 Ly))
        u[c] += (uint64_t)carry;
        carry = ((gbits >> c) & 1) | ((pbits >> c) & carry);
    }
    int zloc = INT_MAX;
#pragma unroll
    for (int c = CH - 1; c >= 0; --c) zloc = u[c] ? l0 + c : zloc;
    if (zloc < Ly) atomicMin(&s_zmin[r], zloc);
    if (l0 <= Ly - 1 && Ly - 1 < l0 + CH) {  // the row's top limb gives the sign
#pragma unroll
        for (int c = 0; c < CH; ++c)
            if (l0 + c == Ly - 1) s_neg[r] = (int)(u[c] >> 63);
    }
    __syncthreads();  // also: every CRT word has been read, the residue area is free
#else
    // (c) all R rows at once: thread t owns limbs [k CH, k CH + CH) of row r = t % R (k = t / R),
    // so the R rows' words of a coefficient are read by adjacent lanes.
    const int S2 = prm.S2, Ly = prm.Ly, w = prm.w;
    const int r = tid % R, k = tid / R, lane_r = lane / R;  // lane_r: position among the row's lanes
    const int64_t row = r0 + r;
    const int l0 = k * CH;
    // Sliding window over consecutive limbs: W[d] holds the shifted words S_0..S_3 and the sign of
    // the coefficient at limb index q = l - d, so every coefficient is read and shifted once.
    struct ShiftedCoef { uint64_t s0, s1, s2, s3; uint32_t neg; };
    auto load_coef = [&](int qq) -> ShiftedCoef {
        ShiftedCoef z = {0, 0, 0, 0, 0};
        if (qq < 0) return z;
        int sh;
        const int sidx = k3_coef_of_limb(qq, w, &sh);
        if (sidx < 0 || sidx >= S2) return z;
#if HK_K3_GARNER_SLOT
        const int cs = (N2 - sidx) & (N2 - 1);  // CRT words of coefficient sidx sit at its residue slot
#else
        const int cs = sidx;
#endif
        const uint64_t C0 = (uint64_t)sm[LY::idx(0, cs, r)] | ((uint64_t)sm[LY::idx(1, cs, r)] << 32);
        const uint64_t C1 = (uint64_t)sm[LY::idx(2, cs, r)] | ((uint64_t)sm[LY::idx(3, cs, r)] << 32);
        const uint32_t w4 = sm[LY::idx(4, cs, r)];
        const uint64_t C2 = (uint64_t)(int64_t)(int32_t)w4;   // sign-extended bits 128..159
        const uint64_t C3 = (uint64_t)((int64_t)C2 >> 63);      // sign word
        if (sh) {
            z.s0 = C0 << sh;
            z.s1 = (C1 << sh) | (C0 >> (64 - sh));
            z.s2 = (C2 << sh) | (C1 >> (64 - sh));
            z.s3 = (C3 << sh) | (C2 >> (64 - sh));
        } else {
            z.s0 = C0; z.s1 = C1; z.s2 = C2; z.s3 = C3;
        }
        z.neg = (uint32_t)(C3 & 1u);  // -1 at limb q + 4 (sign extension beyond S_3)
        return z;
    };
    ShiftedCoef W1 = load_coef(l0 - 1), W2 = load_coef(l0 - 2), W3 = load_coef(l0 - 3),
                W4 = load_coef(l0 - 4);
    uint64_t u[CH];
    int e[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int l = l0 + c;
        uint64_t acc = 0;
        int hi = 0;
        if (l < Ly) {
            const ShiftedCoef W0 = load_coef(l);
            acc = W0.s0;
            acc += W1.s1; hi += acc < W1.s1;
            acc += W2.s2; hi += acc < W2.s2;
            acc += W3.s3; hi += acc < W3.s3;
            hi -= (int)(W4.neg & (acc == 0));
            acc -= W4.neg;
            W4 = W3; W3 = W2; W2 = W1; W1 = W0;
        }
        u[c] = acc;
        e[c] = hi;  // carry into limb l + 1, in [-1, 3]
    }
    // the carry out of the previous chunk of the same row (thread t - R) comes via smem
    __shared__ int8_t s_ecarry[T];
    __shared__ int s_neg[R], s_zmin[R];
    s_ecarry[tid] = (int8_t)e[CH - 1];
    if (tid < R) { s_neg[tid] = 0; s_zmin[tid] = INT_MAX; }
    __syncthreads();
    int F = kTfId;
    int fl[CH];
    int ein = k > 0 ? (int)s_ecarry[tid - R] : 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
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
    // segmented scan of transfer functions over the chunks of each row (lanes r, r + R, ...)
    int incl = F;
#pragma unroll
    for (int off = R; off < 32; off <<= 1) {
        const int other = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl = tf_compose(incl, other);
    }
    if (lane >= 32 - R) s_wtot[warp * R + (lane - (32 - R))] = incl;  // per (warp, row) total
    __syncthreads();
    if (tid < R) {  // carry into each warp's first chunk of row tid
        int c = 0;
        for (int wi = 0; wi < T / 32; ++wi) {
            s_wcarry[wi * R + tid] = c;
            c = tf_apply(s_wtot[wi * R + tid], c);
        }
    }
    __syncthreads();
    const int prev = __shfl_up_sync(0xffffffffu, incl, R);
    int carry = s_wcarry[warp * R + r];
    if (lane_r > 0) carry = tf_apply(prev, carry);
    int zloc = INT_MAX;
#pragma unroll
    for (int c = 0; c < CH; ++c) {  // final limbs (mod 2^(64 Ly))
        const uint64_t v = u[c] + (uint64_t)(int64_t)carry;
        carry = tf_apply(fl[c], carry);
        u[c] = v;
        if (l0 + c < Ly && v && zloc == INT_MAX) zloc = l0 + c;
        if (l0 + c == Ly - 1) s_neg[r] = (int)(v >> 63);
    }
    if (zloc != INT_MAX) atomicMin(&s_zmin[r], zloc);
    __syncthreads();  // also: every CRT word has been read, the residue area is free
#endif
    uint64_t *ybuf = reinterpret_cast<uint64_t *>(sm);  // [R][Ly]
    {  // two's complement -> magnitude: -Y = ~Y + 1, the + 1 rippling through the zero limbs
       // below the lowest nonzero one (zmin): limb l -> (l <= zmin) + ~v
        const bool neg = s_neg[r] != 0;
        const int zmin = s_zmin[r];
        const uint64_t m = neg ? ~0ull : 0ull;
        uint64_t *yb = ybuf + r * Ly + l0;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (l0 + c < Ly) yb[c] = (u[c] ^ m) + (uint64_t)(neg && l0 + c <= zmin);
        }
    }
    __syncthreads();
#if HK_K3_FLAT_STORE
    if (HK_K3_SKIP & 16) {
        if (tid < R && ybuf[tid] == 12345) y_mag[tid] = 1;
    } else if (!prm.round_out) {
        // the R rows' limbs as one flat range (R Ly / T rounds instead of R ceil(Ly / T)); (rr, l)
        // advance incrementally (no division; T may exceed Ly for small P)
        const int nr = (int)(m - r0 < R ? m - r0 : R);
        const int ndst = prm.p2p ? (1 << prm.shard_gamma) : 1;  // peer memory: every rank's y
        for (int d = 0; d < ndst; ++d) {
            uint64_t *ybase = prm.p2p ? prm.peer_ymag[d] : y_mag;
            int rr = 0, l = tid;
            while (l >= Ly) { l -= Ly; ++rr; }
            auto row_ptr = [&](int q) {
                const int64_t o = r0 + q;
                return ybase + (prm.reverse_out ? (prm.y_rows - 1 - o) : o) * Ly;
            };
            uint64_t *yo = row_ptr(rr);
            for (; rr < nr;) {
                yo[l] = ybuf[rr * Ly + l];
                l += T;
                if (l >= Ly) {
                    do { l -= Ly; ++rr; } while (l >= Ly);
                    yo = row_ptr(rr);
                }
            }
            if (tid < nr) {
                const int64_t o = r0 + tid;
                const int64_t orow = prm.reverse_out ? (prm.y_rows - 1 - o) : o;
                (prm.p2p ? prm.peer_ysign[d] : y_sign)[orow] =
                    s_neg[tid] ? (int8_t)-1 : (s_zmin[tid] < Ly ? (int8_t)1 : (int8_t)0);
            }
        }
    } else {
        for (int rr = 0; rr < R && r0 + rr < m; ++rr) {
            const int64_t o = r0 + rr;
            k3_store_rounded(prm, ybuf + (size_t)rr * Ly, s_neg[rr] != 0,
                             prm.reverse_out ? (prm.y_rows - 1 - o) : o, y_mag, y_sign);
        }
    }
#else
    for (int rr = 0; rr < R; ++rr) {
        const int64_t orow_r = r0 + rr;
        if (orow_r >= m) break;
        const int64_t orow = prm.reverse_out ? (prm.y_rows - 1 - orow_r) : orow_r;
        if (!prm.round_out) {
            const int8_t sgn = s_neg[rr] ? (int8_t)-1 : (s_zmin[rr] < Ly ? (int8_t)1 : (int8_t)0);
            // peer-memory exchange: the y all-gather fused into the stores (every rank's y buffer)
            const int ndst = prm.p2p ? (1 << prm.shard_gamma) : 1;
            for (int d = 0; d < ndst; ++d) {
                uint64_t *yo = (prm.p2p ? prm.peer_ymag[d] : y_mag) + orow * Ly;
                for (int l = tid; l < Ly; l += T) yo[l] = ybuf[rr * Ly + l];
                if (tid == 0) (prm.p2p ? prm.peer_ysign[d] : y_sign)[orow] = sgn;
            }
        } else {
            k3_store_rounded(prm, ybuf + (size_t)rr * Ly, s_neg[rr] != 0, orow, y_mag, y_sign);
        }
    }
#endif
    if (prm.p2p) __threadfence_system();  // peer y stores visible before the next barrier
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

template <int LOGN2, int GAMMA>
static int launch_rows_g(const Params &prm0, cudaStream_t st, int tile0, int ntiles) {
    const int ga = (int)((prm0.a_count + kK1Rows - 1) / kK1Rows);
    const int gx = (int)((prm0.n + kK1Rows - 1) / kK1Rows);
    if (ntiles < 0) ntiles = ga + gx - tile0;
    if (ntiles <= 0) return HK_OK;
    Params prm = prm0;
    prm.tile0 = tile0;
    const size_t tab_bytes = (size_t)2 * (1 << LOGN2) * sizeof(uint2);  // 2 twiddle tables
    const size_t smem1 = (size_t)k1_transform_words(k1_row_stride<LOGN2>(), prm.L) * sizeof(uint32_t) + tab_bytes;
    if (ensure_smem((const void *)k1_slice_rowntt<LOGN2, GAMMA>, smem1)) return HK_ECUDA;
    // a launch under one wave (3 CTAs per SM) runs one prime per CTA: 5x the CTAs, each slicing
    // its tile again (C1: 24 tiles -> 120 CTAs)
    static int nsm = 0;
    if (nsm == 0) {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            nsm = v;
        else
            return HK_ECUDA;
    }
    prm.k1_prime_split = (int64_t)ntiles * prm.nvec * kNumPrimes <= (int64_t)k1_minb<LOGN2>() * nsm ? 1 : 0;
    k1_slice_rowntt<LOGN2, GAMMA><<<dim3((unsigned)ntiles, (unsigned)prm.nvec, prm.k1_prime_split ? kNumPrimes : 1),
                                     k1_threads<LOGN2>(), smem1, st>>>(prm, ga);
    return check_launch();
}

template <int LOGN2>
static int launch_rows(const Params &prm, cudaStream_t st, int tile0 = 0, int ntiles = -1) {
    if (prm.slice_mode) return launch_rows_g<LOGN2, -1>(prm, st, tile0, ntiles);  // full slice transform
    switch (prm.shard_gamma) {
        case 0: return launch_rows_g<LOGN2, 0>(prm, st, tile0, ntiles);
        case 1: if constexpr (LOGN2 >= 6) return launch_rows_g<LOGN2, 1>(prm, st, tile0, ntiles); break;
        case 2: if constexpr (LOGN2 >= 7) return launch_rows_g<LOGN2, 2>(prm, st, tile0, ntiles); break;
        case 3: if constexpr (LOGN2 >= 8) return launch_rows_g<LOGN2, 3>(prm, st, tile0, ntiles); break;
    }
    return HK_EUNSUPPORTED;
}

template <int LOGN1, int MODE>
static int launch_cols_m(const Params &prm, cudaStream_t st) {
    const int ncols = kNumPrimes * prm.n2loc;
    const size_t smem = k2_smem_bytes<LOGN1>();
    if (ensure_smem((const void *)k2_column<LOGN1, TwGlobal, MODE>, smem)) return HK_ECUDA;
    k2_column<LOGN1, TwGlobal, MODE><<<ncols, k2_threads<LOGN1>(), smem, st>>>(prm);
    return check_launch();
}
template <int LOGN1, int MODE>
static int launch_cols_mode(const Params &prm, cudaStream_t st);

template <int LOGN1>
static int launch_cols(const Params &prm, cudaStream_t st) {
    if constexpr (LOGN1 >= kSplitLogN1) {  // A^ transform -> AT, then X^ transform x AT + inverse
        if (!prm.split_k2 || !prm.AT) return HK_EINVAL;
        // AT now holds this call's A^: a prepared matrix kept in this workspace is gone
        if (cudaMemsetAsync(&prm.hdr->a_ready, 0, sizeof(int32_t), st) != cudaSuccess) return HK_ECUDA;
        int rc = launch_cols_mode<LOGN1, 1>(prm, st);
        if (rc) return rc;
        return prm.shard_rpr ? launch_cols_mode<LOGN1, 4>(prm, st) : launch_cols_mode<LOGN1, 2>(prm, st);
    } else {
        return prm.shard_rpr ? launch_cols_m<LOGN1, 3>(prm, st) : launch_cols_m<LOGN1, 0>(prm, st);
    }
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
    const int ncols = kNumPrimes * prm.n2loc * (MODE == 2 ? prm.nvec : 1);
    const size_t smem = (size_t)padded_len(1 << LOGN1) * sizeof(uint32_t);
    if (ensure_smem((const void *)k2_column<LOGN1, TwGlobal, MODE>, smem)) return HK_ECUDA;
    k2_column<LOGN1, TwGlobal, MODE><<<ncols, k2_threads<LOGN1>(), smem, st>>>(prm);
    return check_launch();
}

int launch_k2_sliced(const Params &prm, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    switch (prm.log_n1) {
#define HK_CASE(LG) case LG: return launch_cols_m<LG, 5>(prm, st);
        HK_CASE(6) HK_CASE(7) HK_CASE(8) HK_CASE(9) HK_CASE(10) HK_CASE(11) HK_CASE(12)
        HK_CASE(13) HK_CASE(14)
#undef HK_CASE
        default: return HK_EUNSUPPORTED;
    }
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

__global__ void k_set_a_ready(WsHeader *hdr) {
    if (hdr->magic == kWsMagic) hdr->a_ready = hdr->status == HK_OK ? 1 : 0;
}
int launch_set_a_ready(const Params &prm, void *stream) {
    k_set_a_ready<<<1, 1, 0, (cudaStream_t)stream>>>(prm.hdr);
    return check_launch();
}

int k1_tile_rows() { return kK1Rows; }
int k3_tile_rows(int log_n2) { return log_n2 >= 11 ? 2 : HK_K3_ROWS; }
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

template <int LOGN2, int CH>
static int launch_k3(const Params &prm, cudaStream_t st, int64_t nrows) {
    const size_t ybytes = (size_t)k3_rows<LOGN2>() * prm.Ly * sizeof(uint64_t);  // y rows reuse the area
    const size_t rbytes = K3Layout<LOGN2>::res_words() * sizeof(uint32_t);
    const size_t smem = rbytes > ybytes ? rbytes : ybytes;
    if (ensure_smem((const void *)k3_finish<LOGN2, CH>, smem)) return HK_ECUDA;
    const unsigned grid = (unsigned)((nrows + k3_rows<LOGN2>() - 1) / k3_rows<LOGN2>());
    k3_finish<LOGN2, CH><<<dim3(grid, (unsigned)prm.nvec), k3_threads<LOGN2>(), smem, st>>>(prm);
    return check_launch();
}

// limbs per thread reachable for a slice length 2^LOGN2 (the planner picks the smallest N2 with
// 2 ceil(P / w) - 1 <= N2, w in {64, 65}; Ly = 2 ceil(P / 64) + 1 <= kK3MaxLy): only these are built
// (Ly from about N2 / 2 + 1 up to 2 ceil(65 (N2 / 2) / 64) + 1, over TR = threads per row)
template <int LOGN2> constexpr int k3_tr() { return k3_threads<LOGN2>() / k3_rows<LOGN2>(); }
template <int LOGN2> constexpr int k3_ch_lo() {
    return LOGN2 <= 6 ? 1 : (((1 << LOGN2) / 2 + 1 + k3_tr<LOGN2>() - 1) / k3_tr<LOGN2>() - 1 < 1
                                 ? 1 : ((1 << LOGN2) / 2 + 1 + k3_tr<LOGN2>() - 1) / k3_tr<LOGN2>() - 1);
}
template <int LOGN2> constexpr int k3_ch_hi() {
    return ((1 << LOGN2) * 65 / 64 + 3 + k3_tr<LOGN2>() - 1) / k3_tr<LOGN2>();
}
template <int LOGN2, int C>
static int k3_dispatch(const Params &prm, cudaStream_t st, int64_t nrows, int ch) {
    if constexpr (C > k3_ch_hi<LOGN2>()) {
        return HK_EUNSUPPORTED;
    } else {
        if (ch == C) return launch_k3<LOGN2, C>(prm, st, nrows);
        return k3_dispatch<LOGN2, C + 1>(prm, st, nrows, ch);
    }
}
template <int LOGN2>
static int launch_k3_ch(const Params &prm, cudaStream_t st, int64_t nrows) {
    constexpr int TR = k3_threads<LOGN2>() / k3_rows<LOGN2>();  // threads per row
    const int ch = (prm.Ly + TR - 1) / TR;
    if (ch < k3_ch_lo<LOGN2>()) return HK_EUNSUPPORTED;
    return k3_dispatch<LOGN2, k3_ch_lo<LOGN2>()>(prm, st, nrows, ch);
}

int launch_k3_range(const Params &prm0, void *stream, int64_t row0, int64_t nrows) {
    if (nrows <= 0) return HK_OK;
    cudaStream_t st = (cudaStream_t)stream;
    Params prm = prm0;
    prm.row0 = row0;
    switch (prm.log_n2) {
#define HK_CASE(LG) case LG: return launch_k3_ch<LG>(prm, st, nrows);
        HK_CASE(5) HK_CASE(6) HK_CASE(7) HK_CASE(8) HK_CASE(9) HK_CASE(10) HK_CASE(11)
#undef HK_CASE
        default: return HK_EUNSUPPORTED;
    }
}

}  // namespace hk
