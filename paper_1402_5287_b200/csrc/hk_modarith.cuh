// hk_modarith.cuh -- 31-bit prime-field arithmetic and shared-memory NTT passes for sm_100a.
//
// The exact 2-D convolution runs over k = 5 primes p < 2^31 with
// 2^17 | p - 1, so every power-of-two transform length up to 2^17 has a root of unity.
// Residues are kept fully reduced in [0, p): with p < 2^31 the sum of two residues fits in
// 32 bits, the difference plus p as well, so no 64-bit arithmetic appears in a butterfly.
//
//   Shoup product  x*W mod p with W' = floor(W 2^32 / p):  q = hi(x W'), r = x W - q p in [0, 2p)
//                  (3 IMAD; valid for every 32-bit x)
//   Montgomery     a*b*2^-32 mod p (a, b < p):            3 IMAD (IMAD.WIDE + IMAD + IMAD.WIDE)
//   GS butterfly   (u, v) -> (u + v, (u - v) W)            forward DIF, natural -> bit-reversed
//   CT butterfly   (u, v) -> (u + v W, u - v W)            inverse DIT, bit-reversed -> natural
#pragma once
#include <cstdint>

#define HK_DEV __device__ __forceinline__

namespace hk {

constexpr int kPrimes = 5;
// p = c * 2^17 + 1 < 2^31, the five largest such primes; log2(prod) = 154.993
constexpr uint32_t kP[kPrimes] = {2147352577u, 2146959361u, 2146041857u, 2144468993u,
                                  2142502913u};

// Padded shared-memory index: one spare word after every 32 keeps the strided radix passes
// (stride S = 1..16 between a thread's points) free of bank conflicts.
HK_DEV int pad(int i) { return i + (i >> 5); }
HK_DEV unsigned padu(unsigned i) { return i + (i >> 5); }
__host__ __device__ constexpr int padded_len(int n) { return n + (n >> 5); }

HK_DEV uint32_t red1(uint32_t x, uint32_t p) { return min(x, x - p); }  // [0,2p) -> [0,p)
HK_DEV uint32_t addm(uint32_t a, uint32_t b, uint32_t p) {                // [0,p)^2 -> [0,p)
    uint32_t s = a + b;
    return min(s, s - p);
}
HK_DEV uint32_t subm(uint32_t a, uint32_t b, uint32_t p) {                // [0,p)^2 -> [0,p)
    uint32_t d = a - b;
    return min(d, d + p);
}
HK_DEV uint32_t shoup(uint32_t x, uint32_t w, uint32_t wq, uint32_t p) {  // -> [0, 2p)
    uint32_t q = __umulhi(x, wq);
    return x * w - q * p;
}
HK_DEV uint32_t mont(uint32_t a, uint32_t b, uint32_t p, uint32_t pneg) { // a b 2^-32, [0,p)
    uint64_t z = (uint64_t)a * b;
    uint32_t m = (uint32_t)z * pneg;
    uint64_t t = z + (uint64_t)m * p;  // < 2^64 since a, b < p < 2^31
    return red1((uint32_t)(t >> 32), p);
}

// Gentleman-Sande (DIF) butterfly, inputs/outputs in [0, p).
HK_DEV void gs_bfly(uint32_t &u, uint32_t &v, uint2 w, uint32_t p) {
    uint32_t d = u - v + p;  // [1, 2p)
    u = addm(u, v, p);
    v = red1(shoup(d, w.x, w.y, p), p);
}
// Cooley-Tukey (DIT) butterfly, inputs/outputs in [0, p).
HK_DEV void ct_bfly(uint32_t &u, uint32_t &v, uint2 w, uint32_t p) {
    uint32_t t = red1(shoup(v, w.x, w.y, p), p);
    v = subm(u, t, p);
    u = addm(u, t, p);
}

// 4-byte asynchronous global -> shared copy (LDGSTS); completes at cp_async_wait_all().
HK_DEV void cp_async4(uint32_t *smem, const uint32_t *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
HK_DEV void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
HK_DEV void cp_async8(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
HK_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
HK_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>  // wait until at most N committed groups are still in flight
HK_DEV void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// TMA bulk copy (non-tensor) of a contiguous global range into shared memory, completing on an
// mbarrier (sm_90+ async proxy).  dst / src 16-byte aligned, bytes a multiple of 16.
HK_DEV void mbar_init(uint64_t *mbar, unsigned count) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
HK_DEV void bulk_copy_g2s(void *dst, const void *src, unsigned bytes, uint64_t *mbar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(mbar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
}
HK_DEV void mbar_wait_parity(uint64_t *mbar, unsigned parity) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(mbar);
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
            : "=r"(done)
            : "r"(b), "r"(parity)
            : "memory");
    }
}

// Butterfly with twiddle omega^0 = 1 (GS and CT coincide): no multiplication.
HK_DEV void bfly1(uint32_t &u, uint32_t &v, uint32_t p) {
    const uint32_t d = subm(u, v, p);
    u = addm(u, v, p);
    v = d;
}

// Twiddle-load policies: the table lives in global memory (read-only path) or shared memory.
struct TwGlobal {
    static HK_DEV uint2 ld(const uint2 *t, int i) { return __ldg(t + i); }
};
struct TwShared {
    static HK_DEV uint2 ld(const uint2 *t, int i) { return t[i]; }
};

// ------------------------------------------------------------------------------------------
// Shared-memory NTT over `batch` arrays of N = 2^LOGN points: array b, point i lives at
// s[b * rs + pad(i)].  Twiddle table tw[h + j] = (omega_{2h}^{+-j}, Shoup quotient) for every
// half-size h = 1, 2, ..., N/2 and j < h (index 0 unused), read through the read-only path.
//
// A radix-2^R pass holds G = 2^R points x[B + j0 + m S] (m < G) of one group in registers and
// runs R consecutive radix-2 stages on them; S is the smallest half-size of the pass.  Every
// stage of the pass pairs m with m + 2^l and uses twiddle index h + j0 + S (m mod 2^l),
// h = S 2^l (the plain radix-2 DIF/DIT indexing, just blocked).
//
// Only FORWARD tables are used.  The DIT network run with the forward roots computes the
// forward DFT of its bit-reversed input; applied to DIF(x) it returns N * x[(-i) mod N], i.e. the
// inverse transform with the output index negated -- callers read position (N - i) mod N.

// Forward DIF pass: stages h = S 2^(R-1) ... S.  ZERO_UPPER: the array's upper half is known to
// be zero (only legal for the first pass, S G = N).
template <class TW, int LOGN, int R, int S, bool ZERO_UPPER>
HK_DEV void dif_pass(uint32_t *s, int batch, int rs, const uint2 *__restrict__ tw, uint32_t p,
                     int tid, int nthr) {
    constexpr int N = 1 << LOGN;
    constexpr int G = 1 << R;
    constexpr int NG = N / G;
    static_assert(!ZERO_UPPER || S * G == N, "ZERO_UPPER only for the first pass");
    const unsigned total = (unsigned)(batch * NG);
    for (unsigned gi = tid; gi < total; gi += nthr) {
        const unsigned b = gi / NG;
        const unsigned g = gi % NG;
        const unsigned j0 = g % S;
        const unsigned B = (g / S) * (S * G);
        // pad(B + j0 + m S) = pad(B + j0) + pad(m S): B is a multiple of S G and S G | 32 or 32 | S G,
        // so the low part never carries into bit 5 -- the per-point offset is an immediate
        uint32_t *base = s + b * rs + padu(B + j0);
        uint32_t v[G];
#pragma unroll
        for (int m = 0; m < G; ++m) {
            if (ZERO_UPPER && m >= G / 2) v[m] = 0;
            else v[m] = base[padded_len(m * S)];
        }
#pragma unroll
        for (int l = R - 1; l >= 0; --l) {
            const int half = 1 << l;
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & half) continue;
                if (S == 1 && (m & (half - 1)) == 0) {  // j = 0: twiddle 1
                    bfly1(v[m], v[m + half], p);
                    continue;
                }
                const unsigned j = j0 + S * (m & (half - 1));
                const uint2 w = TW::ld(tw, S * half + j);
                gs_bfly(v[m], v[m + half], w, p);
            }
        }
#pragma unroll
        for (int m = 0; m < G; ++m) base[padded_len(m * S)] = v[m];
    }
    __syncthreads();
}

// Inverse DIT pass: stages h = S, 2S, ..., S 2^(R-1).
template <class TW, int LOGN, int R, int S>
HK_DEV void dit_pass(uint32_t *s, int batch, int rs, const uint2 *__restrict__ tw, uint32_t p,
                     int tid, int nthr) {
    constexpr int N = 1 << LOGN;
    constexpr int G = 1 << R;
    constexpr int NG = N / G;
    const unsigned total = (unsigned)(batch * NG);
    for (unsigned gi = tid; gi < total; gi += nthr) {
        const unsigned b = gi / NG;
        const unsigned g = gi % NG;
        const unsigned j0 = g % S;
        const unsigned B = (g / S) * (S * G);
        uint32_t *base = s + b * rs + padu(B + j0);  // see dif_pass
        uint32_t v[G];
#pragma unroll
        for (int m = 0; m < G; ++m) v[m] = base[padded_len(m * S)];
#pragma unroll
        for (int l = 0; l < R; ++l) {
            const int half = 1 << l;
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & half) continue;
                if (S == 1 && (m & (half - 1)) == 0) {  // j = 0: twiddle 1
                    bfly1(v[m], v[m + half], p);
                    continue;
                }
                const unsigned j = j0 + S * (m & (half - 1));
                const uint2 w = TW::ld(tw, S * half + j);
                ct_bfly(v[m], v[m + half], w, p);
            }
        }
#pragma unroll
        for (int m = 0; m < G; ++m) base[padded_len(m * S)] = v[m];
    }
    __syncthreads();
}

// Full forward transform: passes of RMAX stages from the top (HI = number of stages left).
template <class TW, int LOGN, int HI, int RMAX, bool FIRST>
struct DifPasses {
    static HK_DEV void run(uint32_t *s, int batch, int rs, const uint2 *tw, uint32_t p, int tid,
                           int nthr, bool zero_upper) {
        constexpr int R = HI < RMAX ? HI : RMAX;
        constexpr int S = 1 << (HI - R);
        if (FIRST && zero_upper)
            dif_pass<TW, LOGN, R, S, FIRST>(s, batch, rs, tw, p, tid, nthr);
        else
            dif_pass<TW, LOGN, R, S, false>(s, batch, rs, tw, p, tid, nthr);
        DifPasses<TW, LOGN, HI - R, RMAX, false>::run(s, batch, rs, tw, p, tid, nthr, false);
    }
};
template <class TW, int LOGN, int RMAX, bool FIRST>
struct DifPasses<TW, LOGN, 0, RMAX, FIRST> {
    static HK_DEV void run(uint32_t *, int, int, const uint2 *, uint32_t, int, int, bool) {}
};

template <class TW, int LOGN, int LO, int RMAX>
struct DitPasses {
    static HK_DEV void run(uint32_t *s, int batch, int rs, const uint2 *tw, uint32_t p, int tid,
                           int nthr) {
        constexpr int LEFT = LOGN - LO;
        constexpr int R = LEFT < RMAX ? LEFT : RMAX;
        dit_pass<TW, LOGN, R, (1 << LO)>(s, batch, rs, tw, p, tid, nthr);
        DitPasses<TW, LOGN, LO + R, RMAX>::run(s, batch, rs, tw, p, tid, nthr);
    }
};
template <class TW, int LOGN, int RMAX>
struct DitPasses<TW, LOGN, LOGN, RMAX> {
    static HK_DEV void run(uint32_t *, int, int, const uint2 *, uint32_t, int, int) {}
};

// Forward DIF (natural -> bit-reversed).
template <class TW, int LOGN, int RMAX>
HK_DEV void ntt_forward(uint32_t *s, int batch, int rs, const uint2 *tw, uint32_t p, int tid,
                        int nthr, bool zero_upper) {
    DifPasses<TW, LOGN, LOGN, RMAX, true>::run(s, batch, rs, tw, p, tid, nthr, zero_upper);
}
// DIT with the forward table (bit-reversed -> natural, output index negated; see above).
template <class TW, int LOGN, int RMAX>
HK_DEV void ntt_dit_fwdroots(uint32_t *s, int batch, int rs, const uint2 *tw, uint32_t p,
                             int tid, int nthr) {
    DitPasses<TW, LOGN, 0, RMAX>::run(s, batch, rs, tw, p, tid, nthr);
}

}  // namespace hk
