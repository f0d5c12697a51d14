// hk_api.cu -- the C ABI of include/hk.h: planner (exact-capacity proof), workspace layout,
// argument validation and launch sequencing.  Host code only; kernels live in hk_ntt.cu and
// hk_schoolbook.cu.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "hk_internal.h"

namespace hk {
namespace {

constexpr uint32_t kPrimesHost[kNumPrimes] = {2147352577u, 2146959361u, 2146041857u,
                                              2144468993u, 2142502913u};

uint32_t mulmod(uint32_t a, uint32_t b, uint32_t p) { return (uint32_t)(((uint64_t)a * b) % p); }
uint32_t powmod(uint32_t b, uint64_t e, uint32_t p) {
    uint32_t r = 1 % p;
    b %= p;
    while (e) {
        if (e & 1) r = mulmod(r, b, p);
        b = mulmod(b, b, p);
        e >>= 1;
    }
    return r;
}
uint32_t invmod(uint32_t a, uint32_t p) { return powmod(a, p - 2, p); }  // p prime
uint32_t shoup_q(uint32_t w, uint32_t p) { return (uint32_t)(((uint64_t)w << 32) / p); }

uint32_t primitive_root(uint32_t p) {
    std::vector<uint32_t> fac;
    uint32_t r = p - 1;
    for (uint32_t d = 2; (uint64_t)d * d <= r; ++d)
        if (r % d == 0) {
            fac.push_back(d);
            while (r % d == 0) r /= d;
        }
    if (r > 1) fac.push_back(r);
    for (uint32_t g = 2;; ++g) {
        bool ok = true;
        for (uint32_t q : fac)
            if (powmod(g, (p - 1) / q, p) == 1) { ok = false; break; }
        if (ok) return g;
    }
}

// ---- tiny exact big-integer helpers for the capacity proof (little-endian u32 limbs)
using Big = std::vector<uint32_t>;
Big big_from(uint64_t v) { return Big{(uint32_t)v, (uint32_t)(v >> 32)}; }
Big big_mul(const Big &a, const Big &b) {
    Big r(a.size() + b.size(), 0);
    for (size_t i = 0; i < a.size(); ++i) {
        uint64_t c = 0;
        for (size_t j = 0; j < b.size(); ++j) {
            uint64_t t = (uint64_t)a[i] * b[j] + r[i + j] + c;
            r[i + j] = (uint32_t)t;
            c = t >> 32;
        }
        r[i + b.size()] += (uint32_t)c;
    }
    return r;
}
int big_cmp(Big a, Big b) {
    while (a.size() < b.size()) a.push_back(0);
    while (b.size() < a.size()) b.push_back(0);
    for (size_t i = a.size(); i-- > 0;)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}
Big big_pow2_minus1(int w) {  // 2^w - 1
    Big r((w + 31) / 32 + 1, 0);
    for (int b = 0; b < w; ++b) r[b / 32] |= 1u << (b % 32);
    return r;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

int make_plan_uncached(int32_t kind, int64_t m, int64_t n, int32_t P, uint32_t flags, Plan *pl, int32_t G) {
    if (kind < HK_HANKEL || kind > HK_CIRCULANT || n < 1 || m < 1 || P < 1) return HK_EINVAL;
    if (kind != HK_HANKEL && m != n) return HK_EINVAL;
    std::memset(pl, 0, sizeof(*pl));
    hk_plan_info &in = pl->info;
    in.kind = kind;
    in.P = P;
    in.m = m;
    in.n = n;
    in.L = (P + 63) / 64;
    in.Ly = 2 * in.L + 1;
    in.k_primes = kNumPrimes;
    in.a_count = kind == HK_CIRCULANT ? n : m + n - 1;
    if (in.Ly > kK3MaxLy) return HK_EUNSUPPORTED;
    // matrix-index transform length
    int64_t need;
    if (kind == HK_CIRCULANT) {
        const bool pow2 = (n & (n - 1)) == 0;
        if (pow2 && n >= (1 << kMinLogN1)) {
            in.cyclic = 1;
            need = n;
        } else {
            in.fold = 1;
            need = 2 * n - 1;
        }
        pl->x_reversed = 0;
        pl->out_off = 0;
    } else {
        need = in.a_count;
        pl->x_reversed = 1;
        pl->out_off = n - 1;
    }
    pl->reverse_out = kind == HK_TOEPLITZ;
    int lg1 = kMinLogN1;
    while ((int64_t(1) << lg1) < need) ++lg1;
    if (lg1 > kMaxLogN1) return HK_EUNSUPPORTED;
    in.log_n1 = lg1;
    // slice width / slice transform: smallest N2 with an exact plan
    Big M = big_from(1);
    for (int k = 0; k < kNumPrimes; ++k) M = big_mul(M, big_from(kPrimesHost[k]));
    double logM = 0;
    for (int k = 0; k < kNumPrimes; ++k) logM += std::log2((double)kPrimesHost[k]);
    bool found = false;
    // Smallest N2 first; for it the widest slice w in {65, 64} that satisfies the capacity bound.
    // w >= 64 makes the limb index floor(w s / 64) of coefficient s injective, which the carry
    // kernel (K3) relies on.
    for (int lg2 = kMinLogN2; lg2 <= kMaxLogN2 && !found; ++lg2) {
        for (int64_t w = kMaxW; w >= 64 && !found; --w) {
            const int64_t Ls = (P + w - 1) / w;
            if (2 * Ls - 1 > (int64_t(1) << lg2)) continue;
            Big wm = big_pow2_minus1((int)w);
            Big B = big_mul(big_mul(wm, wm), big_mul(big_from((uint64_t)(2 * n)), big_from((uint64_t)Ls)));
            if (big_cmp(B, M) < 0) {
                in.w = (int32_t)w;
                in.Ls = (int32_t)Ls;
                in.log_n2 = lg2;
                in.margin_bits = logM - (1.0 + std::log2((double)n) + std::log2((double)Ls) +
                                         2.0 * std::log2(std::ldexp(1.0, (int)w) - 1.0));
                found = true;
            }
        }
    }
    if (!found) return HK_EUNSUPPORTED;
    // sigma-coset shards: G = 2^gamma <= 8 blocks of the slice transform (N2 / G >= 32)
    if (G < 1 || G > 8 || (G & (G - 1)) || (int64_t(1) << in.log_n2) / G < 32) return HK_EUNSUPPORTED;
    pl->G = G;
    pl->gamma = G == 1 ? 0 : (G == 2 ? 1 : (G == 4 ? 2 : 3));
    pl->rpr = G == 1 ? 0 : ((m + G - 1) / G + 3) / 4 * 4;
    const int64_t N2 = int64_t(1) << in.log_n2;
    const int64_t N2loc = N2 / G;
    const int64_t N1 = int64_t(1) << in.log_n1;
    // A^ / X^ columns: zero-padded up to the extent K2's top pass loads (N1 / 2 when the count fits
    // in the lower half, else N1); K1 writes rows < count only and hk_workspace_init zeroes the rest
    pl->ldA = in.a_count <= N1 / 2 ? N1 / 2 : N1;
    pl->ldX = n <= N1 / 2 ? N1 / 2 : N1;
    pl->ldY = (m + 31) / 32 * 32;
    size_t off = align256(sizeof(WsHeader));
    pl->off_tw = off;
    off = align256(off + (size_t)kNumPrimes * (N1 + N2) * sizeof(uint2));
    pl->off_negK = off;  // K3 v2 tables, padded by kK3TablePad entries past Ly (no bound checks)
    off = align256(off + (size_t)(in.Ly + kK3TablePad) * sizeof(uint64_t));
    pl->off_qmap = off;
    off = align256(off + (size_t)(in.Ly + 3 + kK3TablePad) * sizeof(uint32_t));
    pl->off_A = off;
    off = align256(off + (size_t)kNumPrimes * N2loc * pl->ldA * 4);
    pl->off_X = off;
    off = align256(off + (size_t)kNumPrimes * N2loc * pl->ldX * 4);
    pl->off_Y = off;  // sharded: K2 writes the caller's all-to-all send buffer instead
    if (G == 1) off = align256(off + (size_t)kNumPrimes * N2 * pl->ldY * 4);
    // N1 >= 2^15: K2 runs as two launches (A^'s column transform to AT, then X^'s transform x AT
    // + inverse), since one thread cannot hold N1 / 512 = 64 X^ values beside its working set
    const size_t at_bytes = (size_t)kNumPrimes * N2loc * N1 * 4;
    pl->split_k2 = in.log_n1 >= kSplitLogN1;
    if (pl->split_k2) {
        pl->off_AT = off;
        off = align256(off + at_bytes);
    }
    pl->off_end = off;
    pl->off_stage = off;
    const size_t L = in.L, Ly = in.Ly;
    pl->st_amag = off;  off = align256(off + (size_t)in.a_count * L * 8);
    pl->st_asign = off; off = align256(off + (size_t)in.a_count);
    pl->st_xmag = off;  off = align256(off + (size_t)n * L * 8);
    pl->st_xsign = off; off = align256(off + (size_t)n);
    pl->st_ymag = off;  off = align256(off + (size_t)m * Ly * 8);
    pl->st_ysign = off; off = align256(off + (size_t)m);
    pl->off_end_staging = off;
    // HK_WS_PREPARED: the 2-D transform of a right after the base layout (already inside it when
    // K2 is split)
    if (!pl->split_k2) pl->off_AT = pl->off_end;
    pl->off_end_prepared = pl->split_k2 ? pl->off_end : align256(pl->off_AT + at_bytes);
    if (G > 1) {  // sliced sharding: each rank slices ldA / G positions of a and ldX / G of x
        pl->rs_a = pl->ldA / G;
        pl->rs_x = pl->ldX / G;
        pl->slice_ok = in.log_n1 <= 14 && pl->rs_a >= 8 && pl->rs_x >= 8 &&
                       (pl->rs_a & (pl->rs_a - 1)) == 0 && (pl->rs_x & (pl->rs_x - 1)) == 0;
        pl->slice_chunk = (int64_t)kNumPrimes * N2loc * (pl->rs_a + pl->rs_x);
    }
    pl->xhat_bytes = align256((size_t)kNumPrimes * N2loc * pl->ldX * 4);
    pl->yhat_bytes = align256((size_t)kNumPrimes * N2 * pl->ldY * 4);
    in.ws_bytes = pl->off_end;
    in.ws_bytes_staging = pl->off_end_staging;
    in.ws_bytes_prepared = pl->off_end_prepared;
    if ((flags & HK_WS_STAGING) && (flags & HK_WS_PREPARED)) return HK_EINVAL;
    if (flags & ~(HK_WS_STAGING | HK_WS_PREPARED)) return HK_EINVAL;
    return HK_OK;
}

// Plans are pure functions of (kind, m, n, P, flags, G): the last 16 are kept, so a repeated call
// skips the capacity search (big-integer bounds) on the host.
int make_plan(int32_t kind, int64_t m, int64_t n, int32_t P, uint32_t flags, Plan *pl, int32_t G = 1) {
    struct Key {
        int32_t kind;
        int64_t m, n;
        int32_t P;
        uint32_t flags;
        int32_t G;
        bool operator==(const Key &o) const {
            return kind == o.kind && m == o.m && n == o.n && P == o.P && flags == o.flags && G == o.G;
        }
    };
    constexpr int kCache = 16;
    static std::mutex mu;
    static Key keys[kCache];
    static Plan plans[kCache];
    static int rcs[kCache];
    static int used = 0, next = 0;
    const Key key{kind, m, n, P, flags, G};
    {
        std::lock_guard<std::mutex> lk(mu);
        for (int k = 0; k < used; ++k)
            if (keys[k] == key) {
                *pl = plans[k];
                return rcs[k];
            }
    }
    const int rc = make_plan_uncached(kind, m, n, P, flags, pl, G);
    std::lock_guard<std::mutex> lk(mu);
    keys[next] = key;
    plans[next] = *pl;
    rcs[next] = rc;
    next = (next + 1) % kCache;
    if (used < kCache) ++used;
    return rc;
}

uint64_t plan_hash(int32_t kind, int64_t m, int64_t n, int32_t P, int32_t G = 1) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) {
        for (int i = 0; i < 8; ++i) { h ^= (v >> (8 * i)) & 0xff; h *= 1099511628211ull; }
    };
    mix((uint64_t)kind); mix((uint64_t)m); mix((uint64_t)n); mix((uint64_t)P);
    if (G != 1) mix(0x5348415244ull + (uint64_t)G);  // "SHARD" + G
    return h;
}

void fill_params(const Plan &pl, void *ws, Params *prm) {
    std::memset(prm, 0, sizeof(*prm));
    const hk_plan_info &in = pl.info;
    prm->kind = in.kind; prm->P = in.P; prm->L = in.L; prm->Ly = in.Ly;
    prm->m = in.m; prm->n = in.n; prm->a_count = in.a_count;
    prm->w = in.w; prm->Ls = in.Ls; prm->S2 = 2 * in.Ls - 1;
    prm->log_n1 = in.log_n1; prm->log_n2 = in.log_n2;
    prm->N1 = 1 << in.log_n1; prm->N2 = 1 << in.log_n2;
    prm->cyclic = in.cyclic; prm->fold = in.fold;
    prm->reverse_out = pl.reverse_out; prm->x_reversed = pl.x_reversed;
    prm->out_off = pl.out_off;
    prm->ldA = pl.ldA; prm->ldX = pl.ldX; prm->ldY = pl.ldY;
    prm->nvec = 1;
    prm->n2loc = prm->N2 / pl.G;
    prm->log_n2loc = in.log_n2 - pl.gamma;
    prm->shard_gamma = pl.gamma;
    prm->shard_rpr = pl.rpr;
    prm->y_rows = pl.G == 1 ? in.m : (int64_t)pl.G * pl.rpr;
    prm->hash = plan_hash(in.kind, in.m, in.n, in.P, pl.G);
    char *base = (char *)ws;
    prm->hdr = (WsHeader *)base;
    prm->tw = (const uint2 *)(base + pl.off_tw);
    prm->negK = (const uint64_t *)(base + pl.off_negK);
    prm->qmap = (const uint32_t *)(base + pl.off_qmap);
    prm->Ahat = (uint32_t *)(base + pl.off_A);
    prm->Xhat = (uint32_t *)(base + pl.off_X);
    prm->AT = pl.split_k2 ? (uint32_t *)(base + pl.off_AT) : nullptr;
    prm->split_k2 = pl.split_k2;
    prm->Yhat = (uint32_t *)(base + pl.off_Y);
    const uint64_t N12 = (uint64_t)prm->N1 * (uint64_t)prm->N2;
    for (int k = 0; k < kNumPrimes; ++k) {
        const uint32_t p = kPrimesHost[k];
        PrimeConsts &c = prm->pc[k];
        c.p = p;
        uint32_t inv = 1;  // Newton: p^-1 mod 2^32
        for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
        c.pneg = 0u - inv;
        const uint32_t r32 = (uint32_t)((uint64_t(1) << 32) % p);
        const uint32_t r64 = mulmod(r32, r32, p);
        const uint32_t f = mulmod(r32, invmod((uint32_t)(N12 % p), p), p);  // 2^32 (N1 N2)^-1
        const uint32_t wa[3] = {1u, r32, r64};
        for (int d = 0; d < 3; ++d) {
            c.fa[d] = wa[d];
            c.fa_q[d] = shoup_q(wa[d], p);
            c.fx[d] = mulmod(wa[d], f, p);
            c.fx_q[d] = shoup_q(c.fx[d], p);
        }
    }
    {
        Big Mb = big_from(1);
        for (int k = 0; k < kNumPrimes; ++k) {
            Mb = big_mul(Mb, big_from(kPrimesHost[k]));
            prm->gc.half[k] = (kPrimesHost[k] - 1) / 2;
        }
        for (int k = 0; k < kNumPrimes; ++k) prm->gc.M[k] = k < (int)Mb.size() ? Mb[k] : 0u;
    }
    for (int j = 0; j < kNumPrimes; ++j)
        for (int k = 0; k < kNumPrimes; ++k) {
            if (j >= k) continue;
            const uint32_t v = invmod(kPrimesHost[j] % kPrimesHost[k], kPrimesHost[k]);
            prm->gc.inv[j][k] = v;
            prm->gc.inv_q[j][k] = shoup_q(v, kPrimesHost[k]);
        }
    // K3 v2: ascending prime order (kPrimesHost is descending), H = (M - 1) / 2 mod p_g
    Garner2Consts &g2 = prm->g2;
    for (int g = 0; g < kNumPrimes; ++g) {
        g2.kp[g] = (uint32_t)(kNumPrimes - 1 - g);
        g2.p[g] = kPrimesHost[g2.kp[g]];
    }
    // M = 0 mod p_g, so H = (M - 1) / 2 = -1 / 2 = (p_g - 1) / 2 (mod p_g)
    for (int g = 0; g < kNumPrimes; ++g) g2.h[g] = (g2.p[g] - 1) / 2;
    for (int j = 0; j < kNumPrimes; ++j)
        for (int g = 0; g < kNumPrimes; ++g) {
            g2.c[j][g] = g2.cq[j][g] = 0;
            if (j >= g) continue;
            const uint32_t v = invmod(g2.p[j] % g2.p[g], g2.p[g]);
            g2.c[j][g] = v;
            g2.cq[j][g] = shoup_q(v, g2.p[g]);
        }
}

// -K mod 2^(64 Ly), K = H sum_{s < S2} 2^(w s), H = (M - 1) / 2 (K3 v2; little-endian u64 limbs)
std::vector<uint64_t> neg_k_limbs(int32_t w, int32_t S2, int32_t Ly) {
    Big Mb = big_from(1);
    for (int k = 0; k < kNumPrimes; ++k) Mb = big_mul(Mb, big_from(kPrimesHost[k]));
    Big H(Mb.size(), 0);  // (M - 1) / 2: M odd, so shift right by one
    for (size_t i = 0; i < Mb.size(); ++i) {
        const uint32_t hi = i + 1 < Mb.size() ? Mb[i + 1] : 0u;
        H[i] = (Mb[i] >> 1) | (hi << 31);
    }
    const size_t NW = (size_t)2 * Ly;  // u32 words of the result
    std::vector<uint32_t> acc(NW, 0);
    for (int64_t s = 0; s < S2; ++s) {
        const int64_t bit = (int64_t)w * s;
        const int64_t w0 = bit >> 5;
        const int sh = (int)(bit & 31);
        if ((size_t)w0 >= NW) break;
        uint64_t carry = 0;
        for (size_t i = 0; (size_t)w0 + i < NW; ++i) {
            const uint64_t lo = i < H.size() ? H[i] : 0u;
            const uint64_t prev = (i >= 1 && i - 1 < H.size()) ? H[i - 1] : 0u;
            const uint32_t word = sh ? (uint32_t)((lo << sh) | (prev >> (32 - sh))) : (uint32_t)lo;
            const uint64_t t = (uint64_t)acc[w0 + i] + word + carry;
            acc[w0 + i] = (uint32_t)t;
            carry = t >> 32;
            if (i > H.size() && carry == 0) break;
        }
    }
    std::vector<uint64_t> out(Ly + kK3TablePad, 0);
    uint64_t borrow = 1;  // two's complement: ~K + 1 (a carry, despite the name)
    for (int32_t l = 0; l < Ly; ++l) {
        const uint64_t v = ~((uint64_t)acc[2 * l] | ((uint64_t)acc[2 * l + 1] << 32));
        const uint64_t r = v + borrow;
        borrow = (borrow && r == 0) ? 1 : 0;
        out[l] = r;
    }
    return out;
}

// Twiddle tables + header (K0), and zeros in the A^ / X^ arrays: their column padding beyond the
// entry count is never written by K1 and must read as zero in K2 (see ldA / ldX in make_plan).
// K3 v2 limb -> coefficient map: limb qq holds coefficient s with
// floor(w s / 64) = qq (w = 65: qq = 65 a + b, s = 64 a + b, b < 64; w = 64: s = qq) shifted by
// w s mod 64; its CRT words sit at residue slot (N2 - s) mod N2 of K3's shared layout (word offset
// pad(slot) R for row 0).  Limbs with no coefficient point at slot 1 (s = N2 - 1 >= S2), which K3
// zeroes.  Entry qq + 3 for qq = -3 .. Ly - 1.
std::vector<uint32_t> k3_qmap(const hk_plan_info &in) {
    const int64_t N2 = int64_t(1) << in.log_n2, R = k3_tile_rows(in.log_n2);
    const int64_t S2 = 2 * (int64_t)in.Ls - 1;
    auto padw = [](int64_t i) { return i + (i >> 5); };
    std::vector<uint32_t> q((size_t)in.Ly + 3 + kK3TablePad);
    for (int64_t qq = -3; qq < in.Ly + kK3TablePad; ++qq) {
        int64_t slot = 1, sh = 0;
        if (qq >= 0) {
            int64_t s = qq, b = 0;
            if (in.w == 65) { const int64_t a = qq / 65; b = qq - 65 * a; s = 64 * a + b; }
            if (qq < in.Ly && b < 64 && s < S2) {
                slot = (N2 - s) & (N2 - 1);
                sh = in.w == 65 ? b : 0;
            }
        }
        q[(size_t)(qq + 3)] = (uint32_t)((padw(slot) * R) << 6 | sh);
    }
    return q;
}

int init_workspace(const Plan &pl, const Params &prm, void *ws, void *stream) {
    if (cudaMemsetAsync((char *)ws + pl.off_A, 0, pl.off_Y - pl.off_A, (cudaStream_t)stream) != cudaSuccess)
        return HK_ECUDA;
    // -K table of K3 v2 (pageable source: the copy is staged before cudaMemcpyAsync returns)
    const std::vector<uint64_t> nk = neg_k_limbs(pl.info.w, 2 * pl.info.Ls - 1, pl.info.Ly);
    const std::vector<uint32_t> qm = k3_qmap(pl.info);
    if (cudaMemcpyAsync((char *)ws + pl.off_negK, nk.data(), nk.size() * sizeof(uint64_t),
                        cudaMemcpyHostToDevice, (cudaStream_t)stream) != cudaSuccess ||
        cudaMemcpyAsync((char *)ws + pl.off_qmap, qm.data(), qm.size() * sizeof(uint32_t),
                        cudaMemcpyHostToDevice, (cudaStream_t)stream) != cudaSuccess)
        return HK_ECUDA;
    uint32_t gens[kNumPrimes];
    for (int k = 0; k < kNumPrimes; ++k) gens[k] = primitive_root(kPrimesHost[k]);
    return launch_init(prm, gens, stream);
}

// Copy streams and events of the synchronous host-buffer call (hk_matvec_host), created once per
// device and reused across calls (a call takes a context from the pool and returns it before it
// returns; concurrent calls get distinct contexts).  Host-side handles only: no device memory.
struct HostCtx {
    static constexpr int kEvents = 24;
    int device;
    cudaStream_t s1, s2;
    cudaEvent_t ev[kEvents];
};
std::mutex g_host_mu;
std::vector<HostCtx *> g_host_pool;

HostCtx *acquire_host_ctx() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    {
        std::lock_guard<std::mutex> lk(g_host_mu);
        for (size_t i = 0; i < g_host_pool.size(); ++i)
            if (g_host_pool[i]->device == dev) {
                HostCtx *c = g_host_pool[i];
                g_host_pool.erase(g_host_pool.begin() + (long)i);
                return c;
            }
    }
    HostCtx *c = new HostCtx();
    c->device = dev;
    bool ok = cudaStreamCreateWithFlags(&c->s1, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->s2, cudaStreamNonBlocking) == cudaSuccess;
    for (int i = 0; ok && i < HostCtx::kEvents; ++i)
        ok = cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        delete c;  // handles of a failed creation are leaked rather than destroyed half-made
        return nullptr;
    }
    return c;
}
void release_host_ctx(HostCtx *c) {
    std::lock_guard<std::mutex> lk(g_host_mu);
    g_host_pool.push_back(c);
}

bool overlaps(const void *a, size_t na, const void *b, size_t nb) {
    const char *pa = (const char *)a, *pb = (const char *)b;
    return pa < pb + nb && pb < pa + na;
}

int run_matvec(int32_t kind, int64_t m, int64_t n, int32_t P, const uint64_t *a_mag,
               const int8_t *a_sign, const uint64_t *x_mag, const int8_t *x_sign,
               uint64_t *y_mag, int8_t *y_sign, void *ws, size_t ws_bytes, void *stream,
               uint32_t stages = HK_STAGE_ALL, bool rounded = false) {
    if (!a_mag || !a_sign || !x_mag || !x_sign || !y_mag || !y_sign || !ws) return HK_EINVAL;
    if ((((uintptr_t)a_mag | (uintptr_t)x_mag) & 15) != 0) return HK_EINVAL;  // 16-byte staging
    Plan pl;
    int rc = make_plan(kind, m, n, P, 0, &pl);
    if (rc) return rc;
    if (((uintptr_t)ws & 255) != 0) return HK_EINVAL;
    if (ws_bytes < pl.info.ws_bytes) return HK_ENOMEM;
    const size_t L = pl.info.L, Ly = rounded ? pl.info.L + 1 : pl.info.Ly;
    const size_t ya = (size_t)m * Ly * 8, ys = (size_t)m;
    const size_t aa = (size_t)pl.info.a_count * L * 8, as = (size_t)pl.info.a_count;
    const size_t xa = (size_t)n * L * 8, xs = (size_t)n;
    if (overlaps(y_mag, ya, a_mag, aa) || overlaps(y_mag, ya, x_mag, xa) ||
        overlaps(y_sign, ys, a_sign, as) || overlaps(y_sign, ys, x_sign, xs) ||
        overlaps(y_mag, ya, y_sign, ys) || overlaps(y_mag, ya, ws, pl.info.ws_bytes) ||
        overlaps(y_sign, ys, ws, pl.info.ws_bytes))
        return HK_EINVAL;
    Params prm;
    fill_params(pl, ws, &prm);
    prm.a_mag = a_mag; prm.a_sign = a_sign; prm.x_mag = x_mag; prm.x_sign = x_sign;
    prm.y_mag = y_mag; prm.y_sign = y_sign;
    prm.round_out = rounded ? 1 : 0;
    if ((stages & HK_STAGE_SLICE_ROWS) &&
        cudaMemsetAsync(&prm.hdr->status, 0, sizeof(int32_t), (cudaStream_t)stream) != cudaSuccess)
        return HK_ECUDA;
    return launch_ntt_path(prm, stream, stages);
}

}  // namespace
}  // namespace hk

using namespace hk;

extern "C" {

int32_t hk_limbs(int32_t P) { return P < 1 ? -1 : (P + 63) / 64; }
int32_t hk_out_limbs(int32_t P) { return P < 1 ? -1 : 2 * ((P + 63) / 64) + 1; }

const char *hk_status_string(int32_t s) {
    switch (s) {
        case HK_OK: return "HK_OK";
        case HK_EINVAL: return "HK_EINVAL: invalid argument or workspace";
        case HK_ERANGE: return "HK_ERANGE: non-canonical input data";
        case HK_ENOMEM: return "HK_ENOMEM: workspace too small";
        case HK_EUNSUPPORTED: return "HK_EUNSUPPORTED: no exact plan within limits";
        case HK_ECUDA: return "HK_ECUDA: CUDA error";
        default: return "unknown hk_status";
    }
}

int32_t hk_plan(int32_t kind, int64_t m, int64_t n, int32_t P, hk_plan_info *out) {
    if (!out) return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, m, n, P, 0, &pl);
    if (rc) return rc;
    *out = pl.info;
    return HK_OK;
}

int32_t hk_workspace_size(int32_t kind, int64_t m, int64_t n, int32_t P, uint32_t flags,
                          size_t *bytes) {
    if (!bytes) return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, m, n, P, flags, &pl);
    if (rc) return rc;
    *bytes = (flags & HK_WS_STAGING) ? pl.info.ws_bytes_staging
             : (flags & HK_WS_PREPARED) ? pl.info.ws_bytes_prepared : pl.info.ws_bytes;
    return HK_OK;
}

int32_t hk_workspace_init(int32_t kind, int64_t m, int64_t n, int32_t P, uint32_t flags,
                          void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_workspace_init");
    if (!ws || ((uintptr_t)ws & 255) != 0) return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, m, n, P, flags, &pl);
    if (rc) return rc;
    const size_t need = (flags & HK_WS_STAGING) ? pl.info.ws_bytes_staging
                        : (flags & HK_WS_PREPARED) ? pl.info.ws_bytes_prepared : pl.info.ws_bytes;
    if (ws_bytes < need) return HK_ENOMEM;
    Params prm;
    fill_params(pl, ws, &prm);
    return init_workspace(pl, prm, ws, stream);
}

// ---- F1 kernel-level batch: a prepared workspace followed by nvec X^ regions and nvec Y^ regions
int32_t hk_batch_workspace_size(int32_t kind, int64_t m, int64_t n, int32_t P, int32_t nvec,
                                size_t *bytes) {
    if (!bytes || nvec < 1) return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, m, n, P, HK_WS_PREPARED, &pl);
    if (rc) return rc;
    *bytes = pl.info.ws_bytes_prepared + (size_t)nvec * (pl.xhat_bytes + pl.yhat_bytes);
    return HK_OK;
}

int32_t hk_batch_workspace_init(int32_t kind, int64_t m, int64_t n, int32_t P, int32_t nvec,
                                void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_batch_workspace_init");
    if (!ws || ((uintptr_t)ws & 255) != 0 || nvec < 1) return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, m, n, P, HK_WS_PREPARED, &pl);
    if (rc) return rc;
    const size_t need = pl.info.ws_bytes_prepared + (size_t)nvec * (pl.xhat_bytes + pl.yhat_bytes);
    if (ws_bytes < need) return HK_ENOMEM;
    Params prm;
    fill_params(pl, ws, &prm);
    if ((rc = init_workspace(pl, prm, ws, stream))) return rc;
    // the vectors' X^ columns are zero-padded past n rows (K2's top pass reads ldX rows)
    if (cudaMemsetAsync((char *)ws + pl.info.ws_bytes_prepared, 0, (size_t)nvec * pl.xhat_bytes,
                        (cudaStream_t)stream) != cudaSuccess)
        return HK_ECUDA;
    return HK_OK;
}

int32_t hk_matvec_prepared_batch(int32_t kind, int64_t m, int64_t n, int32_t P, int32_t nvec,
                                 const uint64_t *x_mag, const int8_t *x_sign, uint64_t *y_mag,
                                 int8_t *y_sign, void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_matvec_prepared_batch");
    if (!x_mag || !x_sign || !y_mag || !y_sign || !ws || ((uintptr_t)ws & 255) != 0 ||
        ((uintptr_t)x_mag & 15) != 0 || nvec < 1 || nvec > 65535)
        return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, m, n, P, HK_WS_PREPARED, &pl);
    if (rc) return rc;
    // capacity of the workspace (its X^ regions come first, then its Y^ regions): from ws_bytes,
    // which must be the size the workspace was initialised with
    if (ws_bytes < pl.info.ws_bytes_prepared) return HK_ENOMEM;
    const size_t cap = (ws_bytes - pl.info.ws_bytes_prepared) / (pl.xhat_bytes + pl.yhat_bytes);
    if (cap < (size_t)nvec) return HK_ENOMEM;
    const size_t need = pl.info.ws_bytes_prepared + cap * (pl.xhat_bytes + pl.yhat_bytes);
    const size_t Ly = pl.info.Ly, L = pl.info.L, V = (size_t)nvec;
    if (((n * L * 8) & 15) != 0 && nvec > 1) return HK_EINVAL;  // every vector 16-byte aligned
    if (overlaps(y_mag, V * m * Ly * 8, x_mag, V * n * L * 8) || overlaps(y_sign, V * m, x_sign, V * n) ||
        overlaps(y_mag, V * m * Ly * 8, ws, need) || overlaps(y_sign, V * m, ws, need))
        return HK_EINVAL;
    Params prm;
    fill_params(pl, ws, &prm);
    prm.x_mag = x_mag; prm.x_sign = x_sign; prm.y_mag = y_mag; prm.y_sign = y_sign;
    prm.AT = (uint32_t *)((char *)ws + pl.off_AT);
    prm.Xhat = (uint32_t *)((char *)ws + pl.info.ws_bytes_prepared);
    prm.Yhat = (uint32_t *)((char *)ws + pl.info.ws_bytes_prepared + cap * pl.xhat_bytes);
    prm.nvec = nvec;
    prm.x_vstride = n;
    prm.y_vstride = m;
    prm.need_a_ready = 1;
    if (pl.xhat_bytes != (size_t)kNumPrimes * prm.n2loc * prm.ldX * 4 ||
        pl.yhat_bytes != (size_t)kNumPrimes * prm.N2 * prm.ldY * 4)
        return HK_EUNSUPPORTED;  // vector regions must continue the column index (256-byte multiples)
    if (cudaMemsetAsync(&prm.hdr->status, 0, sizeof(int32_t), (cudaStream_t)stream) != cudaSuccess)
        return HK_ECUDA;
    const int ga = k1_tiles_a(prm);
    if ((rc = launch_k1_range(prm, stream, ga, k1_tiles_x(prm)))) return rc;
    if ((rc = launch_k2_mode(prm, stream, 2))) return rc;
    return launch_k3_range(prm, stream, 0, m);
}

int32_t hk_workspace_status(void *ws, void *stream, int32_t *data_status) {
    if (!ws || !data_status) return HK_EINVAL;
    int32_t v = HK_ECUDA;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemcpyAsync(&v, &((WsHeader *)ws)->status, sizeof(v), cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return HK_ECUDA;
    *data_status = v;
    return HK_OK;
}

int32_t hk_hankel_matvec(int64_t n, int32_t P, const uint64_t *a_mag, const int8_t *a_sign,
                         const uint64_t *x_mag, const int8_t *x_sign, uint64_t *y_mag,
                         int8_t *y_sign, void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_hankel_matvec");
    return run_matvec(HK_HANKEL, n, n, P, a_mag, a_sign, x_mag, x_sign, y_mag, y_sign, ws,
                      ws_bytes, stream);
}

int32_t hk_toeplitz_matvec(int64_t n, int32_t P, const uint64_t *a_mag, const int8_t *a_sign,
                           const uint64_t *x_mag, const int8_t *x_sign, uint64_t *y_mag,
                           int8_t *y_sign, void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_toeplitz_matvec");
    return run_matvec(HK_TOEPLITZ, n, n, P, a_mag, a_sign, x_mag, x_sign, y_mag, y_sign, ws,
                      ws_bytes, stream);
}

int32_t hk_circulant_matvec(int64_t n, int32_t P, const uint64_t *c_mag, const int8_t *c_sign,
                            const uint64_t *x_mag, const int8_t *x_sign, uint64_t *y_mag,
                            int8_t *y_sign, void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_circulant_matvec");
    return run_matvec(HK_CIRCULANT, n, n, P, c_mag, c_sign, x_mag, x_sign, y_mag, y_sign, ws,
                      ws_bytes, stream);
}

int32_t hk_matvec_rounded(int32_t kind, int64_t m, int64_t n, int32_t P, const uint64_t *a_mag,
                          const int8_t *a_sign, const uint64_t *x_mag, const int8_t *x_sign,
                          uint64_t *y_mag, int8_t *y_sign, void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_matvec_rounded");
    return run_matvec(kind, m, n, P, a_mag, a_sign, x_mag, x_sign, y_mag, y_sign, ws, ws_bytes,
                      stream, HK_STAGE_ALL, true);
}

int32_t hk_hankel_rect_matvec(int64_t m, int64_t n, int32_t P, const uint64_t *a_mag,
                              const int8_t *a_sign, const uint64_t *x_mag, const int8_t *x_sign,
                              uint64_t *y_mag, int8_t *y_sign, void *ws, size_t ws_bytes,
                              void *stream) {
    HK_NVTX("hk_hankel_rect_matvec");
    return run_matvec(HK_HANKEL, m, n, P, a_mag, a_sign, x_mag, x_sign, y_mag, y_sign, ws,
                      ws_bytes, stream);
}

int32_t hk_matvec_host(int32_t kind, int64_t m, int64_t n, int32_t P, const uint64_t *a_mag_host,
                       const int8_t *a_sign_host, const uint64_t *x_mag_host,
                       const int8_t *x_sign_host, uint64_t *y_mag_host, int8_t *y_sign_host,
                       void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_matvec_host");
    if (!a_mag_host || !a_sign_host || !x_mag_host || !x_sign_host || !y_mag_host ||
        !y_sign_host || !ws)
        return HK_EINVAL;
    if (((uintptr_t)ws & 255) != 0) return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, m, n, P, HK_WS_STAGING, &pl);
    if (rc) return rc;
    if (ws_bytes < pl.info.ws_bytes_staging) return HK_ENOMEM;
    // Pipeline (all stream-ordered, host synchronises once at the end):
    //   s1: H2D of x then a in chunks  ->  s0: K1 over the tiles of each chunk as it lands
    //   s0: K2  ->  K3 per chunk of output rows  ->  s2: D2H of that chunk of y
    cudaStream_t s0 = (cudaStream_t)stream;
    HostCtx *ctx = acquire_host_ctx();
    if (!ctx) return HK_ECUDA;
    cudaStream_t s1 = ctx->s1, s2 = ctx->s2;
    int nev = 0;
    auto cleanup = [&]() { release_host_ctx(ctx); };
    auto new_event = [&]() -> cudaEvent_t { return nev < HostCtx::kEvents ? ctx->ev[nev++] : nullptr; };
    char *base = (char *)ws;
    const size_t L = pl.info.L, Ly = pl.info.Ly, na = pl.info.a_count;
    uint64_t *d_am = (uint64_t *)(base + pl.st_amag);
    int8_t *d_as = (int8_t *)(base + pl.st_asign);
    uint64_t *d_xm = (uint64_t *)(base + pl.st_xmag);
    int8_t *d_xs = (int8_t *)(base + pl.st_xsign);
    uint64_t *d_ym = (uint64_t *)(base + pl.st_ymag);
    int8_t *d_ys = (int8_t *)(base + pl.st_ysign);
    Params prm;
    fill_params(pl, ws, &prm);
    prm.a_mag = d_am; prm.a_sign = d_as; prm.x_mag = d_xm; prm.x_sign = d_xs;
    prm.y_mag = d_ym; prm.y_sign = d_ys;
    bool ok = true;
    cudaEvent_t e0 = new_event();
    ok = ok && e0 && cudaEventRecord(e0, s0) == cudaSuccess &&
         cudaStreamWaitEvent(s1, e0, 0) == cudaSuccess && cudaStreamWaitEvent(s2, e0, 0) == cudaSuccess;
    ok = ok && cudaMemsetAsync(&prm.hdr->status, 0, sizeof(int32_t), s0) == cudaSuccess;
    const int ga = k1_tiles_a(prm), gx = k1_tiles_x(prm);
    const int kTile = k1_tile_rows();
    struct Chunk { int t0, nt; };
    Chunk chunks[6];
    int nch = 0;
    for (int c = 0; c < 2; ++c) {  // x first (smaller), then a
        const int t0 = ga + gx * c / 2, t1 = ga + gx * (c + 1) / 2;
        if (t1 > t0) chunks[nch++] = {t0, t1 - t0};
    }
    for (int c = 0; c < 4; ++c) {
        const int t0 = ga * c / 4, t1 = ga * (c + 1) / 4;
        if (t1 > t0) chunks[nch++] = {t0, t1 - t0};
    }
    for (int c = 0; c < nch && ok; ++c) {
        const bool is_x = chunks[c].t0 >= ga;
        const int64_t cnt = is_x ? n : (int64_t)na;
        const int64_t r0 = (int64_t)(chunks[c].t0 - (is_x ? ga : 0)) * kTile;
        int64_t r1 = r0 + (int64_t)chunks[c].nt * kTile;
        if (r1 > cnt) r1 = cnt;
        const uint64_t *hm = is_x ? x_mag_host : a_mag_host;
        const int8_t *hs = is_x ? x_sign_host : a_sign_host;
        uint64_t *dm = is_x ? d_xm : d_am;
        int8_t *dsg = is_x ? d_xs : d_as;
        ok = cudaMemcpyAsync(dm + r0 * L, hm + r0 * L, (r1 - r0) * L * 8, cudaMemcpyHostToDevice,
                             s1) == cudaSuccess &&
             cudaMemcpyAsync(dsg + r0, hs + r0, r1 - r0, cudaMemcpyHostToDevice, s1) == cudaSuccess;
        cudaEvent_t e = new_event();
        ok = ok && e && cudaEventRecord(e, s1) == cudaSuccess &&
             cudaStreamWaitEvent(s0, e, 0) == cudaSuccess;
        if (ok && (rc = launch_k1_range(prm, s0, chunks[c].t0, chunks[c].nt))) { cleanup(); return rc; }
    }
    if (ok && (rc = launch_ntt_path(prm, s0, HK_STAGE_COLUMNS))) { cleanup(); return rc; }
    const int ncy = m >= 64 ? 4 : 1;
    for (int c = 0; c < ncy && ok; ++c) {
        int64_t r0 = m * c / ncy / 8 * 8, r1 = c + 1 == ncy ? m : m * (c + 1) / ncy / 8 * 8;
        if (r1 <= r0) continue;
        if ((rc = launch_k3_range(prm, s0, r0, r1 - r0))) { cleanup(); return rc; }
        // y rows of this chunk (Toeplitz writes rows reversed: m-1-r)
        const int64_t o0 = pl.reverse_out ? m - r1 : r0, o1 = pl.reverse_out ? m - r0 : r1;
        cudaEvent_t e = new_event();
        ok = e && cudaEventRecord(e, s0) == cudaSuccess && cudaStreamWaitEvent(s2, e, 0) == cudaSuccess &&
             cudaMemcpyAsync(y_mag_host + o0 * Ly, d_ym + o0 * Ly, (o1 - o0) * Ly * 8,
                             cudaMemcpyDeviceToHost, s2) == cudaSuccess &&
             cudaMemcpyAsync(y_sign_host + o0, d_ys + o0, o1 - o0, cudaMemcpyDeviceToHost, s2) ==
                 cudaSuccess;
    }
    cudaEvent_t ed = new_event();
    ok = ok && ed && cudaEventRecord(ed, s2) == cudaSuccess && cudaStreamWaitEvent(s0, ed, 0) == cudaSuccess;
    int32_t ds = HK_ECUDA;
    rc = ok ? hk_workspace_status(ws, stream, &ds) : HK_ECUDA;
    cleanup();
    if (rc) return rc;
    return ds;
}

int32_t hk_matvec_host_async(int32_t kind, int64_t m, int64_t n, int32_t P,
                             const uint64_t *a_mag_host, const int8_t *a_sign_host,
                             const uint64_t *x_mag_host, const int8_t *x_sign_host,
                             uint64_t *y_mag_host, int8_t *y_sign_host, int32_t *status_host,
                             void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_matvec_host_async");
    if (!a_mag_host || !a_sign_host || !x_mag_host || !x_sign_host || !y_mag_host ||
        !y_sign_host || !status_host || !ws)
        return HK_EINVAL;
    if (((uintptr_t)ws & 255) != 0) return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, m, n, P, HK_WS_STAGING, &pl);
    if (rc) return rc;
    if (ws_bytes < pl.info.ws_bytes_staging) return HK_ENOMEM;
    cudaStream_t s = (cudaStream_t)stream;
    char *base = (char *)ws;
    const size_t L = pl.info.L, Ly = pl.info.Ly, na = pl.info.a_count;
    Params prm;
    fill_params(pl, ws, &prm);
    prm.a_mag = (const uint64_t *)(base + pl.st_amag);
    prm.a_sign = (const int8_t *)(base + pl.st_asign);
    prm.x_mag = (const uint64_t *)(base + pl.st_xmag);
    prm.x_sign = (const int8_t *)(base + pl.st_xsign);
    prm.y_mag = (uint64_t *)(base + pl.st_ymag);
    prm.y_sign = (int8_t *)(base + pl.st_ysign);
    const cudaMemcpyKind h2d = cudaMemcpyHostToDevice, d2h = cudaMemcpyDeviceToHost;
    if (cudaMemsetAsync(&prm.hdr->status, 0, sizeof(int32_t), s) != cudaSuccess ||
        cudaMemcpyAsync((void *)prm.x_mag, x_mag_host, (size_t)n * L * 8, h2d, s) != cudaSuccess ||
        cudaMemcpyAsync((void *)prm.x_sign, x_sign_host, (size_t)n, h2d, s) != cudaSuccess ||
        cudaMemcpyAsync((void *)prm.a_mag, a_mag_host, na * L * 8, h2d, s) != cudaSuccess ||
        cudaMemcpyAsync((void *)prm.a_sign, a_sign_host, na, h2d, s) != cudaSuccess)
        return HK_ECUDA;
    if ((rc = launch_ntt_path(prm, stream, HK_STAGE_ALL))) return rc;
    if (cudaMemcpyAsync(y_mag_host, prm.y_mag, (size_t)m * Ly * 8, d2h, s) != cudaSuccess ||
        cudaMemcpyAsync(y_sign_host, prm.y_sign, (size_t)m, d2h, s) != cudaSuccess ||
        cudaMemcpyAsync(status_host, &prm.hdr->status, sizeof(int32_t), d2h, s) != cudaSuccess)
        return HK_ECUDA;
    return HK_OK;
}

// ---- sigma-coset sharding (SURVEY.md 8(e) plan P-2)
int32_t hk_shard_plan(int32_t kind, int64_t n, int32_t P, int32_t G, hk_shard_info *out) {
    if (!out) return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, n, n, P, 0, &pl, G);
    if (rc) return rc;
    out->G = G;
    out->gamma = pl.gamma;
    out->block_cols = (int64_t(1) << pl.info.log_n2) / G;
    out->rows_per_rank = pl.rpr;
    out->y_rows = (int64_t)G * pl.rpr;
    out->chunk_words = (int64_t)kNumPrimes * out->block_cols * pl.rpr;
    out->buffer_words = (int64_t)G * out->chunk_words;
    out->ws_bytes = pl.info.ws_bytes;
    out->slice_chunk_words = pl.slice_ok ? pl.slice_chunk : 0;
    out->slice_buffer_words = pl.slice_ok ? (int64_t)G * pl.slice_chunk : 0;
    out->slice_rows_a = pl.slice_ok ? pl.rs_a : 0;
    out->slice_rows_x = pl.slice_ok ? pl.rs_x : 0;
    return HK_OK;
}

int32_t hk_shard_workspace_init(int32_t kind, int64_t n, int32_t P, int32_t G, void *ws,
                                size_t ws_bytes, void *stream) {
    HK_NVTX("hk_shard_workspace_init");
    if (!ws || ((uintptr_t)ws & 255) != 0 || G < 2) return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, n, n, P, 0, &pl, G);
    if (rc) return rc;
    if (ws_bytes < pl.info.ws_bytes) return HK_ENOMEM;
    Params prm;
    fill_params(pl, ws, &prm);
    return init_workspace(pl, prm, ws, stream);
}

static int shard_common(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g, void *ws,
                        size_t ws_bytes, Plan *pl, Params *prm) {
    if (!ws || ((uintptr_t)ws & 255) != 0 || G < 2 || g < 0 || g >= G) return HK_EINVAL;
    int rc = make_plan(kind, n, n, P, 0, pl, G);
    if (rc) return rc;
    if (ws_bytes < pl->info.ws_bytes) return HK_ENOMEM;
    fill_params(*pl, ws, prm);
    prm->k1_block = g;  // rank g keeps output block g (frequencies = bitrev(g) mod G)
    // internal rows finished here (rows reversed for Toeplitz: see yhat_at in hk_k2.cuh)
    prm->shard_row0 = (int64_t)(pl->info.kind == HK_TOEPLITZ ? G - 1 - g : g) * pl->rpr;
    return HK_OK;
}

int32_t hk_hankel_shard_forward(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                const uint64_t *a_mag, const int8_t *a_sign,
                                const uint64_t *x_mag, const int8_t *x_sign, uint32_t *send,
                                void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_hankel_shard_forward");
    if (!a_mag || !a_sign || !x_mag || !x_sign || !send) return HK_EINVAL;
    if ((((uintptr_t)a_mag | (uintptr_t)x_mag) & 15) != 0) return HK_EINVAL;
    Plan pl;
    Params prm;
    int rc = shard_common(kind, n, P, G, g, ws, ws_bytes, &pl, &prm);
    if (rc) return rc;
    prm.a_mag = a_mag; prm.a_sign = a_sign; prm.x_mag = x_mag; prm.x_sign = x_sign;
    prm.Yhat = send;
    if (cudaMemsetAsync(&prm.hdr->status, 0, sizeof(int32_t), (cudaStream_t)stream) != cudaSuccess)
        return HK_ECUDA;
    return launch_ntt_path(prm, stream, HK_STAGE_SLICE_ROWS | HK_STAGE_COLUMNS);
}

int32_t hk_hankel_shard_finish(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                               const uint32_t *recv, uint64_t *y_mag, int8_t *y_sign, void *ws,
                               size_t ws_bytes, void *stream) {
    HK_NVTX("hk_hankel_shard_finish");
    if (!recv || !y_mag || !y_sign) return HK_EINVAL;
    Plan pl;
    Params prm;
    int rc = shard_common(kind, n, P, G, g, ws, ws_bytes, &pl, &prm);
    if (rc) return rc;
    prm.Yhat = const_cast<uint32_t *>(recv);
    prm.y_mag = y_mag; prm.y_sign = y_sign;
    const int64_t row0 = prm.shard_row0;
    const int64_t nrows = (n - row0) < pl.rpr ? (n - row0) : pl.rpr;
    return launch_k3_range(prm, stream, row0, nrows);
}

// ---- sliced sharding: phase 1a (K1 over this rank's positions, scatter) and 1b (K2 gathers)
static int slice_common(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g, void *ws,
                        size_t ws_bytes, Plan *pl, Params *prm) {
    int rc = shard_common(kind, n, P, G, g, ws, ws_bytes, pl, prm);
    if (rc) return rc;
    if (!pl->slice_ok) return HK_EUNSUPPORTED;
    prm->slice_mode = 1;
    int lg = 0;
    while ((int64_t(1) << lg) < pl->rs_a) ++lg;
    prm->lg_rs_a = lg;
    lg = 0;
    while ((int64_t(1) << lg) < pl->rs_x) ++lg;
    prm->lg_rs_x = lg;
    prm->slice_chunk = pl->slice_chunk;
    prm->slice_xoff = (int64_t)kNumPrimes * prm->n2loc * pl->rs_a;
    return HK_OK;
}

// K1 tiles covering matrix positions [g Rs, (g+1) Rs) of a, then of x (x positions are reversed
// rows for Hankel / Toeplitz); tiles straddling two ranks' ranges are run by both, each storing
// its own positions only
static int launch_slice_k1(const Plan &pl, const Params &prm, int32_t g, void *stream) {
    const int kT = k1_tile_rows();
    const int ga = k1_tiles_a(prm), gx = k1_tiles_x(prm);
    const int64_t na = pl.info.a_count, n = pl.info.n;
    int a0 = 0, a1 = 0, x0 = 0, x1 = 0;  // tile ranges (x: combined index ga + t)
    int64_t lo = (int64_t)g * pl.rs_a, hi = lo + pl.rs_a < na ? lo + pl.rs_a : na;
    if (hi > lo) a0 = (int)(lo / kT), a1 = (int)((hi + kT - 1) / kT);
    lo = (int64_t)g * pl.rs_x;
    hi = lo + pl.rs_x < n ? lo + pl.rs_x : n;
    if (hi > lo) {
        const int64_t r_lo = pl.x_reversed ? n - hi : lo, r_hi = pl.x_reversed ? n - lo : hi;
        x0 = ga + (int)(r_lo / kT), x1 = ga + (int)((r_hi + kT - 1) / kT);
    }
    (void)gx;
    if (a1 == a0 && x1 == x0) return HK_OK;
    if (a1 == a0) return launch_k1_range(prm, stream, x0, x1 - x0);
    if (x1 == x0) return launch_k1_range(prm, stream, a0, a1 - a0);
    // both ranges in one launch (each alone is well under one wave at G >= 4)
    Params p2 = prm;
    p2.tile_split = a1 - a0;
    p2.tile_skip = x0 - a1;
    return launch_k1_range(p2, stream, a0, (a1 - a0) + (x1 - x0));
}

int32_t hk_hankel_shard_slice(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                              const uint64_t *a_mag, const int8_t *a_sign, const uint64_t *x_mag,
                              const int8_t *x_sign, uint32_t *slice_send, void *ws, size_t ws_bytes,
                              void *stream) {
    HK_NVTX("hk_hankel_shard_slice");
    if (!a_mag || !a_sign || !x_mag || !x_sign || !slice_send) return HK_EINVAL;
    if ((((uintptr_t)a_mag | (uintptr_t)x_mag) & 15) != 0) return HK_EINVAL;
    Plan pl;
    Params prm;
    int rc = slice_common(kind, n, P, G, g, ws, ws_bytes, &pl, &prm);
    if (rc) return rc;
    prm.a_mag = a_mag; prm.a_sign = a_sign; prm.x_mag = x_mag; prm.x_sign = x_sign;
    prm.slice_out = slice_send;
    if (cudaMemsetAsync(&prm.hdr->status, 0, sizeof(int32_t), (cudaStream_t)stream) != cudaSuccess)
        return HK_ECUDA;
    return launch_slice_k1(pl, prm, g, stream);
}

int32_t hk_hankel_shard_slice_p2p(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                  const uint64_t *a_mag, const int8_t *a_sign, const uint64_t *x_mag,
                                  const int8_t *x_sign, uint32_t *const *slice_recv_ptrs, void *ws,
                                  size_t ws_bytes, void *stream) {
    HK_NVTX("hk_hankel_shard_slice_p2p");
    if (!a_mag || !a_sign || !x_mag || !x_sign || !slice_recv_ptrs) return HK_EINVAL;
    if ((((uintptr_t)a_mag | (uintptr_t)x_mag) & 15) != 0) return HK_EINVAL;
    Plan pl;
    Params prm;
    int rc = slice_common(kind, n, P, G, g, ws, ws_bytes, &pl, &prm);
    if (rc) return rc;
    for (int d = 0; d < G; ++d) {
        if (!slice_recv_ptrs[d]) return HK_EINVAL;
        prm.peer_slice[d] = slice_recv_ptrs[d];
    }
    prm.p2p = 1;
    prm.a_mag = a_mag; prm.a_sign = a_sign; prm.x_mag = x_mag; prm.x_sign = x_sign;
    if (cudaMemsetAsync(&prm.hdr->status, 0, sizeof(int32_t), (cudaStream_t)stream) != cudaSuccess)
        return HK_ECUDA;
    return launch_slice_k1(pl, prm, g, stream);
}

int32_t hk_hankel_shard_columns(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                const uint32_t *slice_recv, uint32_t *send, void *ws, size_t ws_bytes,
                                void *stream) {
    HK_NVTX("hk_hankel_shard_columns");
    if (!slice_recv || !send) return HK_EINVAL;
    Plan pl;
    Params prm;
    int rc = slice_common(kind, n, P, G, g, ws, ws_bytes, &pl, &prm);
    if (rc) return rc;
    prm.slice_in = slice_recv;
    prm.Yhat = send;
    return launch_k2_sliced(prm, stream);
}

int32_t hk_hankel_shard_columns_p2p(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                    const uint32_t *slice_recv, uint32_t *const *recv_ptrs, void *ws,
                                    size_t ws_bytes, void *stream) {
    HK_NVTX("hk_hankel_shard_columns_p2p");
    if (!slice_recv || !recv_ptrs) return HK_EINVAL;
    Plan pl;
    Params prm;
    int rc = slice_common(kind, n, P, G, g, ws, ws_bytes, &pl, &prm);
    if (rc) return rc;
    for (int d = 0; d < G; ++d) {
        if (!recv_ptrs[d]) return HK_EINVAL;
        prm.peer_recv[d] = recv_ptrs[d];
    }
    prm.p2p = 1;
    prm.slice_in = slice_recv;
    prm.Yhat = recv_ptrs[g];
    return launch_k2_sliced(prm, stream);
}

int32_t hk_hankel_shard_forward_p2p(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                    const uint64_t *a_mag, const int8_t *a_sign,
                                    const uint64_t *x_mag, const int8_t *x_sign,
                                    uint32_t *const *recv_ptrs, void *ws, size_t ws_bytes,
                                    void *stream) {
    HK_NVTX("hk_hankel_shard_forward_p2p");
    if (!a_mag || !a_sign || !x_mag || !x_sign || !recv_ptrs) return HK_EINVAL;
    if ((((uintptr_t)a_mag | (uintptr_t)x_mag) & 15) != 0) return HK_EINVAL;
    Plan pl;
    Params prm;
    int rc = shard_common(kind, n, P, G, g, ws, ws_bytes, &pl, &prm);
    if (rc) return rc;
    for (int d = 0; d < G; ++d) {
        if (!recv_ptrs[d]) return HK_EINVAL;
        prm.peer_recv[d] = recv_ptrs[d];
    }
    prm.p2p = 1;
    prm.a_mag = a_mag; prm.a_sign = a_sign; prm.x_mag = x_mag; prm.x_sign = x_sign;
    prm.Yhat = recv_ptrs[g];  // unused by the p2p stores; a valid buffer of this rank
    if (cudaMemsetAsync(&prm.hdr->status, 0, sizeof(int32_t), (cudaStream_t)stream) != cudaSuccess)
        return HK_ECUDA;
    return launch_ntt_path(prm, stream, HK_STAGE_SLICE_ROWS | HK_STAGE_COLUMNS);
}

int32_t hk_hankel_shard_finish_p2p(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                   const uint32_t *recv, uint64_t *const *y_mag_ptrs,
                                   int8_t *const *y_sign_ptrs, void *ws, size_t ws_bytes,
                                   void *stream) {
    HK_NVTX("hk_hankel_shard_finish_p2p");
    if (!recv || !y_mag_ptrs || !y_sign_ptrs) return HK_EINVAL;
    Plan pl;
    Params prm;
    int rc = shard_common(kind, n, P, G, g, ws, ws_bytes, &pl, &prm);
    if (rc) return rc;
    for (int d = 0; d < G; ++d) {
        if (!y_mag_ptrs[d] || !y_sign_ptrs[d]) return HK_EINVAL;
        prm.peer_ymag[d] = y_mag_ptrs[d];
        prm.peer_ysign[d] = y_sign_ptrs[d];
    }
    prm.p2p = 1;
    prm.Yhat = const_cast<uint32_t *>(recv);
    prm.y_mag = y_mag_ptrs[g]; prm.y_sign = y_sign_ptrs[g];
    const int64_t row0 = prm.shard_row0;
    const int64_t nrows = (n - row0) < pl.rpr ? (n - row0) : pl.rpr;
    return launch_k3_range(prm, stream, row0, nrows);
}

int32_t hk_prepare_a(int32_t kind, int64_t m, int64_t n, int32_t P, const uint64_t *a_mag,
                     const int8_t *a_sign, void *ws, size_t ws_bytes, void *stream) {
    HK_NVTX("hk_prepare_a");
    if (!a_mag || !a_sign || !ws || ((uintptr_t)ws & 255) != 0 || ((uintptr_t)a_mag & 15) != 0)
        return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, m, n, P, HK_WS_PREPARED, &pl);
    if (rc) return rc;
    if (ws_bytes < pl.info.ws_bytes_prepared) return HK_ENOMEM;
    Params prm;
    fill_params(pl, ws, &prm);
    prm.a_mag = a_mag; prm.a_sign = a_sign;
    prm.AT = (uint32_t *)((char *)ws + pl.off_AT);
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(&prm.hdr->status, 0, 2 * sizeof(int32_t), st) != cudaSuccess)  // + a_ready
        return HK_ECUDA;
    if ((rc = launch_k1_range(prm, stream, 0, k1_tiles_a(prm)))) return rc;
    if ((rc = launch_k2_mode(prm, stream, 1))) return rc;
    // a_ready = 1 only if a passed validation (stream-ordered after the transforms): a prepare
    // that saw HK_ERANGE leaves a_ready = 0, so every later hk_matvec_prepared reports HK_EINVAL
    // instead of computing with a rejected matrix
    return launch_set_a_ready(prm, stream);
}

int32_t hk_matvec_prepared(int32_t kind, int64_t m, int64_t n, int32_t P, const uint64_t *x_mag,
                           const int8_t *x_sign, uint64_t *y_mag, int8_t *y_sign, void *ws,
                           size_t ws_bytes, void *stream) {
    HK_NVTX("hk_matvec_prepared");
    if (!x_mag || !x_sign || !y_mag || !y_sign || !ws || ((uintptr_t)ws & 255) != 0 ||
        ((uintptr_t)x_mag & 15) != 0)
        return HK_EINVAL;
    Plan pl;
    int rc = make_plan(kind, m, n, P, HK_WS_PREPARED, &pl);
    if (rc) return rc;
    if (ws_bytes < pl.info.ws_bytes_prepared) return HK_ENOMEM;
    const size_t Ly = pl.info.Ly, L = pl.info.L;
    if (overlaps(y_mag, (size_t)m * Ly * 8, x_mag, (size_t)n * L * 8) ||
        overlaps(y_sign, (size_t)m, x_sign, (size_t)n) ||
        overlaps(y_mag, (size_t)m * Ly * 8, ws, pl.info.ws_bytes_prepared) ||
        overlaps(y_sign, (size_t)m, ws, pl.info.ws_bytes_prepared))
        return HK_EINVAL;
    Params prm;
    fill_params(pl, ws, &prm);
    prm.x_mag = x_mag; prm.x_sign = x_sign; prm.y_mag = y_mag; prm.y_sign = y_sign;
    prm.AT = (uint32_t *)((char *)ws + pl.off_AT);
    prm.need_a_ready = 1;
    if (cudaMemsetAsync(&prm.hdr->status, 0, sizeof(int32_t), (cudaStream_t)stream) != cudaSuccess)
        return HK_ECUDA;
    const int ga = k1_tiles_a(prm);
    if ((rc = launch_k1_range(prm, stream, ga, k1_tiles_x(prm)))) return rc;
    if ((rc = launch_k2_mode(prm, stream, 2))) return rc;
    return launch_k3_range(prm, stream, 0, m);
}

int32_t hk_matvec_stages(int32_t kind, int64_t m, int64_t n, int32_t P, uint32_t stages,
                         const uint64_t *a_mag, const int8_t *a_sign, const uint64_t *x_mag,
                         const int8_t *x_sign, uint64_t *y_mag, int8_t *y_sign, void *ws,
                         size_t ws_bytes, void *stream) {
    HK_NVTX("hk_matvec_stages");
    if (stages == 0 || (stages & ~HK_STAGE_ALL)) return HK_EINVAL;
    return run_matvec(kind, m, n, P, a_mag, a_sign, x_mag, x_sign, y_mag, y_sign, ws, ws_bytes,
                      stream, stages);
}

int32_t hk_schoolbook_matvec(int32_t kind, int64_t m, int64_t n, int32_t P,
                             const uint64_t *a_mag, const int8_t *a_sign, const uint64_t *x_mag,
                             const int8_t *x_sign, uint64_t *y_mag, int8_t *y_sign, void *stream) {
    HK_NVTX("hk_schoolbook_matvec");
    if (!a_mag || !a_sign || !x_mag || !x_sign || !y_mag || !y_sign) return HK_EINVAL;
    if (kind < HK_HANKEL || kind > HK_CIRCULANT || n < 1 || m < 1 || P < 1) return HK_EINVAL;
    if (kind != HK_HANKEL && m != n) return HK_EINVAL;
    return launch_schoolbook(kind, m, n, P, a_mag, a_sign, x_mag, x_sign, y_mag, y_sign, stream);
}

int32_t hk_karatsuba_workspace_size(int64_t n, int32_t P, int32_t cutoff, size_t *bytes) {
    if (!bytes) return HK_EINVAL;
    return karatsuba_workspace_size(n, P, cutoff, bytes);
}

int32_t hk_karatsuba_matvec(int64_t n, int32_t P, int32_t cutoff, const uint64_t *a_mag,
                            const int8_t *a_sign, const uint64_t *x_mag, const int8_t *x_sign,
                            uint64_t *y_mag, int8_t *y_sign, void *ws, size_t ws_bytes,
                            void *stream) {
    HK_NVTX("hk_karatsuba_matvec");
    if (!a_mag || !a_sign || !x_mag || !x_sign || !y_mag || !y_sign || !ws) return HK_EINVAL;
    if (((uintptr_t)ws & 255) != 0) return HK_EINVAL;
    return launch_karatsuba(n, P, cutoff, a_mag, a_sign, x_mag, x_sign, y_mag, y_sign, ws,
                            ws_bytes, stream);
}

}  // extern "C"
