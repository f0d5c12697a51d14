// hk_k2.cuh -- K2, the matrix-index (column) pass of the 2-D NTT convolution (SURVEY.md 8(a)
// rows A2/A3).  One CTA handles one (prime, sigma) column of N1 = 2^LOGN points:
//
//   X^ : first DIF pass straight from HBM -> middle passes in smem -> last pass kept in registers
//   A^ : first DIF pass straight from HBM -> middle passes -> last pass in registers,
//        pointwise Montgomery product with the held X^ values, first DIT pass (same groups) in
//        registers -> middle DIT passes -> last DIT pass stored straight to Y^ in HBM
//
// Pass plan: forward passes of radix 2^5 from the top; the last (S = 1) pass takes the remainder
// RL = LOGN - 5 (NP - 1).  The inverse mirrors it (RL first, then radix-2^5 passes).  The DIT
// runs with the FORWARD roots, which yields the inverse transform with the output index negated
// (hk_modarith.cuh), so output row i is read from position (N1 - out_off - i) mod N1.
#pragma once
#include <type_traits>
#include "hk_internal.h"
#include "hk_modarith.cuh"

namespace hk {

// N1 = 2^14 (C3): 256 threads (two top-pass groups each), 2 CTAs per SM, no A^ staging: two
// independent columns per SM desynchronise their barrier / load / arithmetic phases, which beats
// one 512-thread CTA with A^ staged in smem (0.70 vs 0.76 ms at C3) despite 148 B of spills
#ifndef HK_K2_T14
#define HK_K2_T14 256  // threads per CTA at N1 = 2^14
#endif
#ifndef HK_K2_MINB14
#define HK_K2_MINB14 2  // resident CTAs per SM at N1 = 2^14
#endif
#ifndef HK_K2_L2PF
#define HK_K2_L2PF 1  // bulk-prefetch the A^ column into L2 when it is not staged in smem
#endif
#ifndef HK_K2_L2PF_NEXT
#define HK_K2_L2PF_NEXT 148  // columns ahead whose X^ is also prefetched into L2 (0: off)
#endif
#ifndef HK_K2_PRUNE
#define HK_K2_PRUNE 1  // last inverse stage forms / stores only the output whose row is kept (C3 K2 -2.8%)
#endif
#ifndef HK_K2_XPF
#define HK_K2_XPF 1  // X^ top pass: both groups' loads issued before the first group's butterflies (C3 K2 -0.2%)
#endif
#ifndef HK_K2_STAGE14
#define HK_K2_STAGE14 0  // stage the A^ column in smem by cp.async at N1 = 2^14
#endif
template <int LOGN1>
constexpr int k2_threads() {
    if (LOGN1 == 14) return HK_K2_T14;
    return (1 << LOGN1) / 32 < 32 ? 32 : ((1 << LOGN1) / 32 > 512 ? 512 : (1 << LOGN1) / 32);
}
#ifndef HK_K2_WARPS_SMALL
#define HK_K2_WARPS_SMALL 24  // N1 <= 2^13: resident warps per SM asked of the register allocator (0: no
                              // bound; 24 caps at 80 registers: K2 -9% at C2 and C5 circulant, -4% at C5 Toeplitz)
#endif
template <int LOGN1>
constexpr int k2_min_blocks() {
    return LOGN1 == 14 ? HK_K2_MINB14
                       : (LOGN1 < 14 && HK_K2_WARPS_SMALL > 0 ? HK_K2_WARPS_SMALL * 32 / k2_threads<LOGN1>() : 1);
}

template <int LOGN>
struct ColPlan {
    static constexpr int NP = (LOGN + 4) / 5;         // passes per transform (>= 2 for LOGN >= 6)
    static constexpr int RL = LOGN - 5 * (NP - 1);    // log2 radix of the bottom pass
    static constexpr int T = k2_threads<LOGN>();
    static constexpr int GL = 1 << RL;                // points per bottom-pass group
    static constexpr int GPT = (1 << LOGN) / GL / T;  // bottom-pass groups per thread
    static_assert(NP >= 2, "column transforms need LOGN >= 6");
    static_assert(GPT >= 1 && GPT * GL * T == (1 << LOGN), "bottom pass must tile the threads");
};

// Top forward pass (R = 5, S = N/32, single block) reading the column straight from HBM
// (SRC_SMEM = false) or from a shared-memory staging copy (SRC_SMEM = true).  The column is zero-
// padded in the workspace up to its loaded extent (N/2 when the upper half is known to be zero, ZU,
// else N; hk_api.cu make_plan), so the loads need no bounds checks.
template <class TW, int LOGN, int T, bool SRC_SMEM, bool ZU>
HK_DEV void k2_dif_top_load(const uint32_t *__restrict__ src, uint32_t *sm, const uint2 *tw,
                            uint32_t p) {
    constexpr int N = 1 << LOGN, R = 5, G = 32, S = N / G;
#if HK_K2_XPF
    if constexpr (ZU && !SRC_SMEM && S == 2 * T) {
        // upper half zero: both of this thread's groups fit in 32 registers, so all their loads are
        // issued before the first group's butterflies (twice the loads in flight)
        uint32_t v2[G / 2];
        const int j1 = threadIdx.x + T;
#pragma unroll
        for (int m = 0; m < G / 2; ++m) v2[m] = __ldcs(src + j1 + m * S);
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
            const int j0 = threadIdx.x + pass * T;
            uint32_t v[G];
#pragma unroll
            for (int m = 0; m < G / 2; ++m) v[m] = pass ? v2[m] : __ldcs(src + j0 + m * S);
#pragma unroll
            for (int m = 0; m < G / 2; ++m) {  // (u, 0) -> (u, u W)
                const uint2 w = TW::ld(tw, S * (G / 2) + j0 + S * m);
                v[m + G / 2] = red1(shoup(v[m], w.x, w.y, p), p);
            }
#pragma unroll
            for (int l = R - 2; l >= 0; --l) {
                const int half = 1 << l;
#pragma unroll
                for (int m = 0; m < G; ++m) {
                    if (m & half) continue;
                    const uint2 w = TW::ld(tw, S * half + j0 + S * (m & (half - 1)));
                    gs_bfly(v[m], v[m + half], w, p);
                }
            }
            uint32_t *b0 = sm + pad(j0);
#pragma unroll
            for (int m = 0; m < G; ++m) b0[padded_len(m * S)] = v[m];
        }
        __syncthreads();
        return;
    }
#endif
    for (int j0 = threadIdx.x; j0 < S; j0 += T) {
        uint32_t v[G];
#pragma unroll
        for (int m = 0; m < G; ++m) {
            if (ZU && m >= G / 2) v[m] = 0u;
            else if (SRC_SMEM) v[m] = src[j0 + m * S];
            else v[m] = __ldcs(src + j0 + m * S);
        }
#pragma unroll
        for (int l = R - 1; l >= 0; --l) {
            const int half = 1 << l;
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & half) continue;
                if (ZU && l == R - 1) {  // (u, 0) -> (u, u W)
                    const uint2 w = TW::ld(tw, S * half + j0 + S * m);
                    v[m + half] = red1(shoup(v[m], w.x, w.y, p), p);
                    continue;
                }
                const uint2 w = TW::ld(tw, S * half + j0 + S * (m & (half - 1)));
                gs_bfly(v[m], v[m + half], w, p);
            }
        }
        uint32_t *b0 = sm + pad(j0);  // pad(j0 + m S) = pad(j0) + pad(m S) (S multiple of 32)
#pragma unroll
        for (int m = 0; m < G; ++m) b0[padded_len(m * S)] = v[m];
    }
    __syncthreads();
}
template <class TW, int LOGN, int T, bool SRC_SMEM = false>
HK_DEV void k2_dif_top_from_global(const uint32_t *__restrict__ src, bool zu, uint32_t *sm,
                                   const uint2 *tw, uint32_t p) {
    if (zu) k2_dif_top_load<TW, LOGN, T, SRC_SMEM, true>(src, sm, tw, p);
    else k2_dif_top_load<TW, LOGN, T, SRC_SMEM, false>(src, sm, tw, p);
}

// Sliced shards: the same top pass with the column gathered from the slice receive buffer, where
// matrix position i of this column sits in source (i >> lg)'s chunk at offset i & (2^lg - 1).
// Point m of group j0 is position j0 + m S.  When 2^lg >= S (Q = lg - log2 S >= 0) a group never
// crosses a segment boundary: point m lies in segment m >> Q at offset (m mod 2^Q) S + j0, so with Q
// a template parameter each segment is one base pointer and the loads take immediate offsets.
template <class TW, int LOGN, int T, bool ZU, int Q>
HK_DEV void k2_dif_top_gather_q(const uint32_t *__restrict__ src, size_t chunk, int lg, uint32_t *sm,
                                const uint2 *tw, uint32_t p) {
    constexpr int N = 1 << LOGN, R = 5, G = 32, S = N / G;
    const unsigned mask = (1u << lg) - 1u;
    for (int j0 = threadIdx.x; j0 < S; j0 += T) {
        uint32_t v[G];
#pragma unroll
        for (int m = 0; m < G; ++m) {
            if (ZU && m >= G / 2) {
                v[m] = 0u;
            } else if constexpr (Q >= 0) {
                const uint32_t *seg = src + (size_t)(m >> Q) * chunk + j0;
                v[m] = __ldcs(seg + (m & ((1 << Q) - 1)) * S);
            } else {
                const unsigned i = (unsigned)(j0 + m * S);
                v[m] = __ldcs(src + (size_t)(i >> lg) * chunk + (i & mask));
            }
        }
#pragma unroll
        for (int l = R - 1; l >= 0; --l) {
            const int half = 1 << l;
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & half) continue;
                if (ZU && l == R - 1) {  // (u, 0) -> (u, u W)
                    const uint2 w = TW::ld(tw, S * half + j0 + S * m);
                    v[m + half] = red1(shoup(v[m], w.x, w.y, p), p);
                    continue;
                }
                const uint2 w = TW::ld(tw, S * half + j0 + S * (m & (half - 1)));
                gs_bfly(v[m], v[m + half], w, p);
            }
        }
        uint32_t *b0 = sm + pad(j0);
#pragma unroll
        for (int m = 0; m < G; ++m) b0[padded_len(m * S)] = v[m];
    }
    __syncthreads();
}
template <class TW, int LOGN, int T, bool ZU>
HK_DEV void k2_dif_top_gather(const uint32_t *__restrict__ src, size_t chunk, int lg, uint32_t *sm,
                              const uint2 *tw, uint32_t p) {
    switch (lg - (LOGN - 5)) {
        case 0: k2_dif_top_gather_q<TW, LOGN, T, ZU, 0>(src, chunk, lg, sm, tw, p); break;
        case 1: k2_dif_top_gather_q<TW, LOGN, T, ZU, 1>(src, chunk, lg, sm, tw, p); break;
        case 2: k2_dif_top_gather_q<TW, LOGN, T, ZU, 2>(src, chunk, lg, sm, tw, p); break;
        case 3: k2_dif_top_gather_q<TW, LOGN, T, ZU, 3>(src, chunk, lg, sm, tw, p); break;
        case 4: k2_dif_top_gather_q<TW, LOGN, T, ZU, 4>(src, chunk, lg, sm, tw, p); break;
        default: k2_dif_top_gather_q<TW, LOGN, T, ZU, -1>(src, chunk, lg, sm, tw, p); break;
    }
}

// Middle forward passes (R = 5), k = 1 .. NP-2.
template <class TW, int LOGN, int K>
struct K2DifMiddle {
    static HK_DEV void run(uint32_t *sm, const uint2 *tw, uint32_t p) {
        constexpr int NP = ColPlan<LOGN>::NP;
        if constexpr (K <= NP - 2) {
            constexpr int S = 1 << (LOGN - 5 * (K + 1));
            dif_pass<TW, LOGN, 5, S, false>(sm, 1, 0, tw, p, threadIdx.x, ColPlan<LOGN>::T);
            K2DifMiddle<TW, LOGN, K + 1>::run(sm, tw, p);
        }
    }
};

// Middle inverse passes (R = 5), from S = 2^RL upwards, all but the top one.
template <class TW, int LOGN, int LO>
struct K2DitMiddle {
    static HK_DEV void run(uint32_t *sm, const uint2 *tw, uint32_t p) {
        if constexpr (LO + 5 < LOGN) {
            dit_pass<TW, LOGN, 5, (1 << LO)>(sm, 1, 0, tw, p, threadIdx.x, ColPlan<LOGN>::T);
            K2DitMiddle<TW, LOGN, LO + 5>::run(sm, tw, p);
        }
    }
};

// Bottom DIF pass (S = 1) of group g held in v[].
template <class TW, int RL>
HK_DEV void dif_bottom_regs(uint32_t (&v)[1 << RL], const uint2 *tw, uint32_t p) {
#pragma unroll
    for (int l = RL - 1; l >= 0; --l) {
        const int half = 1 << l;
#pragma unroll
        for (int m = 0; m < (1 << RL); ++m) {
            if (m & half) continue;
            if ((m & (half - 1)) == 0) bfly1(v[m], v[m + half], p);  // twiddle 1
            else gs_bfly(v[m], v[m + half], TW::ld(tw, half + (m & (half - 1))), p);
        }
    }
}
template <class TW, int RL>
HK_DEV void dit_bottom_regs(uint32_t (&v)[1 << RL], const uint2 *tw, uint32_t p) {
#pragma unroll
    for (int l = 0; l < RL; ++l) {
        const int half = 1 << l;
#pragma unroll
        for (int m = 0; m < (1 << RL); ++m) {
            if (m & half) continue;
            if ((m & (half - 1)) == 0) bfly1(v[m], v[m + half], p);  // twiddle 1
            else ct_bfly(v[m], v[m + half], TW::ld(tw, half + (m & (half - 1))), p);
        }
    }
}

// Y^ element (column cidx, output row i): the single-GPU layout [column][ldY], or, for sigma-coset
// shards, the all-to-all send buffer [dest rank][column][rpr]: row block i / rpr goes to rank
// i / rpr (to rank G - 1 - i / rpr when the rows are reversed, Toeplitz, so that every rank's
// final y rows form block `rank` of the padded y and the all-gather is in rank order).
// With peer-memory exchange (prm.p2p) the chunk goes straight into rank dst's receive buffer, at
// this rank's (source) chunk slot -- the all-to-all fused into K2's stores.
template <bool SHARD>
HK_DEV uint32_t *yhat_at(const Params &prm, size_t cidx, int i) {
    if constexpr (!SHARD) return prm.Yhat + cidx * prm.ldY + i;
    const unsigned rpr = (unsigned)prm.shard_rpr, blk = (unsigned)i / rpr;
    const unsigned dst = prm.reverse_out ? (1u << prm.shard_gamma) - 1u - blk : blk;
    const size_t chunk = (size_t)kNumPrimes * prm.n2loc;
    if (prm.p2p)
        return prm.peer_recv[dst] + ((size_t)prm.k1_block * chunk + cidx) * rpr + ((unsigned)i - blk * rpr);
    return prm.Yhat + ((size_t)dst * chunk + cidx) * rpr + ((unsigned)i - blk * rpr);
}

// Top inverse pass (R = 5, S = N/32) with the result going to HBM (or back to smem for fold).
template <class TW, int LOGN, int T, bool SHARD = false>
HK_DEV void k2_dit_top(uint32_t *sm, const uint2 *tw, uint32_t p, const Params &prm, size_t cidx,
                       int mrows, int off, bool to_smem) {
    constexpr int N = 1 << LOGN, R = 5, G = 32, S = N / G;
#if HK_K2_PRUNE
    if (!to_smem && mrows <= N / 2) {
        // Output pruning: the last stage pairs positions p and p + N/2, whose output rows differ by
        // N/2 (row(p) = (N - p - off) mod N), so at most one of the two is among the mrows <= N/2
        // rows kept -- only that output is formed (u + t, or u - t = u + (p - t)) and stored.
        for (int j0 = threadIdx.x; j0 < S; j0 += T) {
            uint32_t v[G];
            uint32_t *b0 = sm + pad(j0);
#pragma unroll
            for (int m = 0; m < G; ++m) v[m] = b0[padded_len(m * S)];
#pragma unroll
            for (int l = 0; l < R - 1; ++l) {
                const int half = 1 << l;
#pragma unroll
                for (int m = 0; m < G; ++m) {
                    if (m & half) continue;
                    const uint2 w = TW::ld(tw, S * half + j0 + S * (m & (half - 1)));
                    ct_bfly(v[m], v[m + half], w, p);
                }
            }
#pragma unroll
            for (int m = 0; m < G / 2; ++m) {
                const uint2 w = TW::ld(tw, S * (G / 2) + j0 + S * m);
                const uint32_t t = red1(shoup(v[m + G / 2], w.x, w.y, p), p);
                const int ilo = (N - (j0 + m * S) - off) & (N - 1);  // row of position j0 + m S
                const uint32_t tt = (ilo & (N / 2)) ? p - t : t;     // the partner's row is ilo - N/2
                const int i = ilo & (N / 2 - 1);
                if (i < mrows) __stcs(yhat_at<SHARD>(prm, cidx, i), addm(v[m], tt, p));
            }
        }
        __syncthreads();
        return;
    }
#endif
    for (int j0 = threadIdx.x; j0 < S; j0 += T) {
        uint32_t v[G];
        uint32_t *b0 = sm + pad(j0);  // S multiple of 32
#pragma unroll
        for (int m = 0; m < G; ++m) v[m] = b0[padded_len(m * S)];
#pragma unroll
        for (int l = 0; l < R; ++l) {
            const int half = 1 << l;
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & half) continue;
                const uint2 w = TW::ld(tw, S * half + j0 + S * (m & (half - 1)));
                ct_bfly(v[m], v[m + half], w, p);
            }
        }
        if (to_smem) {
#pragma unroll
            for (int m = 0; m < G; ++m) b0[padded_len(m * S)] = v[m];
        } else {
#pragma unroll
            for (int m = 0; m < G; ++m) {
                const int i = (N - (j0 + m * S) - off) & (N - 1);  // output row of this position
                if (i < mrows) __stcs(yhat_at<SHARD>(prm, cidx, i), v[m]);
            }
        }
    }
    __syncthreads();
}

// A^ column staged in shared memory by cp.async while X^ is transformed (hides the HBM
// latency of A^'s top pass); needs N1 more words of smem, so only for N1 <= 16384.
template <int LOGN1>
constexpr bool k2_stage_a() { return LOGN1 < 14 || (LOGN1 == 14 && HK_K2_STAGE14); }
template <int LOGN1>
constexpr int k2_stage_off() { return (padded_len(1 << LOGN1) + 3) & ~3; }  // 16-byte aligned
#ifndef HK_K2_SMTW
#define HK_K2_SMTW 1  // middle / bottom-pass twiddles (table entries < 512) copied into smem
#endif
constexpr int kK2LowTw = 512;
template <int LOGN1>
constexpr bool k2_smtw() { return HK_K2_SMTW && !k2_stage_a<LOGN1>() && (1 << LOGN1) / 32 >= kK2LowTw / 32; }
template <int LOGN1>
constexpr size_t k2_smem_bytes() {
    return k2_stage_a<LOGN1>() ? (size_t)(k2_stage_off<LOGN1>() + (1 << LOGN1)) * 4
                               : (size_t)padded_len(1 << LOGN1) * 4 + (k2_smtw<LOGN1>() ? 16 + kK2LowTw * 8 : 0);
}

template <class TW, int LOGN1, bool SHARD, bool SLICED = false>
HK_DEV void k2_column_body(const Params &prm, uint32_t *sm, const uint2 *twf, int kp, int sigma) {
    using PL = ColPlan<LOGN1>;
    constexpr int N1 = 1 << LOGN1, T = PL::T, RL = PL::RL, GL = PL::GL, GPT = PL::GPT;
    constexpr bool STAGE = k2_stage_a<LOGN1>();
    const int tid = threadIdx.x;
    const uint32_t p = prm.pc[kp].p, pneg = prm.pc[kp].pneg;
    const size_t cidx = (size_t)kp * prm.n2loc + sigma;
    uint32_t *sA = sm + k2_stage_off<LOGN1>();
    // sliced shards: this column's positions in the slice receive buffer (source 0's chunk)
    const uint32_t *slA = SLICED ? prm.slice_in + (cidx << prm.lg_rs_a) : nullptr;
    const uint32_t *slX = SLICED ? prm.slice_in + prm.slice_xoff + (cidx << prm.lg_rs_x) : nullptr;
    if constexpr (STAGE) {  // issue the A^ column copy now; consumed after X^'s transform
        const int nch = (int)prm.ldA >> 2;  // the zero-padded column (ldA = N1 or N1 / 2)
        if constexpr (SLICED) {  // 4-position segments never straddle two sources (Rs >= 8)
            const unsigned mask = (1u << prm.lg_rs_a) - 1u;
            for (int c = tid; c < nch; c += T) {
                const unsigned i = 4u * c;
                cp_async16(sA + i, slA + (size_t)(i >> prm.lg_rs_a) * prm.slice_chunk + (i & mask));
            }
        } else {
            const uint32_t *g = prm.Ahat + cidx * prm.ldA;
            for (int c = tid; c < nch; c += T) cp_async16(sA + 4 * c, g + 4 * c);
        }
    } else if (HK_K2_L2PF && SLICED) {
        // the A^ column's G segments (one per source rank) into L2 during X^'s transform, and the
        // X^ segments of the column about one wave ahead
        const int G = 1 << prm.shard_gamma;
        if (tid < G)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(slA + (size_t)tid * prm.slice_chunk),
                         "r"(4u << prm.lg_rs_a) : "memory");
        const size_t nxt = cidx + HK_K2_L2PF_NEXT;
        if (HK_K2_L2PF_NEXT && tid >= 32 && tid < 32 + G && nxt < (size_t)kNumPrimes * prm.n2loc)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n"
                         ::"l"(prm.slice_in + prm.slice_xoff + (nxt << prm.lg_rs_x) + (size_t)(tid - 32) * prm.slice_chunk),
                         "r"(4u << prm.lg_rs_x) : "memory");
    } else if (HK_K2_L2PF && !SLICED && tid == 0) {
        // no staging room: have the A^ column brought into L2 (bulk prefetch) during X^'s transform
        const uint32_t *g = prm.Ahat + cidx * prm.ldA;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(g),
                     "r"((unsigned)(prm.ldA * 4)) : "memory");
        if (HK_K2_L2PF_NEXT) {  // and the X^ column of a CTA about one wave ahead
            const size_t nxt = cidx + HK_K2_L2PF_NEXT;
            if (nxt < (size_t)kNumPrimes * prm.n2loc)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(prm.Xhat + nxt * prm.ldX),
                             "r"((unsigned)(prm.ldX * 4)) : "memory");
        }
    }

    // low twiddle levels (h < 512: the middle and bottom passes) in shared memory when enabled
    using TWM = typename std::conditional<k2_smtw<LOGN1>(), TwShared, TW>::type;
    const uint2 *twm = twf;
    if constexpr (k2_smtw<LOGN1>()) {
        uint2 *tl = reinterpret_cast<uint2 *>(sm + ((padded_len(N1) + 3) & ~3));
        for (int i = tid; i < kK2LowTw; i += T) tl[i] = __ldg(twf + i);
        twm = tl;  // visible after the first pass's barrier
    }
    // ---- X^: forward, bottom pass kept in registers
    {
        const int nx = (int)prm.n;
        if constexpr (SLICED) {
            if (nx <= N1 / 2) k2_dif_top_gather<TW, LOGN1, T, true>(slX, prm.slice_chunk, prm.lg_rs_x, sm, twf, p);
            else k2_dif_top_gather<TW, LOGN1, T, false>(slX, prm.slice_chunk, prm.lg_rs_x, sm, twf, p);
        } else {
            k2_dif_top_from_global<TW, LOGN1, T>(prm.Xhat + cidx * prm.ldX, nx <= N1 / 2, sm, twf, p);
        }
        K2DifMiddle<TWM, LOGN1, 1>::run(sm, twm, p);
    }
    uint32_t xr[GPT][GL];
#pragma unroll
    for (int k = 0; k < GPT; ++k) {
        const int g = tid + k * T;
#pragma unroll
        for (int m = 0; m < GL; ++m) xr[k][m] = sm[pad(g * GL) + m];
        dif_bottom_regs<TWM, RL>(xr[k], twm, p);
    }
    __syncthreads();
    // ---- A^: forward; bottom pass + pointwise + first inverse pass in registers
    {
        const int na = (int)prm.a_count;
        if constexpr (STAGE) {
            cp_async_wait_all();
            __syncthreads();
            k2_dif_top_from_global<TW, LOGN1, T, true>(sA, na <= N1 / 2, sm, twf, p);
        } else if constexpr (SLICED) {
            if (na <= N1 / 2) k2_dif_top_gather<TW, LOGN1, T, true>(slA, prm.slice_chunk, prm.lg_rs_a, sm, twf, p);
            else k2_dif_top_gather<TW, LOGN1, T, false>(slA, prm.slice_chunk, prm.lg_rs_a, sm, twf, p);
        } else {
            k2_dif_top_from_global<TW, LOGN1, T>(prm.Ahat + cidx * prm.ldA, na <= N1 / 2, sm, twf, p);
        }
        K2DifMiddle<TWM, LOGN1, 1>::run(sm, twm, p);
    }
#pragma unroll
    for (int k = 0; k < GPT; ++k) {
        const int g = tid + k * T;
        uint32_t v[GL];
#pragma unroll
        for (int m = 0; m < GL; ++m) v[m] = sm[pad(g * GL) + m];
        dif_bottom_regs<TWM, RL>(v, twm, p);
#pragma unroll
        for (int m = 0; m < GL; ++m) v[m] = mont(v[m], xr[k][m], p, pneg);
        dit_bottom_regs<TWM, RL>(v, twm, p);
#pragma unroll
        for (int m = 0; m < GL; ++m) sm[pad(g * GL) + m] = v[m];
    }
    __syncthreads();
    K2DitMiddle<TWM, LOGN1, RL>::run(sm, twm, p);
    const int mrows = (int)prm.m, off = (int)prm.out_off;
    if (!prm.fold) {
        k2_dit_top<TW, LOGN1, T, SHARD>(sm, twf, p, prm, cidx, mrows, off, false);
    } else {  // circulant via linear convolution: y[i] = z[i] + z[i + n]
        k2_dit_top<TW, LOGN1, T, SHARD>(sm, twf, p, prm, cidx, mrows, off, true);
        const int nn = (int)prm.n;
        for (int i = tid; i < mrows; i += T) {
            const uint32_t v = sm[pad((N1 - (off + i)) & (N1 - 1))];
            *yhat_at<SHARD>(prm, cidx, i) = addm(v, sm[pad((N1 - (off + i + nn)) & (N1 - 1))], p);
        }
        __syncthreads();
    }
    if (SHARD && prm.p2p) __threadfence_system();  // peer stores visible before the next barrier
}

// Inverse passes above the bottom one, output to Y^ (shared by the full and prepared bodies).
template <class TW, int LOGN1, bool SHARD = false>
HK_DEV void k2_inverse_tail(const Params &prm, uint32_t *sm, const uint2 *twf, uint32_t p,
                            size_t cidx) {
    using PL = ColPlan<LOGN1>;
    constexpr int N1 = 1 << LOGN1, T = PL::T, RL = PL::RL;
    K2DitMiddle<TW, LOGN1, RL>::run(sm, twf, p);
    const int mrows = (int)prm.m, off = (int)prm.out_off;
    if (!prm.fold) {
        k2_dit_top<TW, LOGN1, T, SHARD>(sm, twf, p, prm, cidx, mrows, off, false);
    } else {
        k2_dit_top<TW, LOGN1, T, SHARD>(sm, twf, p, prm, cidx, mrows, off, true);
        const int nn = (int)prm.n;
        for (int i = threadIdx.x; i < mrows; i += T) {
            const uint32_t v = sm[pad((N1 - (off + i)) & (N1 - 1))];
            *yhat_at<SHARD>(prm, cidx, i) = addm(v, sm[pad((N1 - (off + i + nn)) & (N1 - 1))], p);
        }
        __syncthreads();
    }
    if (SHARD && prm.p2p) __threadfence_system();  // peer stores visible before the next barrier
}

// F1 prepare: A^'s forward column transform only, stored to AT in the bottom-pass register
// layout AT[col][k GL + m][T] (coalesced, read back by the same thread slot in k2_prepared).
template <class TW, int LOGN1>
HK_DEV void k2_prepare_body(const Params &prm, uint32_t *sm, const uint2 *twf, int kp, int sigma) {
    using PL = ColPlan<LOGN1>;
    constexpr int N1 = 1 << LOGN1, T = PL::T, RL = PL::RL, GL = PL::GL, GPT = PL::GPT;
    const int tid = threadIdx.x;
    const uint32_t p = prm.pc[kp].p;
    const size_t cidx = (size_t)kp * prm.n2loc + sigma;
    const int na = (int)prm.a_count;
    k2_dif_top_from_global<TW, LOGN1, T>(prm.Ahat + cidx * prm.ldA, na <= N1 / 2, sm, twf, p);
    K2DifMiddle<TW, LOGN1, 1>::run(sm, twf, p);
    uint32_t *at = prm.AT + cidx * N1;
#pragma unroll
    for (int k = 0; k < GPT; ++k) {
        const int g = tid + k * T;
        uint32_t v[GL];
#pragma unroll
        for (int m = 0; m < GL; ++m) v[m] = sm[pad(g * GL) + m];
        dif_bottom_regs<TW, RL>(v, twf, p);
#pragma unroll
        for (int m = 0; m < GL; ++m) at[(k * GL + m) * T + tid] = v[m];
    }
}

// F1 prepared matvec: X^ forward, pointwise with the stored A^ transform, inverse.
template <class TW, int LOGN1, bool SHARD = false>
HK_DEV void k2_prepared_body(const Params &prm, uint32_t *sm, const uint2 *twf, int kp, int sigma,
                             int vb = 0) {
    using PL = ColPlan<LOGN1>;
    constexpr int N1 = 1 << LOGN1, T = PL::T, RL = PL::RL, GL = PL::GL, GPT = PL::GPT;
    const int tid = threadIdx.x;
    const uint32_t p = prm.pc[kp].p, pneg = prm.pc[kp].pneg;
    const size_t cidx = (size_t)kp * prm.n2loc + sigma;         // A^ (AT) column
    const size_t ncols = (size_t)kNumPrimes * prm.n2loc;
    const size_t cxy = (size_t)vb * ncols + cidx;                // X^ / Y^ column of batch vector vb
    const int nx = (int)prm.n;
    if (HK_K2_L2PF && tid == 0) {  // the stored A^ transform of this column and the next wave's X^
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(prm.AT + cidx * N1),
                     "r"((unsigned)(N1 * 4)) : "memory");
        const size_t nxt = cxy + HK_K2_L2PF_NEXT;
        if (HK_K2_L2PF_NEXT && nxt < ncols * (size_t)prm.nvec)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(prm.Xhat + nxt * prm.ldX),
                         "r"((unsigned)(prm.ldX * 4)) : "memory");
    }
    k2_dif_top_from_global<TW, LOGN1, T>(prm.Xhat + cxy * prm.ldX, nx <= N1 / 2, sm, twf, p);
    K2DifMiddle<TW, LOGN1, 1>::run(sm, twf, p);
    const uint32_t *at = prm.AT + cidx * N1;
#pragma unroll
    for (int k = 0; k < GPT; ++k) {
        const int g = tid + k * T;
        uint32_t v[GL], av[GL];
#pragma unroll
        for (int m = 0; m < GL; ++m) av[m] = __ldcs(at + (k * GL + m) * T + tid);
#pragma unroll
        for (int m = 0; m < GL; ++m) v[m] = sm[pad(g * GL) + m];
        dif_bottom_regs<TW, RL>(v, twf, p);
#pragma unroll
        for (int m = 0; m < GL; ++m) v[m] = mont(av[m], v[m], p, pneg);
        dit_bottom_regs<TW, RL>(v, twf, p);
#pragma unroll
        for (int m = 0; m < GL; ++m) sm[pad(g * GL) + m] = v[m];
    }
    __syncthreads();
    k2_inverse_tail<TW, LOGN1, SHARD>(prm, sm, twf, p, SHARD ? cidx : cxy);
}

// One CTA per column; the N1 forward table is read through the read-only/L1 path.
// MODE 0: full column (X^ and A^ transforms); 1: prepare A^ -> AT; 2: prepared (X^ x AT);
// 3: full column of a sigma-coset shard (output to the all-to-all send buffer); 4: prepared column
// of a shard; 5: full column of a sliced shard (inputs gathered from the slice receive buffer).  N1 >= 2^15 runs MODE 1 then MODE 2 (4 for shards) instead of MODE 0 (3).
template <int LOGN1, class TW = TwGlobal, int MODE = 0>
__global__ void __launch_bounds__(k2_threads<LOGN1>(), k2_min_blocks<LOGN1>()) k2_column(Params prm) {
    extern __shared__ uint32_t sm[];
    // prepared batch (MODE 2, nvec vectors): consecutive CTAs take the same A^ column for the nvec
    // vectors, so the stored AT column is read from HBM once and from L2 after that
    const int col = MODE == 2 ? (int)(blockIdx.x / (unsigned)prm.nvec) : (int)blockIdx.x;
    const int vb = MODE == 2 ? (int)(blockIdx.x % (unsigned)prm.nvec) : 0;
    const int kp = col >> prm.log_n2loc;  // columns (prime, sigma) held here: n2loc per prime
    const int sigma = col & (prm.n2loc - 1);
    const uint2 *twf = prm.tw + (size_t)kp * (prm.N2 + prm.N1) + prm.N2;
    if constexpr (MODE == 0) k2_column_body<TW, LOGN1, false>(prm, sm, twf, kp, sigma);
    else if constexpr (MODE == 3) k2_column_body<TW, LOGN1, true>(prm, sm, twf, kp, sigma);
    else if constexpr (MODE == 5) k2_column_body<TW, LOGN1, true, true>(prm, sm, twf, kp, sigma);
    else if constexpr (MODE == 1) k2_prepare_body<TW, LOGN1>(prm, sm, twf, kp, sigma);
    else if constexpr (MODE == 2) k2_prepared_body<TW, LOGN1>(prm, sm, twf, kp, sigma, vb);
    else k2_prepared_body<TW, LOGN1, true>(prm, sm, twf, kp, sigma);
}

}  // namespace hk
