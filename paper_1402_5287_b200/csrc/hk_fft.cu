// hk_fft.cu -- SURVEY.md 8(f) F3: the paper's decomposition approach with a double-precision FFT
// ("decompose each multiprecision number into a sum of float or double precision
// numbers, then applied a standard FFT library ... and eventually reconstructed"), as an exact product
// path whose rounding error carries a PROVEN bound < 1/2 (reading R24).
//
//   digits   every mantissa |m| < 2^P is cut into Ls balanced w-bit digits d_t in [-2^(w-1), 2^(w-1)]
//            with m = sum_t d_t 2^(w t) (d_t = u_t - 2^w b_t + b_(t-1), u_t the t-th unsigned w-bit
//            field, b_t = [u_t >= 2^(w-1)]; no carry chain), times the entry's sign.
//   FFT      the exact 2-D convolution of DESIGN.md section 3 (matrix index x digit index) is computed
//            with a complex FP64 FFT of N1 x N2 points: F1 row FFTs (N2, per entry), F2 column FFTs
//            (N1) of a and x, pointwise product, inverse column FFT, F3 inverse row FFT -- every
//            butterfly radix-2 with round-to-nearest DADD / DMUL (no FMA contraction, so Percival's
//            per-operation error model holds), twiddles precomputed on the host in long double.
//   bound    Percival (2003, Math. Comp. 72, Thm. 5.1): for a length-2^k cyclic convolution computed
//            this way, |z' - z|_inf < |x|_2 |y|_2 ((1+e)^3k (1+e sqrt5)^(3k+1) (1+b)^3k - 1),
//            e = 2^-53 (unit roundoff), b = twiddle error.  The 2-D transform is a network of
//            k = log2(N1 N2) radix-2 stages of the same kind (reading R24).  With |d_t| <= 2^(w-1):
//            |a|_2 |x|_2 <= sqrt(rows_a n) Ls 2^(2w-2); the planner takes the widest w whose bound is
//            <= 0.49, so rint() of every output coefficient is the exact integer.
//   carry    c_s (|c_s| < Cb = 2^cb) biased to c_s + Cb >= 0, placed at bit w s: per limb q the
//            128-bit sum of the coefficients whose bit offset falls in it, then the binary carry
//            lookahead of K3 v2 and -Cb sum_s 2^(w s) added limb by limb (table in the workspace).
//
// Scope: N2 <= 8192, N1 <= 32768 -- every BASELINE config.  N1 <= 2048: the a and x columns in
// shared memory per CTA (F2); N1 = 2^(11+g): the first g forward and last g inverse column stages
// run from HBM (f2_top / f2_bottom) around 2048-point blocks in shared memory (2 CTAs per SM).  The NTT path stays
// the product headline (this one moves complex doubles: ~20 GB of HBM traffic per C3 matvec).
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hk_internal.h"

namespace hk {
namespace {

constexpr uint64_t kFftMagic = 0x484b464654504c4eull;  // "HKFFTPLN"
constexpr int kFftMaxLogN1 = 15, kFftMaxLogN2 = 13, kFftMinLog = 5;
constexpr int kFftPad = 1024;  // -K table entries past Ly

struct FftPlan {
    hk_fft_plan_info info;
    int64_t out_off;
    int32_t reverse_out, x_reversed, cyclic, fold;
    int32_t cb;                    // coefficient bias 2^cb
    size_t off_tw1, off_tw2, off_negk, off_A, off_X, off_end;
};

struct FftParams {
    int32_t kind, P, L, Ly, w, Ls, S2, log_n1, log_n2, N1, N2;
    int64_t m, n, a_count, out_off;
    int32_t reverse_out, x_reversed, fold, cb;
    uint64_t hash;
    WsHeader *hdr;
    const double2 *tw1, *tw2;      // N1 / N2 forward tables, entry h + j = exp(-2 pi i j / (2h))
    const uint64_t *negk;          // -(2^cb sum_{s < S2} 2^(w s)) mod 2^(64 Ly), zero-padded
    double2 *A, *X;                // [N1][N2] row-major (sigma contiguous)
    const uint64_t *a_mag, *x_mag;
    const int8_t *a_sign, *x_sign;
    uint64_t *y_mag;
    int8_t *y_sign;
    unsigned long long *resid;     // F3 accuracy study: max |v - rint(v)| over the coefficients
                                   // (bits of a non-negative double; nullptr in the product path)
};

// ---------------------------------------------------------------------------------------------
// complex arithmetic with explicit round-to-nearest DADD / DMUL (no contraction into DFMA)
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 w) {  // a * conj(w)
    return make_double2(__dadd_rn(__dmul_rn(a.x, w.x), __dmul_rn(a.y, w.y)),
                        __dsub_rn(__dmul_rn(a.y, w.x), __dmul_rn(a.x, w.y)));
}
__host__ __device__ __forceinline__ int cpad(int i) { return i + (i >> 3); }  // shared-memory padding
__device__ __forceinline__ void fcp_async16(double2 *smem, const double2 *gmem) {  // LDGSTS, 16 bytes
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// One radix-2^R pass over `batch` arrays of N = 2^LOGN points (array b at s + b * rs, point i at
// cpad(i)).  DIF (INV = false): stages h = S 2^(R-1) .. S, (u, v) -> (u + v, (u - v) w);
// DIT (INV = true): stages h = S .. S 2^(R-1), (u, v) -> (u + v conj(w), u - v conj(w)):
// natural -> bit-reversed -> natural, the DIT with conjugate roots being the unnormalised inverse.
template <int LOGN, int R, int S, bool INV>
__device__ void cfft_pass(double2 *s, int batch, int rs, const double2 *__restrict__ tw) {
    constexpr int N = 1 << LOGN, G = 1 << R, NG = N / G;
    for (int gi = threadIdx.x; gi < batch * NG; gi += blockDim.x) {
        const int b = gi / NG, g = gi % NG;
        const int j0 = g % S, B = (g / S) * (S * G);
        double2 *base = s + b * rs;
        double2 v[G];
#pragma unroll
        for (int m = 0; m < G; ++m) v[m] = base[cpad(B + j0 + m * S)];
        if (!INV) {
#pragma unroll
            for (int l = R - 1; l >= 0; --l) {
                const int half = 1 << l;
#pragma unroll
                for (int m = 0; m < G; ++m) {
                    if (m & half) continue;
                    const int j = j0 + S * (m & (half - 1));
                    const double2 d = csub(v[m], v[m + half]);
                    v[m] = cadd(v[m], v[m + half]);
                    v[m + half] = cmul(d, __ldg(tw + S * half + j));
                }
            }
        } else {
#pragma unroll
            for (int l = 0; l < R; ++l) {
                const int half = 1 << l;
#pragma unroll
                for (int m = 0; m < G; ++m) {
                    if (m & half) continue;
                    const int j = j0 + S * (m & (half - 1));
                    const double2 t = cmulc(v[m + half], __ldg(tw + S * half + j));
                    v[m + half] = csub(v[m], t);
                    v[m] = cadd(v[m], t);
                }
            }
        }
#pragma unroll
        for (int m = 0; m < G; ++m) base[cpad(B + j0 + m * S)] = v[m];
    }
    __syncthreads();
}
template <int LOGN, int HI>  // forward passes of radix <= 16 from the top
struct CDif {
    static __device__ void run(double2 *s, int batch, int rs, const double2 *tw) {
        if constexpr (HI > 0) {
            constexpr int R = HI < 4 ? HI : 4;
            cfft_pass<LOGN, R, (1 << (HI - R)), false>(s, batch, rs, tw);
            CDif<LOGN, HI - R>::run(s, batch, rs, tw);
        }
    }
};
template <int LOGN, int LO>  // inverse passes of radix <= 16 from the bottom
struct CDit {
    static __device__ void run(double2 *s, int batch, int rs, const double2 *tw) {
        if constexpr (LO < LOGN) {
            constexpr int R = (LOGN - LO) < 4 ? (LOGN - LO) : 4;
            cfft_pass<LOGN, R, (1 << LO), true>(s, batch, rs, tw);
            CDit<LOGN, LO + R>::run(s, batch, rs, tw);
        }
    }
};

constexpr int kFftThreads = 512;

// ---------------------------------------------------------------------------------------------
// F1: validation + balanced digits + forward row FFT (N2) of one entry of a or x per CTA
template <int LOGN2>
__global__ void __launch_bounds__(kFftThreads) f1_rows(FftParams prm) {
    constexpr int N2 = 1 << LOGN2;
    extern __shared__ double2 cs[];
    if (prm.hdr->magic != kFftMagic || prm.hdr->hash != prm.hash) {
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicMin(&prm.hdr->status, (int)HK_EINVAL);
        return;
    }
    const int64_t r = blockIdx.x;
    const bool is_x = r >= prm.a_count;
    const int64_t e = is_x ? r - prm.a_count : r;
    const uint64_t *mag = (is_x ? prm.x_mag : prm.a_mag) + e * prm.L;
    const int sg = (is_x ? prm.x_sign : prm.a_sign)[e];
    const int L = prm.L, w = prm.w, Ls = prm.Ls;
    {  // A1 validation: bits >= P zero, sign in {-1, 0, 1}, sign == 0 <=> magnitude == 0
        int nz = 0;
        for (int u = threadIdx.x; u < L; u += blockDim.x) nz |= mag[u] != 0;
        nz = __syncthreads_or(nz);
        if (threadIdx.x == 0) {
            const int rem = prm.P - 64 * (L - 1);
            const uint64_t topmask = rem >= 64 ? ~0ull : ((1ull << rem) - 1);
            if ((mag[L - 1] & ~topmask) || sg < -1 || sg > 1 || ((sg == 0) == (nz != 0)))
                atomicMin(&prm.hdr->status, (int)HK_ERANGE);
        }
    }
    auto field = [&](int t) -> int64_t {  // u_t = bits [w t, w t + w) of |m| (0 beyond P)
        if (t < 0 || t >= Ls) return 0;
        const int o = w * t, q = o >> 6, sh = o & 63;
        if (q >= L) return 0;
        const uint64_t l0 = mag[q], l1 = q + 1 < L ? mag[q + 1] : 0ull;
        const uint64_t v = sh ? ((l0 >> sh) | (l1 << (64 - sh))) : l0;
        return (int64_t)(v & ((1ull << w) - 1));
    };
    const int64_t half = int64_t(1) << (w - 1);
    for (int t = threadIdx.x; t < N2; t += blockDim.x) {
        double d = 0.0;
        if (t < Ls && sg != 0) {
            const int64_t u = field(t), up = field(t - 1);
            const int64_t dt = u - ((u >= half) ? (int64_t(1) << w) : 0) + (up >= half ? 1 : 0);
            d = (double)(sg * dt);  // |d| <= 2^(w-1): exact
        }
        cs[cpad(t)] = make_double2(d, 0.0);
    }
    __syncthreads();
    CDif<LOGN2, LOGN2>::run(cs, 1, 0, prm.tw2);
    const int64_t pos = is_x ? (prm.x_reversed ? prm.n - 1 - e : e) : e;
    double2 *out = (is_x ? prm.X : prm.A) + pos * N2;
    for (int t = threadIdx.x; t < N2; t += blockDim.x) out[t] = cs[cpad(t)];
}

// F2: per pair of columns: forward column FFTs (N1) of a and x, pointwise product, inverse FFT;
// the result replaces x's columns (all N1 rows)
// SPLIT (N1 > 2^LOGN1 = 2048): block blockIdx.y of 2048 consecutive rows after f2_top's first
// stages; the block is then an independent 2048-point transform (its stages' twiddles are the
// N1 table's first 2048 entries) and every row holds data (no zero masking)
constexpr int kF2Threads = 256, kF2LogBlock = 11;  // F2: 2048-row blocks, 2 CTAs (74 KB smem) per SM
template <int LOGN1, int TC, bool SPLIT>
__global__ void __launch_bounds__(kF2Threads, 2) f2_cols(FftParams prm) {
    constexpr int N1 = 1 << LOGN1, RS = N1 + N1 / 8;
    extern __shared__ double2 cs[];  // [2 arrays][TC columns][RS]
    const int sig0 = blockIdx.x * TC, N2 = prm.N2;
    const int64_t na = SPLIT ? N1 : prm.a_count, nx = SPLIT ? N1 : prm.n;
    const size_t row0 = SPLIT ? (size_t)blockIdx.y * N1 : 0;
    for (int e = threadIdx.x; e < N1 * TC; e += blockDim.x) {  // asynchronous 16-byte copies
        const int i = e / TC, c = e % TC;
        const size_t g = (row0 + i) * N2 + sig0 + c;
        double2 *da = &cs[c * RS + cpad(i)], *dx = &cs[(TC + c) * RS + cpad(i)];
        if (i < na) fcp_async16(da, prm.A + g); else *da = make_double2(0.0, 0.0);
        if (i < nx) fcp_async16(dx, prm.X + g); else *dx = make_double2(0.0, 0.0);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    CDif<LOGN1, LOGN1>::run(cs, 2 * TC, RS, prm.tw1);
    for (int e = threadIdx.x; e < N1 * TC; e += blockDim.x) {
        const int i = e / TC, c = e % TC;
        double2 &x = cs[(TC + c) * RS + cpad(i)];
        x = cmul(x, cs[c * RS + cpad(i)]);
    }
    __syncthreads();
    CDit<LOGN1, 0>::run(cs + TC * RS, TC, RS, prm.tw1);
    for (int e = threadIdx.x; e < N1 * TC; e += blockDim.x) {
        const int i = e / TC, c = e % TC;
        prm.X[(row0 + i) * N2 + sig0 + c] = cs[(TC + c) * RS + cpad(i)];
    }
}

// N1 = 2^(11 + GAMMA) > 2048: the first GAMMA forward stages (half-sizes N1/2 .. 2048) of the a and
// x columns from HBM, in place; thread item = (array, j0 < 2048, sigma), sigma fastest (coalesced)
template <int GAMMA>
__global__ void __launch_bounds__(256) f2_top(FftParams prm) {
    constexpr int G = 1 << GAMMA, S = 1 << kF2LogBlock;
    const int N2 = prm.N2;
    const int64_t items = (int64_t)2 * S * N2;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int sig = (int)(it % N2);
        const int64_t rest = it / N2;
        const int j0 = (int)(rest % S);
        const bool isx = rest >= S;
        double2 *arr = isx ? prm.X : prm.A;
        const int64_t cnt = isx ? prm.n : prm.a_count;
        double2 v[G];
#pragma unroll
        for (int m = 0; m < G; ++m) {
            const int64_t i = j0 + (int64_t)m * S;
            v[m] = i < cnt ? arr[i * N2 + sig] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int l = GAMMA - 1; l >= 0; --l) {
            const int half = 1 << l;
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & half) continue;
                const int j = j0 + S * (m & (half - 1));
                const double2 d = csub(v[m], v[m + half]);
                v[m] = cadd(v[m], v[m + half]);
                v[m + half] = cmul(d, __ldg(prm.tw1 + S * half + j));
            }
        }
#pragma unroll
        for (int m = 0; m < G; ++m) arr[(j0 + (int64_t)m * S) * N2 + sig] = v[m];
    }
}

// ... and the last GAMMA inverse stages (half-sizes 4096 .. N1/2) of the product, in place
template <int GAMMA>
__global__ void __launch_bounds__(256) f2_bottom(FftParams prm) {
    constexpr int G = 1 << GAMMA, S = 1 << kF2LogBlock;
    const int N2 = prm.N2;
    const int64_t items = (int64_t)S * N2;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int sig = (int)(it % N2);
        const int j0 = (int)(it / N2);
        double2 v[G];
#pragma unroll
        for (int m = 0; m < G; ++m) v[m] = prm.X[(j0 + (int64_t)m * S) * N2 + sig];
#pragma unroll
        for (int l = 0; l < GAMMA; ++l) {
            const int half = 1 << l;
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & half) continue;
                const int j = j0 + S * (m & (half - 1));
                const double2 t = cmulc(v[m + half], __ldg(prm.tw1 + S * half + j));
                v[m + half] = csub(v[m], t);
                v[m] = cadd(v[m], t);
            }
        }
#pragma unroll
        for (int m = 0; m < G; ++m) prm.X[(j0 + (int64_t)m * S) * N2 + sig] = v[m];
    }
}

// F3: per output row: inverse row FFT (both folded rows for a non-cyclic circulant), rint of the
// scaled real parts (exact by the planner's bound), biased coefficients, carry, sign-magnitude y
template <int LOGN2>
__global__ void __launch_bounds__(kFftThreads) f3_finish(FftParams prm) {
    constexpr int N2 = 1 << LOGN2, T = kFftThreads;
    extern __shared__ double2 cs[];
    __shared__ int s_wg[T / 32], s_wc[T / 32];
    __shared__ int s_neg, s_zmin;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t i = blockIdx.x;  // output row (internal order)
    const int N1 = prm.N1, S2 = prm.S2, Ly = prm.Ly, w = prm.w;
    const double scale = 1.0 / ((double)N1 * (double)N2);  // a power of two: exact
    uint64_t *coef = reinterpret_cast<uint64_t *>(cs + cpad(N2));  // [N2] biased coefficients
    const int nrep = prm.fold ? 2 : 1;
    for (int rep = 0; rep < nrep; ++rep) {
        const int64_t pos = (prm.out_off + i + (rep ? prm.n : 0)) & (N1 - 1);
        const double2 *src = prm.X + pos * N2;
        for (int t = tid; t < N2; t += T) fcp_async16(&cs[cpad(t)], src + t);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        CDit<LOGN2, 0>::run(cs, 1, 0, prm.tw2);
        double rmax = 0.0;
        for (int t = tid; t < N2; t += T) {
            const double v = cs[cpad(t)].x * scale, r = rint(v);
            const int64_t c = (int64_t)r;
            rmax = fmax(rmax, fabs(v - r));
            if (rep == 0) coef[t] = (uint64_t)c + (t < S2 ? (1ull << prm.cb) : 0ull);
            else coef[t] += (uint64_t)c;
        }
        if (prm.resid) {  // study only: one atomic per warp (non-negative doubles order as integers)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
            if (lane == 0) atomicMax(prm.resid, (unsigned long long)__double_as_longlong(rmax));
        }
        __syncthreads();
    }
    // limbs: thread owns CHL consecutive limbs; T_q = sum of c_s 2^(w s - 64 q) over s with
    // floor(w s / 64) = q (unsigned 128-bit); limb q = lo(T_q) + hi(T_(q-1)) + (-K)_q
    constexpr int CHL = 5;  // >= ceil(kK3MaxLy / T)
    const int l0 = tid * CHL;
    auto tq = [&](int q, uint64_t &lo, uint64_t &hi) {
        lo = hi = 0;
        if (q < 0) return;
        const int s_lo = (64 * q + w - 1) / w, s_hi = (64 * q + 63) / w;  // w s in [64 q, 64 q + 63]
        for (int s = s_lo; s <= s_hi && s < S2; ++s) {
            const uint64_t c = coef[s];
            const int b = w * s - 64 * q;
            const uint64_t plo = c << b, phi = b ? (c >> (64 - b)) : 0ull;
            lo += plo;
            hi += phi + (lo < plo);
        }
    };
    uint64_t u[CHL];
    int e[CHL];
    uint64_t plo, phi;
    tq(l0 - 1, plo, phi);
#pragma unroll
    for (int c = 0; c < CHL; ++c) {
        uint64_t lo, hi;
        tq(l0 + c, lo, hi);
        const uint64_t nk = l0 + c < Ly ? prm.negk[l0 + c] : 0ull;
        uint64_t v = lo + phi;
        int cnt = v < lo;
        const uint64_t v2 = v + nk;
        cnt += v2 < v;
        u[c] = v2;
        e[c] = cnt;
        phi = hi;
    }
    // binary lookahead: w_c = u_c + e_(c-1) (the previous thread's last e for c = 0)
    __shared__ int8_t s_e[T];
    s_e[tid] = (int8_t)e[CHL - 1];
    if (tid == 0) { s_neg = 0; s_zmin = INT_MAX; }
    __syncthreads();
    uint32_t gb = 0, pb = 0;
    int G = 0, Pp = 1;
#pragma unroll
    for (int c = 0; c < CHL; ++c) {
        const uint64_t ein = c == 0 ? (tid > 0 ? (uint64_t)s_e[tid - 1] : 0ull) : (uint64_t)e[c - 1];
        const uint64_t v = u[c] + ein;
        const int g = v < u[c], p = v == ~0ull;
        u[c] = v;
        gb |= (uint32_t)g << c;
        pb |= (uint32_t)p << c;
        G = g | (p & G);
        Pp &= p;
    }
    int incl = G | (Pp << 1);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl = ((incl | ((incl >> 1) & o)) & 1) | ((incl & o) & 2);
    }
    if (lane == 31) s_wg[warp] = incl;
    __syncthreads();
    if (tid == 0) {
        int c = 0;
        for (int wi = 0; wi < T / 32; ++wi) {
            s_wc[wi] = c;
            c = (s_wg[wi] & 1) | ((s_wg[wi] >> 1) & c);
        }
    }
    __syncthreads();
    const int prev = __shfl_up_sync(0xffffffffu, incl, 1);
    int carry = s_wc[warp];
    if (lane > 0) carry = (prev & 1) | ((prev >> 1) & carry);
#pragma unroll
    for (int c = 0; c < CHL; ++c) {
        u[c] += (uint64_t)carry;
        carry = ((gb >> c) & 1) | ((pb >> c) & carry);
    }
    int zloc = INT_MAX;
#pragma unroll
    for (int c = CHL - 1; c >= 0; --c) zloc = (l0 + c < Ly && u[c]) ? l0 + c : zloc;
    if (zloc < Ly) atomicMin(&s_zmin, zloc);
#pragma unroll
    for (int c = 0; c < CHL; ++c)
        if (l0 + c == Ly - 1) s_neg = (int)(u[c] >> 63);
    __syncthreads();
    const bool neg = s_neg != 0;
    const int zmin = s_zmin;
    const uint64_t msk = neg ? ~0ull : 0ull;
    const int64_t orow = prm.reverse_out ? prm.m - 1 - i : i;
    uint64_t *yo = prm.y_mag + orow * Ly;
#pragma unroll
    for (int c = 0; c < CHL; ++c)
        if (l0 + c < Ly) yo[l0 + c] = (u[c] ^ msk) + (uint64_t)(neg && l0 + c <= zmin);
    if (tid == 0) prm.y_sign[orow] = neg ? (int8_t)-1 : (zmin < Ly ? (int8_t)1 : (int8_t)0);
}

__global__ void f0_header(WsHeader *hdr, uint64_t hash) {
    hdr->magic = kFftMagic;
    hdr->hash = hash;
    hdr->status = HK_OK;
    hdr->a_ready = 0;
}

// ---------------------------------------------------------------------------------------------
// host: planner with the Percival bound, workspace, launches
size_t align256f(size_t x) { return (x + 255) & ~size_t(255); }

long double percival_factor(int k, long double eps, long double beta) {
    // (1+e)^3k (1+e sqrt5)^(3k+1) (1+b)^3k - 1
    const long double lg = 3.0L * k * log1pl(eps) + (3.0L * k + 1.0L) * log1pl(eps * sqrtl(5.0L)) +
                           3.0L * k * log1pl(beta);
    return expm1l(lg);
}

uint64_t fft_hash(int32_t kind, int64_t n, int32_t P, int32_t w) {
    uint64_t h = 1469598103934665603ull ^ 0x464654ull;
    auto mix = [&](uint64_t v) {
        for (int i = 0; i < 8; ++i) { h ^= (v >> (8 * i)) & 0xff; h *= 1099511628211ull; }
    };
    mix((uint64_t)kind); mix((uint64_t)n); mix((uint64_t)P); mix((uint64_t)w);
    return h;
}

// w_force = 0: the widest w whose Percival bound is <= 0.49 (the exact product path);
// w_force > 0 (F3 accuracy study, hk_fft_plan_w): that digit width, whatever its bound (reported),
// as long as the transform fits and |coefficient| < 2^62 (the bias / carry arithmetic)
int fft_plan(int32_t kind, int64_t n, int32_t P, FftPlan *pl, int32_t w_force = 0) {
    if (kind < HK_HANKEL || kind > HK_CIRCULANT || n < 1 || P < 1 || w_force < 0 || w_force > 30) return HK_EINVAL;
    std::memset(pl, 0, sizeof(*pl));
    hk_fft_plan_info &in = pl->info;
    in.kind = kind; in.P = P; in.m = n; in.n = n;
    in.L = (P + 63) / 64;
    in.Ly = 2 * in.L + 1;
    in.a_count = kind == HK_CIRCULANT ? n : 2 * n - 1;
    if (in.Ly > kK3MaxLy) return HK_EUNSUPPORTED;
    int64_t need;
    if (kind == HK_CIRCULANT) {
        const bool pow2 = (n & (n - 1)) == 0;
        if (pow2 && n >= (1 << kFftMinLog)) { in.cyclic = 1; need = n; }
        else { in.fold = 1; need = 2 * n - 1; }
        pl->x_reversed = 0;
        pl->out_off = 0;
    } else {
        need = in.a_count;
        pl->x_reversed = 1;
        pl->out_off = n - 1;
    }
    pl->reverse_out = kind == HK_TOEPLITZ;
    pl->cyclic = in.cyclic; pl->fold = in.fold;
    int lg1 = kFftMinLog;
    while ((int64_t(1) << lg1) < need) ++lg1;
    if (lg1 > kFftMaxLogN1) return HK_EUNSUPPORTED;
    in.log_n1 = lg1;
    in.eps = std::ldexp(1.0, -53);
    in.beta = std::ldexp(1.0, -52);
    const long double rows_a = (long double)in.a_count;
    bool found = false;
    for (int w = w_force ? w_force : 30; w >= 2 && !found; --w) {
        if (w_force && w != w_force) break;
        const int64_t Ls = (P + w - 1) / w + 1;
        int lg2 = kFftMinLog;
        while ((int64_t(1) << lg2) < 2 * Ls - 1) ++lg2;
        if (lg2 > kFftMaxLogN2) continue;
        const int k = lg1 + lg2;
        const long double dmax = ldexpl(1.0L, w - 1);
        const long double norm = sqrtl(rows_a * (long double)n) * (long double)Ls * dmax * dmax;
        const long double B = norm * percival_factor(k, in.eps, in.beta);
        const long double cmax = (long double)n * (long double)Ls * dmax * dmax;  // |c_s| bound
        if (w_force ? cmax < ldexpl(1.0L, 62) : (B <= 0.49L && cmax < ldexpl(1.0L, 52))) {
            in.w = w; in.Ls = (int32_t)Ls; in.log_n2 = lg2; in.bound = (double)B;
            int cb = 0;
            while (ldexpl(1.0L, cb) <= cmax) ++cb;
            pl->cb = cb;
            found = true;
        }
    }
    if (!found) return HK_EUNSUPPORTED;
    const size_t N1 = size_t(1) << in.log_n1, N2 = size_t(1) << in.log_n2;
    size_t off = align256f(sizeof(WsHeader));
    pl->off_tw1 = off; off = align256f(off + N1 * sizeof(double2));
    pl->off_tw2 = off; off = align256f(off + N2 * sizeof(double2));
    pl->off_negk = off; off = align256f(off + (size_t)(in.Ly + kFftPad) * sizeof(uint64_t));
    pl->off_A = off; off = align256f(off + N1 * N2 * sizeof(double2));
    pl->off_X = off; off = align256f(off + N1 * N2 * sizeof(double2));
    pl->off_end = off;
    in.ws_bytes = off;
    return HK_OK;
}

void fft_fill(const FftPlan &pl, void *ws, FftParams *prm) {
    std::memset(prm, 0, sizeof(*prm));
    const hk_fft_plan_info &in = pl.info;
    prm->kind = in.kind; prm->P = in.P; prm->L = in.L; prm->Ly = in.Ly; prm->w = in.w; prm->Ls = in.Ls;
    prm->S2 = 2 * in.Ls - 1;
    prm->log_n1 = in.log_n1; prm->log_n2 = in.log_n2;
    prm->N1 = 1 << in.log_n1; prm->N2 = 1 << in.log_n2;
    prm->m = in.m; prm->n = in.n; prm->a_count = in.a_count; prm->out_off = pl.out_off;
    prm->reverse_out = pl.reverse_out; prm->x_reversed = pl.x_reversed; prm->fold = pl.fold;
    prm->cb = pl.cb;
    prm->hash = fft_hash(in.kind, in.n, in.P, in.w);
    char *base = (char *)ws;
    prm->hdr = (WsHeader *)base;
    prm->tw1 = (const double2 *)(base + pl.off_tw1);
    prm->tw2 = (const double2 *)(base + pl.off_tw2);
    prm->negk = (const uint64_t *)(base + pl.off_negk);
    prm->A = (double2 *)(base + pl.off_A);
    prm->X = (double2 *)(base + pl.off_X);
}

std::vector<double2> twiddle_table(int logn) {  // entry h + j = exp(-2 pi i j / (2h)), long double
    const size_t N = size_t(1) << logn;
    std::vector<double2> t(N);
    t[0] = make_double2(1.0, 0.0);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (size_t h = 1; h < N; h <<= 1)
        for (size_t j = 0; j < h; ++j) {
            const long double a = -pi * (long double)j / (long double)h;
            t[h + j] = make_double2((double)cosl(a), (double)sinl(a));
        }
    return t;
}

std::vector<uint64_t> fft_negk(const FftPlan &pl) {  // -(2^cb sum_{s < S2} 2^(w s)) mod 2^(64 Ly)
    const hk_fft_plan_info &in = pl.info;
    const int Ly = in.Ly, w = in.w, S2 = 2 * in.Ls - 1;
    std::vector<uint32_t> acc((size_t)2 * Ly + 4, 0);
    for (int64_t s = 0; s < S2; ++s) {
        const int64_t bit = (int64_t)w * s + pl.cb;
        if (bit >= 64ll * Ly) break;
        size_t wd = (size_t)(bit >> 5);
        uint64_t carry = (uint64_t)1 << (bit & 31);
        while (carry && wd < acc.size()) {
            const uint64_t t = (uint64_t)acc[wd] + carry;
            acc[wd] = (uint32_t)t;
            carry = t >> 32;
            ++wd;
        }
    }
    std::vector<uint64_t> out((size_t)Ly + kFftPad, 0);
    uint64_t c = 1;
    for (int l = 0; l < Ly; ++l) {
        const uint64_t v = ~((uint64_t)acc[2 * l] | ((uint64_t)acc[2 * l + 1] << 32));
        const uint64_t r = v + c;
        c = (c && r == 0) ? 1 : 0;
        out[l] = r;
    }
    return out;
}

int fft_check_launch() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "hk fft: CUDA launch error: %s\n", cudaGetErrorString(e));
        return HK_ECUDA;
    }
    return HK_OK;
}

template <int LOGN2>
int launch_rows_fft(const FftParams &prm, cudaStream_t st) {
    const size_t sm = (size_t)(cpad(1 << LOGN2) + 8) * sizeof(double2);
    if (cudaFuncSetAttribute(f1_rows<LOGN2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return HK_ECUDA;
    f1_rows<LOGN2><<<(unsigned)(prm.a_count + prm.n), kFftThreads, sm, st>>>(prm);
    return fft_check_launch();
}
template <int LOGN1>
int launch_cols_fft(const FftParams &prm, cudaStream_t st) {
    constexpr bool SPLIT = LOGN1 > kF2LogBlock;
    constexpr int LB = SPLIT ? kF2LogBlock : LOGN1, TC = LB >= kF2LogBlock ? 1 : 2;
    const size_t sm = (size_t)2 * TC * ((1 << LB) + (1 << LB) / 8) * sizeof(double2);
    if (cudaFuncSetAttribute(f2_cols<LB, TC, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return HK_ECUDA;
    constexpr int GAMMA = SPLIT ? LOGN1 - kF2LogBlock : 0;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    if constexpr (SPLIT) {
        f2_top<GAMMA><<<(unsigned)(nsm * 8), 256, 0, st>>>(prm);
        if (const int rc = fft_check_launch()) return rc;
    }
    f2_cols<LB, TC, SPLIT><<<dim3((unsigned)(prm.N2 / TC), 1u << GAMMA), kF2Threads, sm, st>>>(prm);
    if (const int rc = fft_check_launch()) return rc;
    if constexpr (SPLIT) {
        f2_bottom<GAMMA><<<(unsigned)(nsm * 8), 256, 0, st>>>(prm);
        return fft_check_launch();
    }
    return HK_OK;
}
template <int LOGN2>
int launch_finish_fft(const FftParams &prm, cudaStream_t st) {
    const size_t sm = (size_t)(cpad(1 << LOGN2) + 8) * sizeof(double2) + (size_t)(1 << LOGN2) * sizeof(uint64_t);
    if (cudaFuncSetAttribute(f3_finish<LOGN2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return HK_ECUDA;
    f3_finish<LOGN2><<<(unsigned)prm.m, kFftThreads, sm, st>>>(prm);
    return fft_check_launch();
}

int fft_dbg(const char *what, cudaStream_t st) {
    static const bool on = getenv("HK_FFT_DEBUG") != nullptr;
    if (!on) return HK_OK;
    const cudaError_t e = cudaStreamSynchronize(st);
    fprintf(stderr, "hk fft debug: after %s: %s\n", what, cudaGetErrorString(e));
    return e == cudaSuccess ? HK_OK : HK_ECUDA;
}

int fft_run(const FftParams &prm, cudaStream_t st) {
    int rc = HK_OK;
    if (fft_dbg("start", st)) return HK_ECUDA;
    switch (prm.log_n2) {
#define HK_C(LG) case LG: rc = launch_rows_fft<LG>(prm, st); break;
        HK_C(5) HK_C(6) HK_C(7) HK_C(8) HK_C(9) HK_C(10) HK_C(11) HK_C(12) HK_C(13)
#undef HK_C
        default: return HK_EUNSUPPORTED;
    }
    if (rc || (rc = fft_dbg("F1 rows", st))) return rc;
    switch (prm.log_n1) {
#define HK_C(LG) case LG: rc = launch_cols_fft<LG>(prm, st); break;
        HK_C(5) HK_C(6) HK_C(7) HK_C(8) HK_C(9) HK_C(10) HK_C(11) HK_C(12) HK_C(13) HK_C(14) HK_C(15)
#undef HK_C
        default: return HK_EUNSUPPORTED;
    }
    if (rc || (rc = fft_dbg("F2 columns", st))) return rc;
    switch (prm.log_n2) {
#define HK_C(LG) case LG: return launch_finish_fft<LG>(prm, st);
        HK_C(5) HK_C(6) HK_C(7) HK_C(8) HK_C(9) HK_C(10) HK_C(11) HK_C(12) HK_C(13)
#undef HK_C
        default: return HK_EUNSUPPORTED;
    }
}

bool ranges_overlap(const void *a, size_t na, const void *b, size_t nb) {
    const char *pa = (const char *)a, *pb = (const char *)b;
    return pa < pb + nb && pb < pa + na;
}

}  // namespace
}  // namespace hk

using namespace hk;

extern "C" {

int32_t hk_fft_plan_w(int32_t kind, int64_t n, int32_t P, int32_t w, hk_fft_plan_info *out) {
    if (!out) return HK_EINVAL;
    FftPlan pl;
    const int rc = fft_plan(kind, n, P, &pl, w);
    if (rc) return rc;
    *out = pl.info;
    return HK_OK;
}

int32_t hk_fft_plan(int32_t kind, int64_t n, int32_t P, hk_fft_plan_info *out) {
    return hk_fft_plan_w(kind, n, P, 0, out);
}

int32_t hk_fft_workspace_init_w(int32_t kind, int64_t n, int32_t P, int32_t w, void *ws, size_t ws_bytes,
                                void *stream) {
    HK_NVTX("hk_fft_workspace_init");
    if (!ws || ((uintptr_t)ws & 255) != 0) return HK_EINVAL;
    FftPlan pl;
    int rc = fft_plan(kind, n, P, &pl, w);
    if (rc) return rc;
    if (ws_bytes < pl.info.ws_bytes) return HK_ENOMEM;
    FftParams prm;
    fft_fill(pl, ws, &prm);
    cudaStream_t st = (cudaStream_t)stream;
    const std::vector<double2> t1 = twiddle_table(pl.info.log_n1), t2 = twiddle_table(pl.info.log_n2);
    const std::vector<uint64_t> nk = fft_negk(pl);
    char *base = (char *)ws;
    if (cudaMemcpyAsync(base + pl.off_tw1, t1.data(), t1.size() * sizeof(double2), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(base + pl.off_tw2, t2.data(), t2.size() * sizeof(double2), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(base + pl.off_negk, nk.data(), nk.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemsetAsync(base + pl.off_A, 0, pl.off_end - pl.off_A, st) != cudaSuccess)
        return HK_ECUDA;
    f0_header<<<1, 1, 0, st>>>(prm.hdr, prm.hash);
    return fft_check_launch();
}

int32_t hk_fft_workspace_init(int32_t kind, int64_t n, int32_t P, void *ws, size_t ws_bytes, void *stream) {
    return hk_fft_workspace_init_w(kind, n, P, 0, ws, ws_bytes, stream);
}

int32_t hk_fft_matvec_w(int32_t kind, int64_t n, int32_t P, int32_t w, const uint64_t *a_mag,
                        const int8_t *a_sign, const uint64_t *x_mag, const int8_t *x_sign, uint64_t *y_mag,
                        int8_t *y_sign, void *ws, size_t ws_bytes, void *stream, double *max_residual) {
    HK_NVTX("hk_fft_matvec");
    if (!a_mag || !a_sign || !x_mag || !x_sign || !y_mag || !y_sign || !ws || ((uintptr_t)ws & 255) != 0 ||
        ((uintptr_t)max_residual & 7) != 0)
        return HK_EINVAL;
    FftPlan pl;
    int rc = fft_plan(kind, n, P, &pl, w);
    if (rc) return rc;
    if (ws_bytes < pl.info.ws_bytes) return HK_ENOMEM;
    const size_t Ly = pl.info.Ly, L = pl.info.L, na = pl.info.a_count;
    if (ranges_overlap(y_mag, n * Ly * 8, a_mag, na * L * 8) || ranges_overlap(y_mag, n * Ly * 8, x_mag, n * L * 8) ||
        ranges_overlap(y_sign, n, a_sign, na) || ranges_overlap(y_sign, n, x_sign, n) ||
        ranges_overlap(y_mag, n * Ly * 8, ws, pl.info.ws_bytes) || ranges_overlap(y_sign, n, ws, pl.info.ws_bytes))
        return HK_EINVAL;
    FftParams prm;
    fft_fill(pl, ws, &prm);
    prm.a_mag = a_mag; prm.a_sign = a_sign; prm.x_mag = x_mag; prm.x_sign = x_sign;
    prm.y_mag = y_mag; prm.y_sign = y_sign;
    prm.resid = reinterpret_cast<unsigned long long *>(max_residual);
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(&prm.hdr->status, 0, sizeof(int32_t), st) != cudaSuccess) return HK_ECUDA;
    return fft_run(prm, st);
}

int32_t hk_fft_matvec(int32_t kind, int64_t n, int32_t P, const uint64_t *a_mag, const int8_t *a_sign,
                      const uint64_t *x_mag, const int8_t *x_sign, uint64_t *y_mag, int8_t *y_sign,
                      void *ws, size_t ws_bytes, void *stream) {
    return hk_fft_matvec_w(kind, n, P, 0, a_mag, a_sign, x_mag, x_sign, y_mag, y_sign, ws, ws_bytes, stream,
                           nullptr);
}

}  // extern "C"
