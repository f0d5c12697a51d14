// tc_ntt_stage.cu -- SURVEY.md 8(f) F4 microbenchmark: one radix-32 NTT stage on the 5th-gen tensor
// cores (tcgen05.mma kind::i8, accumulators in TMEM) against the same stage as radix-2 butterflies on
// the integer pipes.  PAPER.md P:112 ("multiplication cost dominates"): can int8 tensor-core DFT stages
// lift the integer-pipe ceiling of the exact NTT path (DESIGN.md section 12 cost model)?
//
// The stage, for every group n of 32 residues x_j mod p (p = 2147352577, the path's first prime):
//     Y[n][k] = T[n][k] * sum_j w^(jk) x_j  (mod p),   w a primitive 32nd root of unity,
// T[n][k] an arbitrary twiddle (the inter-stage twiddle of a four-step NTT).
//
// Tensor-core form (exact): split x_j = sum_b 2^(8b) X_b[j] (bytes, b < 4) and each of the four matrices
// F^(b)[k][j] = 2^(8b) w^(jk) mod p into bytes F^(b)_c (c < 4).  Then
//     Y[n][k] = sum_c 2^(8c) D[n][4k + c],   D[n][4k + c] = sum_{b, j} X_b[n][j] F^(b)_c[k][j]
// i.e. ONE u8 x u8 -> s32 GEMM D (M = 128 groups) x (N = 128 = 32 k x 4 c) with K = 128 (4 byte planes x
// 32 points); every D entry < 128 * 255^2 < 2^23.  A = the groups' bytes (K-major), B = the constant
// byte planes (K-major), D in TMEM: each thread reads its group's 4 partial sums of each k from its own
// TMEM lane and reduces L + 2^16 H (L = D0 + 2^8 D1, H = D2 + 2^8 D3, both < 2^32) mod p with two Shoup
// products, then applies T with a third.
//
// Both kernels keep a tile of 128 groups in shared memory and apply the stage REPS times to it (the
// output of one repetition is the next one's input), so the timing is the stage's on-chip throughput
// (no HBM).  One launch of each checks the first repetition against a host reference.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o scripts/tc_ntt_stage scripts/tc_ntt_stage.cu
//   scripts/tc_ntt_stage [reps]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr uint32_t P = 2147352577u;
constexpr int NG = 128;         // groups per tile (MMA M)
constexpr int NK = 32;          // points per group (radix)
constexpr int KB = 4 * NK;      // K bytes: 4 byte planes x 32 points
constexpr int MMA_N = 4 * NK;   // 32 outputs x 4 byte planes of F
constexpr int THREADS = 128;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t red1(uint32_t x, uint32_t p) { return min(x, x - p); }
__device__ __forceinline__ uint32_t addm(uint32_t a, uint32_t b, uint32_t p) { return red1(a + b, p); }
__device__ __forceinline__ uint32_t shoup(uint32_t x, uint32_t w, uint32_t wq, uint32_t p) {
    return x * w - __umulhi(x, wq) * p;  // [0, 2p) for every 32-bit x
}
__device__ __forceinline__ void gs(uint32_t &u, uint32_t &v, uint32_t w, uint32_t wq, uint32_t p) {
    const uint32_t d = u - v + p;
    u = addm(u, v, p);
    v = red1(shoup(d, w, wq, p), p);
}

// shared-memory offset of element (row, kbyte) of a K-major operand with 128 K bytes in the canonical
// no-swizzle UMMA layout: 8-row x 16-byte core matrices, K-adjacent cores 128 B apart (LBO), 8-row
// groups 1024 B apart (SBO)
__host__ __device__ constexpr uint32_t kmaj_off(uint32_t row, uint32_t kb) {
    return (row >> 3) * 1024u + (kb >> 4) * 128u + (row & 7u) * 16u + (kb & 15u);
}
__device__ __forceinline__ uint64_t smem_desc(const void *p) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    return (uint64_t)((a & 0x3FFFFu) >> 4) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(1024u >> 4) << 32) |
           (1ull << 46);  // version 1 (sm_100), base offset 0, SWIZZLE_NONE
}
// instruction descriptor: D s32, A u8, B u8, both K-major, N = 128, M = 128
constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(MMA_N >> 3) << 17) |
                            ((uint32_t)(NG >> 4) << 24);

constexpr int TPAD = NK + 4;  // tile row stride (words): 144 B, an odd number of 16-byte units
struct TcSmem {
    uint32_t tile[NG][TPAD];               // 18 KB: current residues
    alignas(1024) uint8_t a[NG * KB];      // 16 KB: A operand (group bytes)
    alignas(1024) uint8_t b[MMA_N * KB];   // 16 KB: B operand (constant F byte planes)
    uint32_t tw[NK][NG], twq[NK][NG];      // 32 KB: twiddles + Shoup quotients, [k][group]
    alignas(8) uint64_t mbar;
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(THREADS, 1) tc_stage(const uint32_t *x_in, uint32_t *y_out, const uint8_t *bmat,
                                                        const uint32_t *tw, const uint32_t *twq, int reps,
                                                        uint32_t r16, uint32_t r16q, uint32_t onq) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    TcSmem &S = *reinterpret_cast<TcSmem *>(smraw);
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t *xin = x_in + (size_t)blockIdx.x * NG * NK;
    for (int i = tid; i < NG * NK; i += THREADS) {
        S.tile[i / NK][i % NK] = xin[i];
        S.tw[i % NK][i / NK] = tw[(size_t)blockIdx.x * NG * NK + i];
        S.twq[i % NK][i / NK] = twq[(size_t)blockIdx.x * NG * NK + i];
    }
    for (int i = tid; i < MMA_N * KB / 16; i += THREADS)
        reinterpret_cast<uint4 *>(S.b)[i] = reinterpret_cast<const uint4 *>(bmat)[i];
    if (warp == 0) {  // TMEM: 128 columns x 128 lanes of s32 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&S.tmem_base)), "n"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&S.mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = S.tmem_base;
    const int n = tid;  // this thread's group (= its TMEM lane)
    for (int rep = 0; rep < reps; ++rep) {
        // (1) A operand: the bytes of this group's 32 residues, plane b at K bytes [32 b, 32 b + 32)
        {
            uint32_t x[NK];
#pragma unroll
            for (int q = 0; q < NK / 4; ++q) {
                const uint4 v = reinterpret_cast<const uint4 *>(&S.tile[n][0])[q];
                x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // K bytes 32 b + 16 h .. + 15: one 16-byte core row
                    uint32_t w4[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int j = 16 * h + 4 * q;
                        const uint32_t lo = __byte_perm(x[j], x[j + 1], 0x0040 + b * 0x0011);    // bytes b of x_j, x_j+1
                        const uint32_t hi = __byte_perm(x[j + 2], x[j + 3], 0x0040 + b * 0x0011);
                        w4[q] = __byte_perm(lo, hi, 0x5410);
                    }
                    *reinterpret_cast<uint4 *>(S.a + kmaj_off(n, 32 * b + 16 * h)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                }
            }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> tensor core
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        // (2) D = A B^T: four K = 32 MMAs issued by one thread, completion on the mbarrier
        if (tid == 0) {
#pragma unroll
            for (int ks = 0; ks < KB / 32; ++ks) {
                const uint64_t da = smem_desc(S.a + 256 * ks), db = smem_desc(S.b + 256 * ks);
                const uint32_t acc = ks > 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(&S.mbar))
                         : "memory");
        }
        {
            const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&S.mbar);
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
                             : "=r"(done) : "r"(mb), "r"((uint32_t)(rep & 1)) : "memory");
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        // (3) epilogue: lane n of TMEM holds D[n][4k + c]; 16 columns (4 outputs k) per load
#pragma unroll
        for (int kq = 0; kq < NK / 4; ++kq) {
            uint32_t d[16];
            const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(16 * kq);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
                : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                  "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
                : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            uint32_t y4[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int k = 4 * kq + t;
                const uint32_t L = d[4 * t] + (d[4 * t + 1] << 8);      // < 2^23 + 2^31
                const uint32_t H = d[4 * t + 2] + (d[4 * t + 3] << 8);  // weight 2^16
                const uint32_t v = addm(red1(shoup(H, r16, r16q, P), P), red1(shoup(L, 1u, onq, P), P), P);
                y4[t] = red1(shoup(v, S.tw[k][n], S.twq[k][n], P), P);
            }
            *reinterpret_cast<uint4 *>(&S.tile[n][4 * kq]) = make_uint4(y4[0], y4[1], y4[2], y4[3]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();  // TMEM reads done before the next MMA; tile rows are thread-private
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    uint32_t *yo = y_out + (size_t)blockIdx.x * NG * NK;
    for (int i = tid; i < NG * NK; i += THREADS) yo[i] = S.tile[i / NK][i % NK];
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(128));
}

// the same stage on the integer pipes: radix-2 DIF (GS) over the 32 points in registers (output in
// bit-reversed order, which the next stage of a four-step NTT would index accordingly), then T
struct AluSmem {
    uint32_t tile[NG][NK + 1];
    uint32_t w[NK], wq[NK];                // w^j, j < 16 (table entries h + j as in the NTT path)
    uint32_t tw[NK][NG], twq[NK][NG];      // [k][group]: consecutive lanes, consecutive banks
};
__global__ void __launch_bounds__(THREADS, 1) alu_stage(const uint32_t *x_in, uint32_t *y_out, const uint32_t *wt,
                                                         const uint32_t *wtq, const uint32_t *tw, const uint32_t *twq,
                                                         int reps) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    AluSmem &S = *reinterpret_cast<AluSmem *>(smraw);
    const int tid = threadIdx.x;
    for (int i = tid; i < NG * NK; i += THREADS) {
        S.tile[i / NK][i % NK] = x_in[(size_t)blockIdx.x * NG * NK + i];
        S.tw[i % NK][i / NK] = tw[(size_t)blockIdx.x * NG * NK + i];
        S.twq[i % NK][i / NK] = twq[(size_t)blockIdx.x * NG * NK + i];
    }
    if (tid < NK) { S.w[tid] = wt[tid]; S.wq[tid] = wtq[tid]; }
    __syncthreads();
    const int n = tid;
    for (int rep = 0; rep < reps; ++rep) {
        uint32_t v[NK];
#pragma unroll
        for (int j = 0; j < NK; ++j) v[j] = S.tile[n][j];
#pragma unroll
        for (int l = 4; l >= 0; --l) {  // half-size h = 2^l, twiddle w_(2h)^j = table[h + j]
            const int h = 1 << l;
#pragma unroll
            for (int m = 0; m < NK; ++m) {
                if (m & h) continue;
                const int j = m & (h - 1);
                if (j == 0) {
                    const uint32_t d = red1(v[m] - v[m + h] + P, P);
                    v[m] = addm(v[m], v[m + h], P);
                    v[m + h] = d;
                } else {
                    gs(v[m], v[m + h], S.w[h + j], S.wq[h + j], P);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NK; ++k) S.tile[n][k] = red1(shoup(v[k], S.tw[k][n], S.twq[k][n], P), P);
    }
    __syncthreads();
    for (int i = tid; i < NG * NK; i += THREADS) y_out[(size_t)blockIdx.x * NG * NK + i] = S.tile[i / NK][i % NK];
}

// ---------------------------------------------------------------------------------------------- host
static uint32_t mulm(uint32_t a, uint32_t b) { return (uint32_t)((uint64_t)a * b % P); }
static uint32_t powm(uint32_t b, uint64_t e) {
    uint32_t r = 1;
    while (e) { if (e & 1) r = mulm(r, b); b = mulm(b, b); e >>= 1; }
    return r;
}
static uint32_t shq(uint32_t w) { return (uint32_t)(((uint64_t)w << 32) / P); }
static int bitrev5(int k) { int r = 0; for (int i = 0; i < 5; ++i) r |= ((k >> i) & 1) << (4 - i); return r; }

int main(int argc, char **argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 4000;
    int dev = 0, nsm = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    // primitive root of P (P - 1 = 2^17 * 3^? ...): smallest g with g^((P-1)/q) != 1 for its prime factors
    uint32_t g = 2;
    {
        std::vector<uint32_t> f;
        uint32_t r = P - 1;
        for (uint32_t d = 2; (uint64_t)d * d <= r; ++d) if (r % d == 0) { f.push_back(d); while (r % d == 0) r /= d; }
        if (r > 1) f.push_back(r);
        for (;; ++g) { bool ok = true; for (uint32_t q : f) if (powm(g, (P - 1) / q) == 1) ok = false; if (ok) break; }
    }
    const uint32_t w32 = powm(g, (P - 1) / 32);
    // B operand: row 4k + c, K byte 32 b + j = byte c of (2^(8b) w^(jk) mod p)
    std::vector<uint8_t> bm(MMA_N * KB);
    for (int k = 0; k < NK; ++k)
        for (int c = 0; c < 4; ++c)
            for (int b = 0; b < 4; ++b)
                for (int j = 0; j < NK; ++j) {
                    const uint32_t f = mulm(powm(2, 8 * b), powm(w32, (uint64_t)j * k));
                    bm[kmaj_off(4 * k + c, 32 * b + j)] = (uint8_t)(f >> (8 * c));
                }
    // radix-2 table: entry h + j = w_(2h)^j for h = 1, 2, 4, 8, 16
    std::vector<uint32_t> wt(NK, 1), wtq(NK);
    for (int h = 1; h < NK; h <<= 1)
        for (int j = 0; j < h; ++j) wt[h + j] = powm(powm(w32, 16 / h), j);
    for (int i = 0; i < NK; ++i) wtq[i] = shq(wt[i]);
    const int ctas = nsm;
    const size_t cnt = (size_t)ctas * NG * NK;
    std::vector<uint32_t> x(cnt), tw(cnt), twq(cnt);
    uint64_t s = 0x9E3779B97F4A7C15ull;
    auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (uint32_t)(s % P); };
    for (size_t i = 0; i < cnt; ++i) { x[i] = rnd(); tw[i] = rnd(); twq[i] = shq(tw[i]); }
    uint32_t *dx, *dy, *dtw, *dtwq, *dwt, *dwtq;
    uint8_t *db;
    CK(cudaMalloc(&dx, cnt * 4)); CK(cudaMalloc(&dy, cnt * 4)); CK(cudaMalloc(&dtw, cnt * 4));
    CK(cudaMalloc(&dtwq, cnt * 4)); CK(cudaMalloc(&db, bm.size())); CK(cudaMalloc(&dwt, NK * 4));
    CK(cudaMalloc(&dwtq, NK * 4));
    CK(cudaMemcpy(dx, x.data(), cnt * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dtw, tw.data(), cnt * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dtwq, twq.data(), cnt * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, bm.data(), bm.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dwt, wt.data(), NK * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dwtq, wtq.data(), NK * 4, cudaMemcpyHostToDevice));
    const uint32_t r16 = powm(2, 16), r16q = shq(r16), onq = shq(1);
    const size_t tcs = sizeof(TcSmem) + 1024, als = sizeof(AluSmem);
    CK(cudaFuncSetAttribute(tc_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tcs));
    CK(cudaFuncSetAttribute(alu_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)als));
    // host reference of one repetition for the first 2 CTAs
    auto check = [&](const std::vector<uint32_t> &y, bool bitrev_out, const char *name) {
        int bad = 0;
        for (size_t grp = 0; grp < 2 * NG; ++grp)
            for (int k = 0; k < NK; ++k) {
                uint64_t acc = 0;
                for (int j = 0; j < NK; ++j) acc = (acc + (uint64_t)mulm(powm(w32, (uint64_t)j * k), x[grp * NK + j])) % P;
                const int pos = bitrev_out ? bitrev5(k) : k;
                const uint32_t want = mulm((uint32_t)acc, tw[grp * NK + pos]);
                if (y[grp * NK + pos] != want) ++bad;
            }
        printf("%s: first repetition vs host reference: %s (%d of %d outputs differ)\n", name, bad ? "MISMATCH" : "ok",
               bad, 2 * NG * NK);
        return bad == 0;
    };
    std::vector<uint32_t> y(cnt);
    tc_stage<<<ctas, THREADS, tcs>>>(dx, dy, db, dtw, dtwq, 1, r16, r16q, onq);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(y.data(), dy, cnt * 4, cudaMemcpyDeviceToHost));
    const bool ok_tc = check(y, false, "tcgen05 kind::i8 stage");
    alu_stage<<<ctas, THREADS, als>>>(dx, dy, dwt, dwtq, dtw, dtwq, 1);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(y.data(), dy, cnt * 4, cudaMemcpyDeviceToHost));
    const bool ok_alu = check(y, true, "radix-2 ALU stage");
    // timing: REPS repetitions per CTA, one CTA (128 threads) per SM and, for the ALU kernel, also
    // with 4 CTAs per SM
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    auto timeit = [&](auto launch, const char *name, int per_sm) {
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double points = (double)nsm * per_sm * NG * NK * reps;
        const double clk_s = (double)clk * 1e3 * ms * 1e-3;  // SM clocks in the interval (nominal)
        printf("%-34s %8.3f ms  %.3e points/s  %.2f points/clk/SM (at the %d MHz attribute clock)\n", name, ms,
               points / (ms * 1e-3), points / clk_s / nsm, clk / 1000);
    };
    for (int per_sm : {1, 2}) {
        const int cs = nsm * per_sm;
        uint32_t *bx, *by, *btw, *btwq;  // per_sm x the inputs (CTA i reads tile i)
        const size_t c2 = (size_t)cs * NG * NK;
        CK(cudaMalloc(&bx, c2 * 4)); CK(cudaMalloc(&by, c2 * 4)); CK(cudaMalloc(&btw, c2 * 4)); CK(cudaMalloc(&btwq, c2 * 4));
        for (int r = 0; r < per_sm; ++r) {
            CK(cudaMemcpy(bx + r * cnt, dx, cnt * 4, cudaMemcpyDeviceToDevice));
            CK(cudaMemcpy(btw + r * cnt, dtw, cnt * 4, cudaMemcpyDeviceToDevice));
            CK(cudaMemcpy(btwq + r * cnt, dtwq, cnt * 4, cudaMemcpyDeviceToDevice));
        }
        char n1[64], n2[64];
        snprintf(n1, sizeof n1, "tcgen05 stage (%d CTA/SM)", per_sm);
        snprintf(n2, sizeof n2, "radix-2 ALU stage (%d CTA/SM)", per_sm);
        timeit([&] { tc_stage<<<cs, THREADS, tcs>>>(bx, by, db, btw, btwq, reps, r16, r16q, onq); }, n1, per_sm);
        timeit([&] { alu_stage<<<cs, THREADS, als>>>(bx, by, dwt, dwtq, btw, btwq, reps); }, n2, per_sm);
        CK(cudaFree(bx)); CK(cudaFree(by)); CK(cudaFree(btw)); CK(cudaFree(btwq));
    }
    {  // ALU stage at 4 CTAs / SM (16 warps): the integer pipes' ceiling for this stage
        const int cs = nsm * 4;
        const size_t c2 = (size_t)cs * NG * NK;
        uint32_t *bx, *by, *btw, *btwq;
        CK(cudaMalloc(&bx, c2 * 4)); CK(cudaMalloc(&by, c2 * 4)); CK(cudaMalloc(&btw, c2 * 4)); CK(cudaMalloc(&btwq, c2 * 4));
        for (int r = 0; r < 4; ++r) {
            CK(cudaMemcpy(bx + r * cnt, dx, cnt * 4, cudaMemcpyDeviceToDevice));
            CK(cudaMemcpy(btw + r * cnt, dtw, cnt * 4, cudaMemcpyDeviceToDevice));
            CK(cudaMemcpy(btwq + r * cnt, dtwq, cnt * 4, cudaMemcpyDeviceToDevice));
        }
        timeit([&] { alu_stage<<<cs, THREADS, als>>>(bx, by, dwt, dwtq, btw, btwq, reps); }, "radix-2 ALU stage (4 CTA/SM)", 4);
    }
    return ok_tc && ok_alu ? 0 : 2;
}
