// hk_internal.h -- plan / parameter structures shared by the host API (hk_api.cu) and the
// kernels (hk_ntt.cu, hk_schoolbook.cu).  Not part of the public ABI (include/hk.h).
#pragma once
#include <cstddef>
#include <cstdint>

#include "../../include/hk.h"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing unless a tool is attached

namespace hk {

// NVTX range over one C-ABI call (nsys / ncu --nvtx show the library's phases by entry point)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define HK_NVTX(name) ::hk::NvtxRange hk_nvtx_range_(name)


constexpr int kNumPrimes = 5;
constexpr uint64_t kWsMagic = 0x484b5753504c414eull;  // "HKWSPLAN"
constexpr int kMaxLogN1 = 15;                           // N1 <= 32768 (K2 register budget)
constexpr int kMinLogN1 = 6;
#ifndef HK_SPLIT_LOGN1
#define HK_SPLIT_LOGN1 15
#endif
constexpr int kSplitLogN1 = HK_SPLIT_LOGN1;             // K2 as prepare + prepared launches from here
constexpr int kMaxShards = 8;                           // sigma-coset shards G <= 8
constexpr int kMaxLogN2 = 11;                           // N2 <= 2048 -> Ls <= 1024
constexpr int kMinLogN2 = 5;
constexpr int kMaxW = 65;                               // a slice spans at most two limbs
constexpr int kK3TablePad = 176;  // K3 v2 tables: entries past Ly (> threads per row, 160, + max CH)
constexpr int kK3MaxLy = 2240;                          // K3 carry: 320 threads, <= 14 limbs per
                                                        // thread over 4 rows / 2 rows (N2 = 2048)

struct PrimeConsts {
    uint32_t p, pneg;          // modulus, -p^-1 mod 2^32 (Montgomery)
    uint32_t fa[3], fa_q[3];   // a digit weights 1, 2^32, 2^64 mod p (+ Shoup quotients)
    uint32_t fx[3], fx_q[3];   // x digit weights times 2^32 (N1 N2)^-1 mod p (+ quotients)
};

struct GarnerConsts {
    uint32_t inv[kNumPrimes][kNumPrimes];    // p_j^-1 mod p_k, j < k
    uint32_t inv_q[kNumPrimes][kNumPrimes];  // Shoup quotients
    uint32_t half[kNumPrimes];               // (p_k - 1) / 2: mixed-radix digits of (M-1)/2
    uint32_t M[kNumPrimes];                  // M = p0 p1 p2 p3 p4 as 32-bit words
};

// K3 v2 CRT: Garner over the primes in ascending order, applied to the
// residues of C + H (H = (M-1)/2), so the mixed-radix value C'' = C + H in [0, M) is the unsigned
// coefficient; the carry phase adds -K, K = H sum_{s < S2} 2^(w s) (mod 2^(64 Ly)), once per limb.
struct Garner2Consts {
    uint32_t p[kNumPrimes];                  // primes in ascending order (digit order)
    uint32_t kp[kNumPrimes];                 // index of digit g's prime in PrimeConsts pc[]
    uint32_t c[kNumPrimes][kNumPrimes];      // p_j^-1 mod p_g (j < g, ascending order)
    uint32_t cq[kNumPrimes][kNumPrimes];     // Shoup quotients
    uint32_t h[kNumPrimes];                  // H mod p_g
};

struct WsHeader {  // first 256 bytes of a workspace
    uint64_t magic;
    uint64_t hash;
    int32_t status;
    int32_t a_ready;   // 1 after hk_prepare_a wrote the 2-D transform of a into AT
    int32_t pad_[58];
};

// Everything a launch needs, passed by value.
struct Params {
    // problem
    int32_t kind, P, L, Ly;
    int64_t m, n, a_count;
    // plan
    int32_t w, Ls, S2;           // S2 = 2Ls-1 output slices
    int32_t log_n1, log_n2, N1, N2;
    int32_t cyclic, fold, reverse_out, x_reversed;
    int64_t out_off;             // first needed index of the matrix-index convolution
    int64_t ldA, ldX, ldY;       // leading dims (elements) of the transform-domain arrays
    uint64_t hash;
    int32_t tile0;               // K1: first tile of this launch (combined [a tiles | x tiles] index)
    int32_t tile_split, tile_skip;  // K1: CTAs >= tile_split skip tile_skip tiles (two ranges, one launch)
    int32_t k1_prime_split;      // K1: one prime per CTA (blockIdx.z) for launches under one wave
    int64_t row0;                // K3: first output row of this launch
    // sigma-coset sharding (SURVEY.md 8(e) plan P-2; 1 shard = the single-GPU path):
    int32_t n2loc, log_n2loc;    // transform-domain columns per prime held here (N2 / G)
    int32_t shard_gamma;         // log2 G (0: not sharded)
    int32_t k1_block;            // K1: slice-transform output block b = bitrev_gamma(g) kept
    int64_t shard_rpr;           // rows per rank block (multiple of 4); 0: not sharded
    int64_t shard_row0;          // K3: first internal row of this rank's block (g * rpr)
    int64_t y_rows;              // rows of the y buffer (m, or G * rpr when sharded)
    int32_t round_out;           // F4: y = round_half_even(Y / 2^P) in L + 1 limbs (2^-P scale)
    // peer-memory exchange (P2P shards): K2 stores row block r of its columns straight into rank
    // r's receive buffer, K3 stores its y rows into every rank's y buffer (pointers mapped into
    // this process, e.g. torch symmetric memory over NVLink); 0 = buffers of this rank only
    int32_t p2p;
    uint32_t *peer_recv[kMaxShards];
    uint64_t *peer_ymag[kMaxShards];
    int8_t *peer_ysign[kMaxShards];
    // inputs / outputs (device)
    const uint64_t *a_mag;
    const int8_t *a_sign;
    const uint64_t *x_mag;
    const int8_t *x_sign;
    uint64_t *y_mag;
    int8_t *y_sign;
    // workspace regions
    WsHeader *hdr;
    const uint2 *tw;             // per prime: [N2 forward table | N1 forward table]
    uint32_t *Ahat, *Xhat, *Yhat;  // K2 writes Yhat; K3 reads it (the all-to-all receive
                                   // buffer when sharded)
    uint32_t *AT;                // prepared 2-D transform of a (HK_WS_PREPARED), or null
    int32_t need_a_ready;        // K1 (x tiles): require hdr->a_ready
    int32_t split_k2;            // K2 as MODE 1 (A^ -> AT) + MODE 2 (X^ x AT, inverse) launches
    PrimeConsts pc[kNumPrimes];
    GarnerConsts gc;
    Garner2Consts g2;
    const uint64_t *negK;        // Ly limbs of -K mod 2^(64 Ly) (K3 v2), in the workspace
    // sliced sharding: K1 slices only this rank's matrix positions [k1_block Rs, (k1_block+1) Rs)
    // and scatters every sigma-block to its destination chunk; K2 gathers its columns from the
    // slice receive buffer [source][a part | x part]
    int32_t slice_mode;
    int32_t lg_rs_a, lg_rs_x;    // log2 Rs of a and x
    int64_t slice_chunk, slice_xoff;  // words per chunk, words of a chunk's a part
    uint32_t *slice_out;         // K1: send buffer [dest][chunk] (NCCL layout)
    uint32_t *peer_slice[kMaxShards];  // K1 p2p: rank d's slice receive buffer
    const uint32_t *slice_in;    // K2: this rank's slice receive buffer [source][chunk]
    // F1 kernel-level batch (hk_matvec_prepared_batch): nvec vectors per launch; vector v's x / y
    // are x_vstride / y_vstride entries after vector v - 1's, its X^ / Y^ columns continue the
    // column index (X^ column c of vector v = column v * ncols + c, likewise Y^); 1 otherwise
    int32_t nvec;
    int64_t x_vstride, y_vstride;
    const uint32_t *qmap;        // K3 v2: entry qq + 3 (qq = -3 .. Ly - 1) = (smem word offset of
                                 // the coefficient at limb qq, or of the zero slot) << 6 | shift
};

struct Plan {
    hk_plan_info info;
    int32_t G, gamma;            // sigma-coset shards (1, 0 unless a shard plan)
    int64_t rpr;                 // rows per rank block (shard plans)
    int64_t out_off;
    int32_t reverse_out, x_reversed;
    int64_t ldA, ldX, ldY;
    size_t off_tw, off_negK, off_qmap, off_A, off_X, off_Y, off_stage, off_end, off_end_staging;
    size_t st_amag, st_asign, st_xmag, st_xsign, st_ymag, st_ysign;
    size_t off_AT, off_end_prepared;
    size_t xhat_bytes, yhat_bytes;   // one vector's X^ / Y^ region (batch workspaces append nvec of each)
    int32_t split_k2;            // N1 >= 2^kSplitLogN1: AT inside the base layout, K2 in two launches
    int32_t slice_ok;            // sliced sharding supported (G > 1, log_n1 <= 14, Rs >= 8)
    int64_t rs_a, rs_x, slice_chunk;
};

// kernels (hk_ntt.cu)
int launch_init(const Params &prm, const uint32_t *gens, void *stream);
int launch_ntt_path(const Params &prm, void *stream, uint32_t stages);
// partial launches for the pipelined host path: K1 over tiles [tile0, tile0 + ntiles) of the
// combined [a | x] tile index (8 rows per tile), K3 over output rows [row0, row0 + nrows)
int k1_tile_rows();  // entries per K1 tile
int k1_tiles_a(const Params &prm);
int k1_tiles_x(const Params &prm);
int launch_k1_range(const Params &prm, void *stream, int tile0, int ntiles);
int launch_k3_range(const Params &prm, void *stream, int64_t row0, int64_t nrows);
// K2 of the sliced shards (columns gathered from the slice receive buffer)
int launch_k2_sliced(const Params &prm, void *stream);
// K2 variants: 0 = full (X^ and A^ transforms), 1 = prepare (A^ transform -> AT),
// 2 = prepared (X^ transform x AT, inverse)
int launch_k2_mode(const Params &prm, void *stream, int mode);
// hdr->a_ready = 1 iff hdr->status == HK_OK (end of hk_prepare_a)
int launch_set_a_ready(const Params &prm, void *stream);
// rows per K3 tile for a slice-transform length 2^log_n2 (the qmap offsets depend on it)
int k3_tile_rows(int log_n2);
// companion (hk_schoolbook.cu)
int launch_schoolbook(int kind, int64_t m, int64_t n, int32_t P, const uint64_t *a_mag,
                      const int8_t *a_sign, const uint64_t *x_mag, const int8_t *x_sign,
                      uint64_t *y_mag, int8_t *y_sign, void *stream);

// companion A5 (hk_karatsuba.cu)
int karatsuba_workspace_size(int64_t n, int32_t P, int32_t cutoff, size_t *bytes);
int launch_karatsuba(int64_t n, int32_t P, int32_t cutoff, const uint64_t *a_mag,
                     const int8_t *a_sign, const uint64_t *x_mag, const int8_t *x_sign,
                     uint64_t *y_mag, int8_t *y_sign, void *ws, size_t ws_bytes, void *stream);

}  // namespace hk
