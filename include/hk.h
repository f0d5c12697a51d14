/*
 * hk.h -- exact multiprecision Hankel / Toeplitz / circulant matrix-vector product on B200.
 *
 * The operation (PAPER.md = G. Beliakov, arXiv:1402.5287; "P:NN" = PAPER.md line NN):
 *   Hankel    y = A_H x,  A_H[i][j] = a_{i+j-1}            (schoolbook P:87-90, read
 *                                                           as y_i = sum_j a_{i+j-1} x_j)
 *   Toeplitz  y = A_T x,  A_T[i][j] = a_{n-i+j}
 *   Circulant y = A_C x,  A_C[i][j] = c_{((i-j) mod n)+1}  (n x n, first column c)
 * Every entry is a multiprecision fixed-point number a = B0 * sum_k B^k a_k with B = 2^64
 * and B0 = 2^-P.  The result is exact (no rounding): y_i = Y_i * 2^-2P.
 *
 * LAYOUT (all arrays row-major, C-contiguous; DEVICE magnitude arrays 16-byte aligned -- they are
 *   staged by 16-byte / TMA bulk copies -- which every cudaMalloc / torch allocation satisfies):
 *   * a vector of `count` numbers is  mag: uint64_t[count][L]  (limb 0 least significant,
 *     L = hk_limbs(P) = ceil(P/64))  plus  sign: int8_t[count]  in {-1, 0, +1};
 *     value = sign * mag * 2^-P.  Inputs must satisfy sign == 0 <=> mag == 0, and every bit >= P
 *     must be zero (violations are DATA errors, see below).
 *   * outputs use Ly = hk_out_limbs(P) = 2L + 1 limbs: value = sign * mag * 2^-2P, canonical
 *     (sign 0 iff the value is 0; |Y| < n (2^P-1)^2 always fits).
 *
 * OWNERSHIP: the caller owns every buffer.  Unless a function says HOST, all array pointers are
 *   DEVICE pointers (e.g. torch CUDA tensors) on the current device.  The library allocates no
 *   device memory and keeps no global mutable state; all per-problem state (plan header,
 *   twiddle tables, transform-domain intermediates, status word) lives in the caller's
 *   workspace `ws`.  y must not overlap a, c or x.  A workspace may be used by one stream at a
 *   time; distinct workspaces may run concurrently.
 *
 * STREAMS: `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All
 *   matvec calls are asynchronous and stream-ordered; they never synchronise the host except
 *   hk_workspace_status and hk_matvec_host (documented there).
 *
 * ERRORS: every function returns an hk_status (int32_t).  ARGUMENT errors are returned
 *   synchronously before anything is enqueued: n < 1, P < 1, null pointers, overlapping y,
 *   undersized workspace (HK_EINVAL / HK_ENOMEM).  Capacity failures (no exact plan, see
 *   hk_plan) return HK_EUNSUPPORTED.  Launch failures return HK_ECUDA.  DATA errors
 *   (non-canonical inputs: bits >= P set, sign outside {-1,0,1}, sign/magnitude mismatch) and a
 *   workspace initialised for a different problem are detected on the device during the call
 *   and recorded in the workspace status word, read by hk_workspace_status; y is unspecified
 *   when that status is not HK_OK.  No C++ exception crosses this ABI.
 *
 * METHOD: each mantissa is cut into w-bit slices (w <= 65);
 *   the product becomes an exact 2-D convolution over (matrix index x slice) computed as a
 *   5-prime 31-bit number-theoretic transform (slice NTT of length N2 per entry, matrix-index
 *   NTT of length N1 per transformed column, pointwise Montgomery product, inverse NTTs),
 *   recombined by Garner CRT into signed coefficients and carried into exact limbs.  The planner
 *   proves 2 n Ls (2^w - 1)^2 < p1 p2 p3 p4 p5 for every call.
 */
#ifndef HK_H
#define HK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HK_OK = 0,
    HK_EINVAL = -1,        /* bad argument / workspace not initialised for this problem     */
    HK_ERANGE = -2,        /* data error: non-canonical input mantissa or sign                */
    HK_ENOMEM = -3,        /* workspace too small                                             */
    HK_EUNSUPPORTED = -4,  /* no exact plan for (kind, m, n, P) within the supported limits   */
    HK_ECUDA = -5          /* a CUDA call or kernel launch failed                             */
} hk_status;

typedef enum { HK_HANKEL = 0, HK_TOEPLITZ = 1, HK_CIRCULANT = 2 } hk_kind;

/* hk_workspace_size / hk_workspace_init flags (mutually exclusive) */
#define HK_WS_STAGING 1u   /* also reserve device staging buffers for hk_matvec_host */
#define HK_WS_PREPARED 2u  /* also reserve room for a prepared 2-D transform of a (hk_prepare_a) */

/* The plan the library chose for a problem (filled by hk_plan; all sizes in elements). */
typedef struct {
    int32_t kind;          /* hk_kind                                                          */
    int32_t P;             /* mantissa bits                                                    */
    int64_t m;             /* output rows (n for square kinds; window rows for rect Hankel)    */
    int64_t n;             /* columns = length of x                                            */
    int64_t a_count;       /* entries of the defining vector: m+n-1 (Hankel/Toeplitz), n (circ)*/
    int32_t L;             /* input limbs  = ceil(P/64)                                        */
    int32_t Ly;            /* output limbs = 2L+1                                              */
    int32_t k_primes;      /* NTT primes (5)                                                   */
    int32_t w;             /* slice width in bits (<= 65)                                      */
    int32_t Ls;            /* slices per mantissa = ceil(P/w)                                  */
    int32_t log_n2;        /* slice-dimension transform length N2 = 2^log_n2 >= 2Ls-1          */
    int32_t log_n1;        /* matrix-index transform length N1 = 2^log_n1                      */
    int32_t cyclic;        /* 1: circulant computed as a length-n cyclic convolution (n = N1)  */
    int32_t fold;          /* 1: circulant via linear convolution folded at n                  */
    double margin_bits;    /* log2(p1..p5) - log2(2 n Ls (2^w-1)^2) > 0                         */
    uint64_t ws_bytes;     /* workspace bytes without staging                                  */
    uint64_t ws_bytes_staging; /* workspace bytes with HK_WS_STAGING                           */
    uint64_t ws_bytes_prepared; /* workspace bytes with HK_WS_PREPARED                         */
} hk_plan_info;

/* L = ceil(P/64) (l = ceil(b / log2 B)); returns -1 if P < 1. */
int32_t hk_limbs(int32_t P);
/* Ly = 2L + 1; returns -1 if P < 1. */
int32_t hk_out_limbs(int32_t P);
/* Static string for a status code. */
const char *hk_status_string(int32_t status);

/* Chooses (w, Ls, N2, N1) for kind / m x n / P and proves the exact-CRT capacity bound.
 * m is the number of output rows: m == n for HK_TOEPLITZ / HK_CIRCULANT; for HK_HANKEL, m <= n is
 * the row window of a rectangular m x n Hankel (a has m+n-1 entries; m == n is the square case).
 * Pure host function.  HK_EUNSUPPORTED if no exact plan exists within the limits
 * (N1 <= 32768, i.e. m+n-1 <= 32768 for Hankel/Toeplitz; P <= 66560). */
int32_t hk_plan(int32_t kind, int64_t m, int64_t n, int32_t P, hk_plan_info *out);

/* Bytes of device workspace for the problem (flags: HK_WS_STAGING). Pure host function. */
int32_t hk_workspace_size(int32_t kind, int64_t m, int64_t n, int32_t P, uint32_t flags,
                          size_t *bytes);

/* Writes the plan header, the per-prime twiddle tables and a zero status word into ws
 * (stream-ordered, asynchronous).  Must run once per (kind, m, n, P, flags) before the matvec
 * calls that use ws.  ws: DEVICE pointer, 256-byte aligned, ws_bytes >= hk_workspace_size. */
int32_t hk_workspace_init(int32_t kind, int64_t m, int64_t n, int32_t P, uint32_t flags,
                          void *ws, size_t ws_bytes, void *stream);

/* Synchronises `stream`, then reads the workspace's data-status word of the last call into
 * *data_status (HK_OK, HK_ERANGE for bad input data, HK_EINVAL for a workspace initialised for a
 * different problem).  Returns HK_ECUDA if the copy fails. */
int32_t hk_workspace_status(void *ws, void *stream, int32_t *data_status);

/* Square Hankel: a_mag[2n-1][L], a_sign[2n-1]; x_mag[n][L], x_sign[n]; y_mag[n][Ly], y_sign[n].
 * y_i = sum_{j=1..n} a_{i+j-1} x_j.  DEVICE pointers. */
int32_t hk_hankel_matvec(int64_t n, int32_t P,
                         const uint64_t *a_mag, const int8_t *a_sign,
                         const uint64_t *x_mag, const int8_t *x_sign,
                         uint64_t *y_mag, int8_t *y_sign,
                         void *ws, size_t ws_bytes, void *stream);

/* Toeplitz: same shapes; y_i = sum_j a_{n-i+j} x_j.  Equals the Hankel product on the
 * same vector with rows reversed.  DEVICE pointers. */
int32_t hk_toeplitz_matvec(int64_t n, int32_t P,
                           const uint64_t *a_mag, const int8_t *a_sign,
                           const uint64_t *x_mag, const int8_t *x_sign,
                           uint64_t *y_mag, int8_t *y_sign,
                           void *ws, size_t ws_bytes, void *stream);

/* Circulant: c_mag[n][L], c_sign[n] (first column); y_i = sum_j c_{((i-j) mod n)+1} x_j.
 * DEVICE pointers. */
int32_t hk_circulant_matvec(int64_t n, int32_t P,
                            const uint64_t *c_mag, const int8_t *c_sign,
                            const uint64_t *x_mag, const int8_t *x_sign,
                            uint64_t *y_mag, int8_t *y_sign,
                            void *ws, size_t ws_bytes, void *stream);

/* Rectangular m x n Hankel window (the row-block shard of SURVEY.md 8(e)):
 * a_mag[m+n-1][L]; y_i = sum_{j=1..n} a_{i+j-1} x_j for i = 1..m.  DEVICE pointers. */
int32_t hk_hankel_rect_matvec(int64_t m, int64_t n, int32_t P,
                              const uint64_t *a_mag, const int8_t *a_sign,
                              const uint64_t *x_mag, const int8_t *x_sign,
                              uint64_t *y_mag, int8_t *y_sign,
                              void *ws, size_t ws_bytes, void *stream);

/* F4: the same product (any kind; m < n allowed for HK_HANKEL as in
 * hk_hankel_rect_matvec) with y rounded back to the input format: y_i = m_i 2^-P with
 * m_i = round_half_even(Y_i / 2^P) (Y_i the exact integer of hk_hankel_matvec, so y_i is the exact
 * product rounded to P fractional bits, ties to even), |m_i| < n 2^P.  y_mag[m][L+1], y_sign[m]
 * (canonical: sign 0 iff m_i = 0).  Workspace and errors as for the exact calls.  DEVICE pointers. */
int32_t hk_matvec_rounded(int32_t kind, int64_t m, int64_t n, int32_t P,
                          const uint64_t *a_mag, const int8_t *a_sign,
                          const uint64_t *x_mag, const int8_t *x_sign,
                          uint64_t *y_mag, int8_t *y_sign,
                          void *ws, size_t ws_bytes, void *stream);

/* End-to-end call with HOST buffers (same shapes as the kind's device call; for HK_HANKEL, m may
 * be < n as in hk_hankel_rect_matvec).  Enqueues on `stream`: H2D copies of a and x into the
 * workspace's staging area, the matvec, and D2H copies of y; then synchronises `stream` and
 * returns the call's data status (so HK_ERANGE is returned directly).  Host buffers should be
 * pinned (cudaHostAlloc / torch pin_memory) for asynchronous copies.  ws must have been sized and
 * initialised with HK_WS_STAGING. */
int32_t hk_matvec_host(int32_t kind, int64_t m, int64_t n, int32_t P,
                       const uint64_t *a_mag_host, const int8_t *a_sign_host,
                       const uint64_t *x_mag_host, const int8_t *x_sign_host,
                       uint64_t *y_mag_host, int8_t *y_sign_host,
                       void *ws, size_t ws_bytes, void *stream);

/* Asynchronous end-to-end call with HOST buffers, for throughput over a stream of independent
 * problems: enqueues on `stream`, in stream order and without synchronising, the H2D copies of a
 * and x into ws's staging area, the matvec, the D2H copies of y and of the call's data status
 * (one int32 hk_status written to *status_host when the stream reaches it).  Returns after
 * enqueueing: argument errors synchronously, HK_OK otherwise; host buffers must stay valid (and
 * y / status unread) until the stream has passed the call.  Several calls may be in flight on
 * different streams with DIFFERENT workspaces; their copies then overlap each other's kernels
 * (PCIe is full duplex).  Host buffers must be pinned for the copies to be asynchronous; ws as
 * for hk_matvec_host (HK_WS_STAGING). */
int32_t hk_matvec_host_async(int32_t kind, int64_t m, int64_t n, int32_t P,
                             const uint64_t *a_mag_host, const int8_t *a_sign_host,
                             const uint64_t *x_mag_host, const int8_t *x_sign_host,
                             uint64_t *y_mag_host, int8_t *y_sign_host, int32_t *status_host,
                             void *ws, size_t ws_bytes, void *stream);

/* ---- Multi-GPU: sigma-coset sharding (SURVEY.md 8(e) plan P-2) ------------------------------
 * The 2-D convolution is split over G = 2, 4 or 8 ranks along the slice-transform dimension
 * (the only coupling between slice frequencies sigma is the slice transform at each end):
 *   rank g: hk_hankel_shard_forward -- slices every entry of a and x (replicated inputs) but
 *           produces only block g of the G blocks of N2/G consecutive (bit-reversed order)
 *           slice-transform outputs per entry, i.e. the frequencies = bitrev(g) mod G (the
 *           coset fold: the first log2 G DIF stages keep one half each), runs the matrix-index
 *           transforms, pointwise product and inverse on its 5 N2/G columns, and writes them into
 *           `send` as G chunks [dest rank r][prime][column][rows_per_rank], chunk r holding the
 *           output rows [r rpr, (r+1) rpr);
 *   all ranks: an all-to-all of the chunks (chunk_words each; torch.distributed over NCCL);
 *   rank g: hk_hankel_shard_finish -- with `recv` = [source rank][prime][column][rpr], the
 *           inverse slice transforms of its rows, Garner CRT, carries, sign-magnitude, written into
 *           rows [g rpr, g rpr + rpr) of the padded y buffer (y_rows = G rpr rows);
 *   all ranks: an all-gather of those equal-size row blocks in rank order.  The final y is rows
 *           [0, n) of the padded buffer (Hankel, circulant) or rows [y_rows - n, y_rows)
 *           (Toeplitz, whose reversed rows are routed to ranks in reverse block order).
 * Bit-identical to the single-GPU call.  Workspaces: hk_shard_plan(...).ws_bytes, initialised by
 * hk_shard_workspace_init; one per rank.  All pointers are DEVICE pointers of the calling rank. */
typedef struct {
    int32_t G;              /* ranks (2, 4 or 8)                                                */
    int32_t gamma;          /* log2 G                                                           */
    int64_t block_cols;     /* slice-transform columns per prime per rank = N2 / G              */
    int64_t rows_per_rank;  /* rpr: output rows per rank block (multiple of 4)                  */
    int64_t y_rows;         /* rows of the padded y buffer = G rpr                              */
    int64_t chunk_words;    /* uint32 words per all-to-all chunk = 5 block_cols rpr             */
    int64_t buffer_words;   /* send / recv buffer words = G chunk_words                        */
    uint64_t ws_bytes;      /* per-rank workspace bytes                                         */
    /* sliced sharding (hk_hankel_shard_slice / _columns below); 0 when unsupported (N1 > 2^14 or
     * fewer than 8 matrix positions per rank)                                                     */
    int64_t slice_chunk_words;   /* words per (source, destination) slice chunk                  */
    int64_t slice_buffer_words;  /* slice send / receive buffer words = G slice_chunk_words      */
    int64_t slice_rows_a;        /* matrix positions of a (and of x) each rank slices: ldA / G   */
    int64_t slice_rows_x;        /*   and ldX / G                                                */
} hk_shard_info;

int32_t hk_shard_plan(int32_t kind, int64_t n, int32_t P, int32_t G, hk_shard_info *out);
int32_t hk_shard_workspace_init(int32_t kind, int64_t n, int32_t P, int32_t G, void *ws,
                                size_t ws_bytes, void *stream);
/* Phase 1 of rank g (see above).  a, x: DEVICE pointers (full, replicated); send: buffer_words. */
int32_t hk_hankel_shard_forward(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                const uint64_t *a_mag, const int8_t *a_sign,
                                const uint64_t *x_mag, const int8_t *x_sign, uint32_t *send,
                                void *ws, size_t ws_bytes, void *stream);
/* Phase 2 of rank g after the all-to-all: recv (buffer_words), y_mag[y_rows][Ly], y_sign[y_rows]. */
int32_t hk_hankel_shard_finish(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                               const uint32_t *recv, uint64_t *y_mag, int8_t *y_sign, void *ws,
                               size_t ws_bytes, void *stream);

/* SLICED sharding (round 2): hk_hankel_shard_forward slices EVERY entry on every rank (its slicing
 * and residues are replicated); this variant splits it too.  Phase 1a, rank g,
 * hk_hankel_shard_slice: slices only the entries at matrix positions [g Rs, (g+1) Rs) of a and of x
 * (Rs = slice_rows_a / slice_rows_x; x positions are reversed rows for Hankel / Toeplitz), runs the
 * full slice transform and scatters block d of its outputs into chunk d of `slice_send`:
 * [dest d][a part: prime][column of block d][Rs_a] then [x part: prime][column][Rs_x]; positions
 * past the entry counts are never written (keep the buffer zero-initialised).  An all-to-all of the
 * slice chunks follows.  Phase 1b, hk_hankel_shard_columns: with `slice_recv` = [source s][...]
 * (source s's positions), the matrix-index transforms of rank g's columns, exactly as
 * hk_hankel_shard_forward's second half, into `send`.  Phase 2 is hk_hankel_shard_finish.
 * The data-status word of a rank covers the entries it sliced: all-reduce the ranks' status. */
int32_t hk_hankel_shard_slice(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                              const uint64_t *a_mag, const int8_t *a_sign,
                              const uint64_t *x_mag, const int8_t *x_sign, uint32_t *slice_send,
                              void *ws, size_t ws_bytes, void *stream);
int32_t hk_hankel_shard_columns(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                const uint32_t *slice_recv, uint32_t *send, void *ws,
                                size_t ws_bytes, void *stream);
/* ... and with the slice exchange fused into K1's stores over peer memory: slice_recv_ptrs[d] = rank
 * d's slice receive buffer (this rank writes chunk g of it); a system-scope fence ends the kernel,
 * the caller barriers before phase 1b; hk_hankel_shard_columns_p2p then stores its row-block chunks
 * straight into the ranks' receive buffers as hk_hankel_shard_forward_p2p does. */
int32_t hk_hankel_shard_slice_p2p(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                  const uint64_t *a_mag, const int8_t *a_sign,
                                  const uint64_t *x_mag, const int8_t *x_sign,
                                  uint32_t *const *slice_recv_ptrs, void *ws, size_t ws_bytes,
                                  void *stream);
int32_t hk_hankel_shard_columns_p2p(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                    const uint32_t *slice_recv, uint32_t *const *recv_ptrs,
                                    void *ws, size_t ws_bytes, void *stream);

/* The same two phases with the collectives fused into the kernels' stores over peer memory
 * (NVLink / NVSwitch P2P; pointers mapped into this process, e.g. torch symmetric memory):
 *   forward_p2p: recv_ptrs[r] (host array of G device pointers) = rank r's receive buffer
 *     (buffer_words); K2 writes this rank's chunk for destination r directly at slot g of rank
 *     r's buffer, so no all-to-all is needed.  Every rank must have finished its forward_p2p before
 *     any rank's finish reads its receive buffer (a device or host barrier after the kernels).
 *   finish_p2p: recv = this rank's receive buffer; y_mag_ptrs[d] / y_sign_ptrs[d] = rank d's padded
 *     y buffers (y_rows rows); K3 writes this rank's rows into all G of them (the all-gather fused
 *     into its stores); a barrier after it completes the exchange.
 * Bit-identical to the NCCL-exchange path. */
int32_t hk_hankel_shard_forward_p2p(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                    const uint64_t *a_mag, const int8_t *a_sign,
                                    const uint64_t *x_mag, const int8_t *x_sign,
                                    uint32_t *const *recv_ptrs, void *ws, size_t ws_bytes,
                                    void *stream);
int32_t hk_hankel_shard_finish_p2p(int32_t kind, int64_t n, int32_t P, int32_t G, int32_t g,
                                   const uint32_t *recv, uint64_t *const *y_mag_ptrs,
                                   int8_t *const *y_sign_ptrs, void *ws, size_t ws_bytes,
                                   void *stream);

/* Pipeline stages of the NTT path, for per-kernel timing (bench.py) and phase-wise use:
 *   HK_STAGE_SLICE_ROWS  K1: validation, slicing, slice-dimension forward NTT of a and x
 *   HK_STAGE_COLUMNS     K2: matrix-index forward NTTs, pointwise product, inverse NTT
 *   HK_STAGE_FINISH      K3: inverse slice-dimension NTT, CRT, carry, sign-magnitude y
 * hk_matvec_stages runs the selected stages, in this order, with exactly the launches the
 * matvec entry points make; a stage reads what the previous stage left in ws, so running
 * HK_STAGE_COLUMNS or HK_STAGE_FINISH without the earlier stages of the same inputs gives an
 * unspecified y.  The data-status word is reset when HK_STAGE_SLICE_ROWS is selected.
 * Arguments as hk_matvec_host but DEVICE pointers. */
#define HK_STAGE_SLICE_ROWS 1u
#define HK_STAGE_COLUMNS 2u
#define HK_STAGE_FINISH 4u
#define HK_STAGE_ALL 7u
int32_t hk_matvec_stages(int32_t kind, int64_t m, int64_t n, int32_t P, uint32_t stages,
                         const uint64_t *a_mag, const int8_t *a_sign,
                         const uint64_t *x_mag, const int8_t *x_sign,
                         uint64_t *y_mag, int8_t *y_sign,
                         void *ws, size_t ws_bytes, void *stream);

/* Fixed-A repeated products (the Lanczos use of the paper): one
 * matrix, many vectors.  hk_prepare_a validates a, runs the slice-dimension and matrix-index
 * forward transforms of a once and keeps the full 2-D transform of a in the workspace (which must
 * have been sized and initialised with HK_WS_PREPARED for the same kind, m, n, P); the data
 * status of a is then readable with hk_workspace_status.  hk_matvec_prepared computes y for a new
 * x with only x's transforms, the pointwise product and the inverse (2 instead of 3 column
 * transforms, and no slicing of a).  If hk_prepare_a has not run on ws, the status of the call is
 * HK_EINVAL.  Shapes/kinds as hk_matvec_host; DEVICE pointers; asynchronous on `stream`. */
int32_t hk_prepare_a(int32_t kind, int64_t m, int64_t n, int32_t P,
                     const uint64_t *a_mag, const int8_t *a_sign,
                     void *ws, size_t ws_bytes, void *stream);
int32_t hk_matvec_prepared(int32_t kind, int64_t m, int64_t n, int32_t P,
                           const uint64_t *x_mag, const int8_t *x_sign,
                           uint64_t *y_mag, int8_t *y_sign,
                           void *ws, size_t ws_bytes, void *stream);

/* Companion A6: direct schoolbook limb-product matvec on the GPU, no
 * transform: y_i = sum_j A_{idx(i,j)} X_j with 32-bit limb products and wide column sums.
 * kind / m / n / shapes as above (HK_HANKEL with m < n = rectangular window).  Needs no
 * workspace; data errors are not checked (inputs must be canonical).  DEVICE pointers. */
int32_t hk_schoolbook_matvec(int32_t kind, int64_t m, int64_t n, int32_t P,
                             const uint64_t *a_mag, const int8_t *a_sign,
                             const uint64_t *x_mag, const int8_t *x_sign,
                             uint64_t *y_mag, int8_t *y_sign, void *stream);

/* Companion A5: the paper's Karatsuba-like Algorithm 1 run level
 * by level on the GPU -- split (steps 3-6), recursion as 3^d batched subproblems per level
 * (step 7; size-m children zero-padded to m1), direct products at subproblems of size
 * <= cutoff (step 1 is cutoff = 2), merge (step 8).  Square Hankel only, shapes as
 * hk_hankel_matvec; DEVICE pointers; inputs must be canonical (not validated).  cutoff >= 2.
 * The workspace (caller-owned, 256-byte aligned) holds every level's operands and results:
 * hk_karatsuba_workspace_size returns its size (pure host).  Asynchronous on `stream`. */
int32_t hk_karatsuba_workspace_size(int64_t n, int32_t P, int32_t cutoff, size_t *bytes);
int32_t hk_karatsuba_matvec(int64_t n, int32_t P, int32_t cutoff,
                            const uint64_t *a_mag, const int8_t *a_sign,
                            const uint64_t *x_mag, const int8_t *x_sign,
                            uint64_t *y_mag, int8_t *y_sign,
                            void *ws, size_t ws_bytes, void *stream);

/* ---- F1 kernel-level batch: nvec vectors against one prepared matrix, one launch per stage ----
 * The paper's Lanczos use multiplies one matrix by many vectors.  A batch workspace is a
 * HK_WS_PREPARED workspace followed by nvec per-vector transform regions (hk_batch_workspace_size,
 * pure host; hk_batch_workspace_init, stream-ordered; the same 256-byte alignment rules).  After
 * hk_prepare_a on it, hk_matvec_prepared_batch computes y_v = A x_v for v < nvec with ONE launch of
 * each of K1 (x slicing), K2 (every A^ column read from HBM once for all vectors) and K3:
 *   x_mag: uint64[nvec][n][L] (each vector 16-byte aligned: n L even or nvec = 1), x_sign: int8[nvec][n]
 *   y_mag: uint64[nvec][m][Ly],  y_sign: int8[nvec][m]    (DEVICE; layouts as hk_matvec_prepared)
 * ws_bytes must be the size the workspace was initialised with (its vector capacity is derived
 * from it; HK_ENOMEM when nvec exceeds it).  The data-status word covers the whole batch (any
 * rejected x -> HK_ERANGE for the call). */
int32_t hk_batch_workspace_size(int32_t kind, int64_t m, int64_t n, int32_t P, int32_t nvec,
                                size_t *bytes);
int32_t hk_batch_workspace_init(int32_t kind, int64_t m, int64_t n, int32_t P, int32_t nvec,
                                void *ws, size_t ws_bytes, void *stream);
int32_t hk_matvec_prepared_batch(int32_t kind, int64_t m, int64_t n, int32_t P, int32_t nvec,
                                 const uint64_t *x_mag, const int8_t *x_sign,
                                 uint64_t *y_mag, int8_t *y_sign,
                                 void *ws, size_t ws_bytes, void *stream);

/* ---- F3: the paper's decomposition approach with a double-precision FFT ----
 * PAPER.md P:119-170 decomposes every multiprecision number into standard-precision pieces and
 * computes the product with one standard FFT, leaving open "whether the loss of accuracy occurs in
 * practice".  This variant makes it exact with a PROOF: mantissas are cut into balanced
 * w-bit digits (|d| <= 2^(w-1)), the 2-D convolution (matrix index x digit) is a complex FP64 FFT
 * of N1 x N2 points with round-to-nearest butterflies, and the planner picks the widest w for which
 * Percival's bound (Math. Comp. 72 (2003), Thm 5.1, with k = log2(N1 N2) radix-2 stages, unit
 * roundoff eps = 2^-53 and twiddle error beta = 2^-52) on |computed - exact| of every output
 * coefficient, evaluated with |a|_2 |x|_2 <= sqrt(a_count n) Ls 2^(2w-2), is <= 0.49; each
 * coefficient is then rounded to its exact integer and carried into y (same layout, canonical
 * form and exactness as hk_hankel_matvec).  Slower than the NTT path; supported for N1 <= 32768 and
 * N2 <= 8192 (else HK_EUNSUPPORTED).  Square problems only (m = n), all three kinds. */
typedef struct {
    int32_t kind;
    int32_t P;
    int64_t m, n, a_count;
    int32_t L, Ly;
    int32_t w;             /* balanced digit width                                             */
    int32_t Ls;            /* digits per mantissa = ceil(P / w) + 1                            */
    int32_t log_n1;        /* matrix-index FFT length 2^log_n1                                 */
    int32_t log_n2;        /* digit FFT length 2^log_n2 >= 2 Ls - 1                            */
    int32_t cyclic, fold;  /* as hk_plan_info                                                  */
    double bound;          /* Percival bound on the coefficient error (<= 0.49 < 1/2)          */
    double eps, beta;      /* unit roundoff and twiddle error the bound assumes                */
    uint64_t ws_bytes;     /* workspace bytes for hk_fft_workspace_init / hk_fft_matvec        */
} hk_fft_plan_info;

/* The plan (pure host; HK_EUNSUPPORTED when no digit width meets the bound within the limits). */
int32_t hk_fft_plan(int32_t kind, int64_t n, int32_t P, hk_fft_plan_info *out);
/* Twiddle tables (host-computed in long double, uploaded), carry table, header; stream-ordered.
 * ws: >= info.ws_bytes DEVICE bytes, 256-byte aligned; HK_ENOMEM when smaller. */
int32_t hk_fft_workspace_init(int32_t kind, int64_t n, int32_t P, void *ws, size_t ws_bytes,
                              void *stream);
/* y = A x through the FP64 FFT path; arguments, layouts, validation and the data-status word
 * (hk_workspace_status) as hk_hankel_matvec / hk_toeplitz_matvec / hk_circulant_matvec (kind). */
int32_t hk_fft_matvec(int32_t kind, int64_t n, int32_t P,
                      const uint64_t *a_mag, const int8_t *a_sign,
                      const uint64_t *x_mag, const int8_t *x_sign,
                      uint64_t *y_mag, int8_t *y_sign,
                      void *ws, size_t ws_bytes, void *stream);

/* F3 accuracy study (second half; "whether the loss of accuracy occurs in
 * practice"): the same plan, workspace and matvec with the digit width FORCED to w (w = 0: the
 * proven planner above, identical to hk_fft_plan / _workspace_init / _matvec).  For w wider than
 * the proven one the Percival bound in info.bound exceeds 1/2 and the result is NOT guaranteed
 * exact -- these entry points exist to measure where exactness is actually lost.  HK_EINVAL for
 * w outside [0, 30]; HK_EUNSUPPORTED when the digit FFT would exceed N2 = 8192 or a coefficient
 * could reach 2^62.  A workspace initialised for one w is rejected (data status HK_EINVAL) by a
 * call with another.  max_residual: optional DEVICE pointer to one 8-byte-aligned double holding
 * a non-negative value (the caller zeroes it); the call raises it to the largest |v - rint(v)|
 * over every scaled output coefficient v it rounds (the distance the bound is about). */
int32_t hk_fft_plan_w(int32_t kind, int64_t n, int32_t P, int32_t w, hk_fft_plan_info *out);
int32_t hk_fft_workspace_init_w(int32_t kind, int64_t n, int32_t P, int32_t w, void *ws,
                                size_t ws_bytes, void *stream);
int32_t hk_fft_matvec_w(int32_t kind, int64_t n, int32_t P, int32_t w,
                        const uint64_t *a_mag, const int8_t *a_sign,
                        const uint64_t *x_mag, const int8_t *x_sign,
                        uint64_t *y_mag, int8_t *y_sign,
                        void *ws, size_t ws_bytes, void *stream, double *max_residual);

#ifdef __cplusplus
}
#endif
#endif /* HK_H */
