/*
 * sffn.h — C ABI of the B200-native (sm_100a) sparse gated-FFN forward (TwELL).
 *
 * Method: arxiv 2603.23198, /root/reference/PAPER.md (cited P:<line>).
 *   Eq.1      h_u = x W_u, h_g = relu(x W_g), h = h_u * h_g, y = h W_d
 *   Alg.1    gate GEMM whose epilogue stores relu(x W_g) in TwELL
 *   Alg.2 / Eq.3  fused up+down projection over the TwELL non-zeros
 *   TwELL, packed 32-bit layout (Listing 1)
 *
 * Conventions (every call):
 *   - All tensor pointers are DEVICE pointers to caller-owned memory.  The library never allocates
 *     device memory, never frees caller memory and never synchronizes the device (except
 *     sffn_overflow_check, which synchronizes the given stream by design).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Every call is
 *     stream-ordered and asynchronous; calls on distinct streams are thread-safe.
 *   - Notation M (tokens), K (model dim), N (hidden dim) as in P:55.
 *   - Weights are hidden-major, [N, K] row-major, for W_g, W_u and W_d alike (DESIGN.md reading
 *     R11: "up projection weight matrix is stored in transposed format" P:1078, Listing 1 NT
 *     GEMM P:464).  W_g and W_u are therefore nn.Linear weights; W_d is [N, K] = the paper's W_d.
 *   - X, W_*, Y, H are bf16 (IEEE bfloat16 bit patterns), row-major, 16-byte aligned.
 *   - Return value: an sffn_status.  Argument/shape errors are detected on the host BEFORE any
 *     launch (nothing is enqueued).  SFFN_ERR_CUDA means a launch failed (cudaGetLastError).
 *   - Data-dependent results (TwELL tile overflow) are never returned synchronously: they are
 *     counted into a caller-owned device uint32 (`d_overflow`, may be NULL), which the caller zeroes
 *     and reads after its own synchronization — the paper's "flag that is reported to the CPU at the
 *     next GPU synchronization point".  sffn_overflow_check does that read for you.
 *
 * TwELL packed layout (bf16 mode): uint32 matrix [M, N/C], row-major.  Row m, tile t
 * (columns [tT, tT+T)) owns words [m*N/C + t*T/C, +T/C): word 0 = count of strictly positive
 * pre-activations in the tile (the TRUE count, may exceed the capacity; reading R5); words 1..
 * = (column & 0xFFFF) | (bf16_rne(value) << 16) in ascending column order (reading R3); capacity
 * T/C - 1 ("the first 31 TwELL indices" at T=256, C=8).  Column indices are local to the
 * weight rows passed in (a shard's row 0 is index 0).  Words past the count are unspecified.
 */
#ifndef SFFN_H_
#define SFFN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SFFN_OK = 0,
    SFFN_ERR_INVALID_ARG = 1,   /* NULL pointer, misaligned pointer (< 16 B), bad T/C combination      */
    SFFN_ERR_SHAPE = 2,         /* M < 0, K % 64 != 0, N % T != 0, N > 65536, workspace too small, ...  */
    SFFN_ERR_TILE_OVERFLOW = 3, /* (sffn_overflow_check only) some (row, tile) had > T/C-1 positives   */
    SFFN_ERR_CUDA = 4,          /* a CUDA runtime / driver call or kernel launch failed                 */
    SFFN_ERR_NCCL = 5,          /* an NCCL call failed                                                  */
    SFFN_ERR_UNSUPPORTED = 6    /* not a B200 (sm_100) device, or a feature not built                   */
} sffn_status;

/* Algorithm of the fused sparse up/down (Alg.2 / Eq.3).  Both compute the same Eq.3 sum:
 *   SFFN_ALGO_GATHER: one CTA per token row, fp32 FMA over coalesced 16-byte gathers of the active
 *                     W_u / W_d rows (the paper's Listing 2 design); needs no workspace.
 *   SFFN_ALGO_UNION : rows reordered by pi (Alg.2 iterates m in pi(0..M-1): descending stored
 *                     non-zeros within each 2048-row sequence window), then
 *                     per block of 128 rows, the union U_b of their active neurons; the up projection
 *                     X_b W_u[U_b]^T and the down projection H_b W_d[U_b] run on tcgen05 tensor cores
 *                     with the gate applied in the epilogue (zero off-pattern, so skipped terms are
 *                     exactly the h_g = 0 terms of Alg.2); W_u / W_d rows gathered with cp.async.
 *                     Needs workspace (sffn_up_down_workspace_bytes) and N % 64 == 0.
 *   SFFN_ALGO_AUTO  : UNION when N % 64 == 0, else GATHER. */
typedef enum { SFFN_ALGO_AUTO = 0, SFFN_ALGO_GATHER = 1, SFFN_ALGO_UNION = 2 } sffn_algo;

/* Human-readable name of a status code (static storage). */
const char* sffn_status_string(int status);
/* Library version / build string (static storage). */
/* Number of CUDA kernels the library has launched so far in this process (host-side counter; a launch
 * captured into a CUDA graph counts once, at capture).  Benchmarks read it around a step to report how
 * many of the library's own kernels a step runs.  Thread-safe, never fails. */
int64_t sffn_launch_count(void);
const char* sffn_version(void);

/* Number of uint32 words of a packed TwELL for [M, N] with tile T and compression C: M * N / C. */
int64_t sffn_twell_words(int64_t M, int64_t N, int T, int C);
/* Bytes of device workspace sffn_up_down needs for `algo` (0 for GATHER). */
size_t sffn_up_down_workspace_bytes(int64_t M, int64_t K, int64_t N, int T, int C, int algo);
/* Bytes of device workspace sffn_forward needs: the TwELL of the gate (4 * sffn_twell_words, rounded
 * to 1 KiB) followed by the up/down workspace of `algo`. */
size_t sffn_forward_workspace_bytes(int64_t M, int64_t K, int64_t N, int T, int C, int algo);

/*
 * sffn_pack — Alg.1: TwELL of relu(X W_g^T), computed by a tcgen05/TMEM tensor-core GEMM
 * (bf16 x bf16 -> fp32 accumulators in TMEM) whose epilogue thresholds the fp32 accumulator with a
 * strict > 0 (Alg.1 line 11; reading R1-R2) and compacts each row-tile in ascending column order.
 *   X      [M, K] bf16            Wg  [N, K] bf16 (hidden-major)
 *   twell  [M, N/C] uint32 (output, packed layout above)
 *   d_overflow  optional device uint32, += 1 per (row, tile) whose count exceeded T/C - 1
 * Constraints: M >= 0, K >= 64, K % 64 == 0, N % T == 0, N % 16 == 0, N <= 65536,
 *              T in {32, 64, 128, 256}, C in {1, 2, 4, 8, 16}, T / C >= 2.
 */
int sffn_pack(const void* X, const void* Wg, int64_t M, int64_t K, int64_t N, int T, int C, uint32_t* twell,
              uint32_t* d_overflow, void* stream);

/*
 * sffn_unpack — verification: TwELL -> dense bf16 (SPEC S:167-175 twell_to_dense).
 * dense[m, col_offset + n] = stored value for the valid prefix min(count, T/C-1) of each tile,
 * +0 for every other n in [0, N).  dense has row stride ld_dense elements (>= col_offset + N);
 * columns outside [col_offset, col_offset + N) are not touched.
 */
int sffn_unpack(const uint32_t* twell, int64_t M, int64_t N, int T, int C, int64_t col_offset, int64_t ld_dense,
                void* dense, void* stream);

/*
 * sffn_up_down — Alg.2 / Eq.3 from an existing TwELL:
 *   Y[m, :] = sum_t sum_{c < min(h_nz, T/C-1)} h_v * (X[m, :] . Wu[n, :]) * Wd[n, :]
 * h_v = the stored bf16 gate value; fp32 accumulation; Y rounded to bf16 (RN).  GATHER keeps h = h_v * u
 * in fp32; UNION rounds h to bf16 before the down GEMM (as the paper's kernel does, L2 P:994-1002).
 *   X [M, K] bf16, twell [M, N/C] uint32, Wu [N, K] bf16, Wd [N, K] bf16, Y [M, K] bf16 (output)
 *   workspace / ws_bytes: >= sffn_up_down_workspace_bytes(M, N, T, C, algo) (may be NULL for GATHER)
 * Constraints: those of sffn_pack, K <= 65536, and K <= 8192 for GATHER (x is held in registers).
 */
int sffn_up_down(const void* X, const uint32_t* twell, const void* Wu, const void* Wd, int64_t M, int64_t K,
                 int64_t N, int T, int C, void* Y, void* workspace, size_t ws_bytes, int algo, void* stream);

/*
 * sffn_forward — the whole sparse FFN forward: sffn_pack into `workspace` (>= sffn_forward_workspace_bytes)
 * then sffn_up_down with the rest of the workspace.  GATHER = the paper's two launches; UNION
 * launches 4 kernels (gate GEMM; one metadata kernel: row order pi, block unions, gate lists, X in pi order;
 * UP and DOWN GEMMs; sffn_launch_count reports them) plus one memset of the row counts / counters.
 * The TwELL left at the start of the workspace
 * is valid after the call (stream-ordered).
 */
int sffn_forward(const void* X, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N,
                 int T, int C, void* Y, void* workspace, size_t ws_bytes, uint32_t* d_overflow, int algo,
                 void* stream);

/* ---------------------------------------------------------------- overflow-exact (hybrid) forward
 * the paper's hybrid idea (rows routed to the compact sparse form or to a dense backup,
 * P:177-182; backup rows sized e.g. M/8) applied to inference.  After sffn_forward, every row
 * whose TwELL has an overflowed tile (count > T/C-1) is recomputed with the dense tcgen05 FFN (Eq.1 over all
 * hidden units: exact) and written over the sparse result, so Y is exact for any sparsity tail.  At most
 * `backup_rows` rows are recomputed; *d_backup_count (device int, optional) receives the number of rows that
 * needed it (if it exceeds backup_rows the remaining rows keep the stored-entries result, reading R5).
 * Requires N % 128 == 0.  Weights as sffn_forward (W_d [N, K] is read MN-major by TMA: no transpose).
 * workspace >= sffn_hybrid_workspace_bytes(...) (= forward workspace + backup buffers). */
size_t sffn_hybrid_workspace_bytes(int64_t M, int64_t K, int64_t N, int T, int C, int algo, int64_t backup_rows);
int sffn_forward_hybrid(const void* X, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K,
                        int64_t N, int T, int C, void* Y, void* workspace, size_t ws_bytes, int64_t backup_rows,
                        int* d_backup_count, uint32_t* d_overflow, int algo, void* stream);

/* ---------------------------------------------------------------- training entry: TwELL -> hybrid (NEXT-4)
 * Listing 4 on the packed TwELL, hybrid format P:177-182: per row, the stored entries in
 * ascending column order compacted into an ELL row of width ell_w (ell_val bf16 [M, ell_w], ell_col int16
 * [M, ell_w], slots past min(nnz, ell_w) untouched); row_nnz[m] = stored count (true occupancy, may exceed
 * ell_w).  Rows with row_nnz > ell_w go to the dense tail: slot s < dense_cap (atomic order), dense_rows[s, :]
 * = the densified row (bf16 [dense_cap, N]), dense_map[s] = m, row_loc[m] = s; row_loc[m] = -1 for ELL rows
 * and -2 when the tail is full (the paper's "discard the excess and set a flag").  *d_dense_count
 * (device int, zeroed by the caller) = rows that needed the tail.  d_l0l1 (device double[2], optional,
 * accumulated): += sum_m nnz_m / M and sum_m sum(values_m) / M (Listing 4's L0 / L1 statistics). */
int sffn_twell_to_hybrid(const uint32_t* twell, int64_t M, int64_t N, int T, int C, int ell_w, void* ell_val,
                         int16_t* ell_col, int32_t* row_nnz, int32_t* row_loc, int64_t dense_cap, void* dense_rows,
                         int32_t* dense_map, int* d_dense_count, double* d_l0l1, void* stream);

/* ---------------------------------------------------------------- non-gated variant (App.C, NEXT-2)
 * h = relu(x W_u), y = h W_d: the TwELL now comes from the UP projection (the same
 * tcgen05 pack kernel applied to W_u), and only the down projection remains (Listing 3,
 * P:1085-1215).
 * sffn_down: Y[m,:] = sum over the stored entries (n, h_v) of h_v * Wd[n,:]  (fp32 accumulate, bf16 Y).
 *   GATHER: one CTA per row, each warp owns a K slice (the paper's SPLIT_OUT_DIM); UNION: the union
 *   pipeline with the scattered TwELL values as H (no up GEMM).  Workspace as sffn_up_down.
 * sffn_forward_nongated: sffn_pack(X, Wu) into the workspace, then sffn_down (workspace as sffn_forward). */
int sffn_down(const uint32_t* twell, const void* Wd, int64_t M, int64_t K, int64_t N, int T, int C, void* Y,
              void* workspace, size_t ws_bytes, int algo, void* stream);
int sffn_forward_nongated(const void* X, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N, int T,
                          int C, void* Y, void* workspace, size_t ws_bytes, uint32_t* d_overflow, int algo,
                          void* stream);

/*
 * sffn_forward_host — sffn_forward with X and Y in HOST memory (page-locked for overlap): rows are
 * processed in chunks of at most `chunk_rows` (a multiple of 128; a multiple of 2048 keeps the UNION row
 * permutation windows, hence the results, identical to one sffn_forward call).  Chunk sizes ramp up
 * geometrically from chunk_rows/4 at the start and back down at the end (short pipeline fill / drain),
 * full-size chunks in between (the forward's per-call cost amortised); the host->device copy of
 * chunk i+1 and the device->host copy of chunk i-1 overlap the compute of chunk i on two internal copy
 * streams (created once per device, event-ordered; no host synchronization).  The call is
 * stream-ordered on `stream`: Y_host is complete when `stream` reaches this point.
 *   stage: device buffer >= sffn_forward_host_stage_bytes(K, chunk_rows) (2 X + 2 Y chunk slots); a larger
 *     buffer gives more slots (stage_bytes / (2 x slot), up to one per chunk), so fewer copies wait for a slot
 *   workspace: >= sffn_forward_workspace_bytes(min(chunk_rows, M), K, N, T, C, algo); with twice that (plus 1 KiB
 *     alignment) consecutive chunks compute on two streams (`stream` and an internal one) so a chunk's kernels
 *     overlap the previous chunk's tail
 */
size_t sffn_forward_host_stage_bytes(int64_t K, int64_t chunk_rows);
/* The chunk schedule sffn_forward_host uses (host only, no device work): writes up to `cap` chunk row
 * counts to `sizes` (may be null) and returns the number of chunks; 0 on a bad argument. */
int64_t sffn_forward_host_chunks(int64_t M, int64_t chunk_rows, int64_t* sizes, int64_t cap);
int sffn_forward_host(const void* X_host, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K,
                      int64_t N, int T, int C, void* Y_host, void* workspace, size_t ws_bytes, void* stage,
                      size_t stage_bytes, uint32_t* d_overflow, int algo, int64_t chunk_rows, void* stream);

/*
 * sffn_dense_forward — the library's own dense tcgen05 FFN (Eq.1 without sparsity): the speedup
 * denominator.  Launch 1: fused gate||up GEMM with epilogue H = bf16(relu(g) * u)   (H [M, N] bf16,
 * caller-owned).  Launch 2: Y = H W_d as a GEMM against WdT = W_d^T stored [K, N] row-major (a
 * one-time weight layout for the dense model; sffn_transpose_bf16 produces it).
 */
int sffn_dense_forward(const void* X, const void* Wg, const void* Wu, const void* WdT, int64_t M, int64_t K,
                       int64_t N, void* H, void* Y, void* stream);

/* out[c, r] = in[r, c] for a bf16 [rows, cols] matrix (weight-layout utility). */
int sffn_transpose_bf16(const void* in, int64_t rows, int64_t cols, void* out, void* stream);

/*
 * sffn_gate_gemm_f32 — verification: the raw fp32 accumulators S = X W_g^T of the same tcgen05
 * mainloop sffn_pack uses (S [M, N] float, output).  Used to prove the tensor-core accumulation is
 * exact on dyadic-grid inputs.
 */
int sffn_gate_gemm_f32(const void* X, const void* Wg, int64_t M, int64_t K, int64_t N, float* S, void* stream);

/*
 * sffn_union_stats — measurement helper for SFFN_ALGO_UNION: after sffn_up_down (workspace = its
 * workspace) synchronizes `stream` and returns the sum over union blocks (B = sffn_union_block_rows()
 * token rows each) of the padded union sizes (the tensor-core work is 4 * B * padded_sum * K FLOP), of
 * the exact union sizes, and the number of up-GEMM tiles.  Any output pointer may be NULL.
 */
/* Token rows per union block of SFFN_ALGO_UNION in this process: 128 (single-CTA union GEMMs, M=128 tiles)
 * or 256 (CTA-pair union GEMMs, cta_group::2 M=256 tiles; environment SFFN_UNION_PAIR=1 at first use). */
int sffn_union_block_rows(void);
int sffn_union_stats(const void* workspace, int64_t M, int64_t K, int64_t N, int64_t* padded_sum, int64_t* real_sum,
                     int64_t* up_tiles, void* stream);

/*
 * sffn_overflow_check — synchronizes `stream`, copies *d_overflow to *host_count (if non-NULL) and
 * returns SFFN_ERR_TILE_OVERFLOW if it is non-zero, else SFFN_OK.
 */
int sffn_overflow_check(const uint32_t* d_overflow, void* stream, uint32_t* host_count);

/* ---------------------------------------------------------------- fp32 mode (reading R19)
 * fp32 inputs and weights, fp32 accumulation everywhere (north_star: Y within 1e-5 relative Frobenius
 * "in an fp32 mode").  The TwELL is the logical (SoA) form of Alg.1's outputs:
 *   h_v float [M, N/C], h_I uint16 [M, N/C] (shard-local column), h_nz uint32 [M, N/T] (true count);
 *   tile t of row m owns slots [t*T/C, (t+1)*T/C) of h_v / h_I (capacity T/C: no count word).
 * The gate GEMM is a SIMT fp32 GEMM (tensor-core tf32 would round the inputs to 10-bit mantissas);
 * its epilogue compacts each row-tile with warp ballot / popc, ascending columns.  Not a perf path.
 * Constraints: K % 4 == 0 (and K <= 8192 for the up/down), N % T == 0, N <= 65536; X/W/Y 16-B aligned. */
size_t sffn_f32_twell_bytes(int64_t M, int64_t N, int T, int C);
int sffn_pack_f32(const float* X, const float* Wg, int64_t M, int64_t K, int64_t N, int T, int C, float* h_v,
                  uint16_t* h_I, uint32_t* h_nz, uint32_t* d_overflow, void* stream);
int sffn_up_down_f32(const float* X, const float* h_v, const uint16_t* h_I, const uint32_t* h_nz, const float* Wu,
                     const float* Wd, int64_t M, int64_t K, int64_t N, int T, int C, float* Y, void* stream);
/* workspace >= sffn_f32_twell_bytes(M, N, T, C): h_v, then h_I, then h_nz (each 1 KiB aligned). */
int sffn_forward_f32(const float* X, const float* Wg, const float* Wu, const float* Wd, int64_t M, int64_t K,
                     int64_t N, int T, int C, float* Y, void* workspace, size_t ws_bytes, uint32_t* d_overflow,
                     void* stream);

/* ---------------------------------------------------------------- training forward on the hybrid format (NEXT-4)
 * After sffn_twell_to_hybrid (the pattern of h_g), the paper's training forward computes h = h_g (.) x W_u on that
 * pattern (dense -> hybrid, Listing 5; dense tail: tensor-core GEMM times the pattern mask, Alg.3
 * P:220-239) and y = h W_d (hybrid -> dense, Listing 6; dense tail: tensor-core GEMM, rows
 * scattered to their tokens, Alg.3 lines 14-17).  Hybrid operands use sffn_twell_to_hybrid's layout: ell_col
 * int16 [M, ell_w] (read as uint16 unit ids), row_nnz [M], row_loc [M] (-1 ELL row, s >= 0 dense-tail slot,
 * -2 dropped), dense_map [D] (slot -> row), *d_dense_count (device; slots used = min(count, D)), values bf16.
 *
 * sffn_hybrid_sddmm: A [M, K] bf16, B [N, K] bf16 (hidden-major, e.g. W_u).  ELL rows: out_ell[m, j] =
 *   bf16(g * sum_k A[m,k] B[ell_col[m,j], k]) for j < min(row_nnz[m], ell_w) (other slots untouched), g =
 *   P_ell[m, j] when gate != 0, else 1; dense tail slots s: out_dense[s, n] = P_dense[s, n] != 0 ?
 *   bf16(g * (A[dense_map[s]] . B[n])) : 0, g = P_dense[s, n] (gate) or 1.  fp32 accumulation (the tail dot
 *   products on tcgen05 in fp32, rounded once with the gate).  Requires K % 64 == 0, N % 16 == 0 and, with a
 *   dense tail (D > 0), N >= 256 and workspace >= sffn_hybrid_mm_workspace_bytes(D, K, N).
 * sffn_hybrid_spmm: Y [M, K] bf16: ELL rows Y[m] = sum_j ell_val[m,j] W[ell_col[m,j], :] (CUDA cores, fp32);
 *   tail slots Y[dense_map[s]] = dense[s, :] W (tcgen05, W [N, K] read MN-major by TMA, no transpose); dropped
 *   rows are zero.  Requires K % 64 == 0, K >= 256, N % 64 == 0; workspace as above when D > 0.
 * Caller-owned device memory, stream-ordered, no host synchronization. */
size_t sffn_hybrid_mm_workspace_bytes(int64_t D, int64_t K, int64_t N);
/* sffn_forward_train — the training forward through the union tensor-core path: sffn_forward (algo UNION) gives
 * Y, then the TwELL is converted to the hybrid format (as sffn_twell_to_hybrid: pattern, h_g values in
 * ell_g / dense_g, dense_map, *d_dense_count zeroed by the caller, L0/L1) and h = h_g (.) x W_u — the values the
 * SDDMM computes on that pattern, already in the union GEMM's H_c buffer — is copied out in the same hybrid
 * layout (ell_h [M, ell_w], dense_h [dense_cap, N], bf16) for the backward pass.  One call instead of
 * pack + SDDMM + SpMM; workspace >= sffn_forward_workspace_bytes(M, K, N, T, C, SFFN_ALGO_UNION); N % 64 == 0. */
int sffn_forward_train(const void* X, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N,
                       int T, int C, void* Y, int ell_w, void* ell_g, void* ell_h, int16_t* ell_col, int32_t* row_nnz,
                       int32_t* row_loc, int64_t dense_cap, void* dense_g, void* dense_h, int32_t* dense_map,
                       int* d_dense_count, double* d_l0l1, void* workspace, size_t ws_bytes, uint32_t* d_overflow,
                       void* stream);
int sffn_hybrid_sddmm(const void* A, const void* B, int64_t M, int64_t K, int64_t N, int ell_w, const int16_t* ell_col,
                      const int32_t* row_nnz, const int32_t* row_loc, const void* P_ell, int64_t D,
                      const int32_t* dense_map, const int* d_dense_count, const void* P_dense, int gate, void* out_ell,
                      void* out_dense, void* workspace, size_t ws_bytes, void* stream);
int sffn_hybrid_spmm(const void* ell_val, const int16_t* ell_col, const int32_t* row_nnz, const int32_t* row_loc,
                     int64_t M, int ell_w, int64_t D, const int32_t* dense_map, const int* d_dense_count,
                     const void* dense, const void* W, int64_t N, int64_t K, void* Y, void* workspace, size_t ws_bytes,
                     void* stream);

/* ---------------------------------------------------------------- multi-GPU (hidden-dim shards)
 * One process per GPU.  Rank r owns hidden units [n_offset, n_offset + N_local) — contiguous row
 * blocks of all three [N, K] weights — packs its own TwELL (local indices), computes the partial
 * Y_r = sum_{n in shard} h W_d[n, :], and the partials are summed with ONE NCCL all-reduce (bf16,
 * sum) over NVLink / NVSwitch (north_star (5)).  X is replicated on every rank.
 */
typedef struct sffn_comm sffn_comm;

/* Fills 128 bytes with a new NCCL unique id (call on rank 0, broadcast it yourself). */
int sffn_comm_unique_id(void* id128);
/* Creates the library's own NCCL communicator on `cuda_device` (must be the current device). */
int sffn_comm_init(sffn_comm** out, int nranks, int rank, const void* id128, int cuda_device);
int sffn_comm_destroy(sffn_comm* comm);
int sffn_comm_size(const sffn_comm* comm);

/*
 * sffn_sharded_forward — sffn_forward on the local shard, then one in-place NCCL all-reduce (sum)
 * of Y [M, K] bf16 on `stream`.  With n_chunks > 1 (and M >= 4096) the M dimension is processed in chunks
 * (multiples of the 2048-row pi windows, so the result is bit-identical to n_chunks = 1) and the
 * all-reduce of chunk i overlaps the compute of chunk i+1 (the library orders
 * them with events on an internal communication stream; still no host synchronization).  The
 * workspace (>= sffn_forward_workspace_bytes(M, K, N_local, T, C, algo)) is reused chunk after chunk.
 */
int sffn_sharded_forward(sffn_comm* comm, const void* X, const void* Wg_s, const void* Wu_s, const void* Wd_s,
                         int64_t M, int64_t K, int64_t N_local, int T, int C, void* Y, void* workspace,
                         size_t ws_bytes, uint32_t* d_overflow, int algo, int n_chunks, void* stream);

/* Plain in-place all-reduce (sum) of a bf16 buffer on the communicator (used by tests). */
int sffn_allreduce_bf16(sffn_comm* comm, void* buf, int64_t count, void* stream);

/* ---------------------------------------------------------------- NEXT-3: symmetric-memory all-reduce
 * The NCCL all-reduce above launches NCCL's kernels.  The symmetric path replaces it with the library's
 * own reduction kernel over peer memory (SURVEY §8(e) "B200-native upgrade", §8(f) NEXT-3):
 *   - sffn_comm_symmetric_init (collective: every rank calls it with the same arguments) allocates one
 *     buffer of max_rows x K bf16 with ncclMemAlloc, registers it as a symmetric window
 *     (ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC) and creates an NCCL device communicator with
 *     SYM_CTAS load/store-accessible (LSA) barriers and, when NCCL can build one (NVSwitch, >= 2 ranks),
 *     a multicast (NVLS) object.  Returns SFFN_ERR_UNSUPPORTED when the platform cannot (the NCCL path
 *     stays available); once per communicator; freed by sffn_comm_destroy.
 *   - sffn_sharded_forward_sym: sffn_forward of the local shard whose DOWN epilogue writes the partial Y
 *     straight into the window, then ONE launch of the library's reduction kernel: LSA barrier; rank r
 *     reduces its 1/G slice of 16-byte chunks — multimem.ld_reduce.add.acc::f32 (the switch sums the G
 *     copies in fp32) + multimem.st (the switch writes the sum into every rank's window) with NVLS, else
 *     P2P loads of the slice from every peer window, fp32 sum, P2P stores into every window; LSA barrier;
 *     local copy window -> Y.  Y [M, K] bf16 (caller-owned device memory), M <= max_rows, same K.
 *     Sum order: fp32 over ranks, one rounding to bf16 (the NCCL bf16 ring rounds per hop).
 *   - sffn_allreduce_sym_bf16: the reduction alone on `rows` x K bf16 (src copied into the window first
 *     unless src is NULL, i.e. already there); result in Y.
 * Errors: SFFN_ERR_UNSUPPORTED if symmetric_init has not succeeded; SFFN_ERR_SHAPE if M > max_rows or K
 * differs; all enqueued on `stream`, no host synchronization.
 */
int sffn_comm_symmetric_init(sffn_comm* comm, int64_t max_rows, int64_t K);
/* multimem = 1 when the NVLS (multicast) reduction is used, 0 for P2P loads / stores. */
int sffn_comm_symmetric_info(const sffn_comm* comm, int* multimem, int64_t* max_rows, int64_t* K);
int sffn_allreduce_sym_bf16(sffn_comm* comm, const void* src, void* Y, int64_t rows, int64_t K, void* stream);
/* Reduce-scatter variant (sequence-parallel consumers): rank r receives the sum over ranks of rows
 * [rows*r/G, rows*(r+1)/G) of the partials (src copied into the window first unless NULL) in Y_slice
 * [*nrows, K] bf16; *row0 / *nrows (may be NULL) report the slice.  Same kernel structure as the all-reduce
 * without the broadcast store. */
int sffn_reduce_scatter_sym_bf16(sffn_comm* comm, const void* src, int64_t rows, int64_t K, void* Y_slice,
                                 int64_t* row0, int64_t* nrows, void* stream);
/* sffn_sharded_forward_fused — the all-reduce fused into the DOWN GEMM at 2048-row-window granularity (one pi
 * window = one DOWN raster group): after each output tile the DOWN epilogue warps count their rows at the window's
 * owner rank (w % G; system-scope atomic on the owner's window counter through the LSA mapping), and an otherwise
 * idle warp of every DOWN CTA waits for the owned windows in raster order and reduces its slice of each across the
 * ranks' windows (NVLS multimem.ld_reduce / multimem.st, else P2P) while later windows still compute; a final LSA
 * barrier and the local copy window -> Y end the call.  Union path only (single-CTA union GEMMs); needs
 * sffn_comm_symmetric_init with max_rows >= M; two counter sets alternate call by call (the closing kernel zeroes
 * the set it used and selects the other one on the device, so CUDA-graph replays alternate too); every rank must
 * make the same sequence of calls (any M <= max_rows).
 * A counter that does not reach its target within about a minute (a rank gone) traps the kernel: the call's
 * stream reports a launch failure instead of hanging. */
int sffn_sharded_forward_fused(sffn_comm* comm, const void* X, const void* Wg_s, const void* Wu_s, const void* Wd_s,
                               int64_t M, int64_t K, int64_t N_local, int T, int C, void* Y, void* workspace,
                               size_t ws_bytes, uint32_t* d_overflow, void* stream);
int sffn_sharded_forward_sym(sffn_comm* comm, const void* X, const void* Wg_s, const void* Wu_s, const void* Wd_s,
                             int64_t M, int64_t K, int64_t N_local, int T, int C, void* Y, void* workspace,
                             size_t ws_bytes, uint32_t* d_overflow, int algo, void* stream);

/* sffn__forward_fused — INTERNAL (the engine of sffn_sharded_forward_fused, exported for the emulated-rank tests;
 * not a stable API).  The union forward of one rank's shard whose DOWN GEMM writes the partial Y into Y (= this
 * rank's window) and runs the window-granular reduction.  ptrs: DEVICE uint64 table of G + 2 entries — the G
 * window base addresses as this rank can address them, the multicast address of the windows (0: P2P path), and
 * the byte offset of the counter set to use (each window: Y region, then the per-2048-row-window uint32
 * counters, zero before the call).  phase 0: the whole forward; 1: pack, metadata and the UP GEMM only; 2: the
 * fused DOWN GEMM only (after a phase-1 call on the same workspace).  The G ranks' DOWN kernels must be able to
 * run concurrently (a counter that never completes traps the kernel after about a minute).  No barrier, no
 * counter reset and no copy-out: the caller does those (sffn_sharded_forward_fused's closing kernel).
 * Errors: as sffn_forward; SFFN_ERR_UNSUPPORTED when the union path does not apply (N, SFFN_UNION_PAIR). */
int sffn__forward_fused(const void* X, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K,
                        int64_t N, int T, int C, void* Y, void* workspace, size_t ws_bytes, uint32_t* d_overflow,
                        const uint64_t* ptrs, int G, int rank, int phase, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SFFN_H_ */
