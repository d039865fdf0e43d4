/*
 * oracle.c — CPU ORACLE for the sparse gated-FFN forward (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_2603_23198_b200/) never links,
 * imports or calls it, and shares no code with it.
 *
 * Plain, slow, obviously-correct definitions, written from /root/reference/PAPER.md
 * (cited as P:<line>).  Floating point is fp64 with k ascending; no blocking, fusion or
 * reordering beyond what the cited definition states.  Rows are independent (OpenMP over
 * rows only), so results do not depend on the thread count.
 *
 * Conventions:
 *   - all weights are stored hidden-major [N, K] row-major (R11: P:55, P:1078, L1 P:464)
 *   - inputs are bf16 bit patterns (uint16), widened exactly to double
 *   - TwELL packed word layout (P:869, L1 P:817-834): per (row, tile) block of T/C
 *     uint32 words, word 0 = count, word 1+j = col | bf16(value) << 16; capacity T/C-1
 *
 * Pins (tests/test_oracle_pins.py): the paper's / SPEC's worked examples
 * (tests/golden/), exact integer arithmetic on dyadic-grid inputs, brute-force
 * compaction, permutation-matrix closed forms, Eq.1 == Eq.3 identity, invariants.
 * Parity unpinned: nothing.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* bf16 is the upper 16 bits of an IEEE binary32 ("bfloat16"); widening is exact. */
double oracle_bf16_to_double(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* float -> bf16, round to nearest even: the paper stores __float2bfloat16(C_accum)
 * (L1 P:824-826), which is IEEE round-to-nearest-even.  NaN is not produced here. */
uint16_t oracle_f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    uint32_t lsb = (u >> 16) & 1u;
    uint32_t rounded = u + 0x7FFFu + lsb;
    return (uint16_t)(rounded >> 16);
}

/* Gate pre-activation of Eq.1: A[m,n] = sum_k x[m,k] * W_g[n,k]  (fp64, k ascending). */
void oracle_gate_preact(const uint16_t* X, const uint16_t* Wg, int64_t M, int64_t K, int64_t N, double* A) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t n = 0; n < N; ++n) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k)
                acc += oracle_bf16_to_double(X[m * K + k]) * oracle_bf16_to_double(Wg[n * K + k]);
            A[m * N + n] = acc;
        }
    }
}

/*
 * Alg.1 lines 7-17 for every row, on the fp32 tile values S (the paper
 * thresholds the fp32 accumulator, L1 P:803-808), packed as in P:869 / L1 P:817-834:
 *
 *   for r: for each tile n0 (T = T_n columns):
 *     z <- 0
 *     for c in 0..T-1:  if S[r, n0+c] > 0:            (strict, Alg.1 line 11)
 *        if z < cap: h_I <- n0+c ; h_v <- S           (lines 12-14; cap = T/C - 1)
 *        z <- z + 1                                   (line 15)
 *     h_nz[r, n0/T] <- z                              (line 17; true count, reading R5)
 *
 * words: uint32 [M, N/C]; counts (may be NULL): uint32 [M, N/T].  Slots beyond the count
 * are left untouched (no padding value).  Returns the number of (row, tile)
 * blocks whose count exceeded the capacity.
 */
int64_t oracle_pack(const float* S, int64_t M, int64_t N, int T, int C, uint32_t* words, uint32_t* counts) {
    const int64_t NT = N / T, W = T / C, cap = W - 1;
    int64_t overflow = 0;
#pragma omp parallel for schedule(static) reduction(+ : overflow)
    for (int64_t r = 0; r < M; ++r) {
        for (int64_t t = 0; t < NT; ++t) {
            const int64_t n0 = t * T;
            uint32_t* blk = words + r * (N / C) + t * W;
            int64_t z = 0;
            for (int64_t c = 0; c < T; ++c) {
                float s = S[r * N + n0 + c];
                if (s > 0.0f) {
                    if (z < cap) {
                        uint32_t idx = (uint32_t)(n0 + c);
                        uint32_t val = oracle_f32_to_bf16_rne(s);
                        blk[1 + z] = (idx & 0xFFFFu) | (val << 16);
                    }
                    z += 1;
                }
            }
            blk[0] = (uint32_t)z;
            if (counts) counts[r * NT + t] = (uint32_t)z;
            if (z > cap) overflow += 1;
        }
    }
    return overflow;
}

/* TwELL -> dense (SPEC S:167-175 twell_to_dense): H[m, col] = value for the valid prefix
 * min(count, cap) of every (row, tile) block, +0 elsewhere.  H is float [M, N]. */
void oracle_unpack(const uint32_t* words, int64_t M, int64_t N, int T, int C, float* H) {
    const int64_t NT = N / T, W = T / C, cap = W - 1;
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t n = 0; n < N; ++n) H[m * N + n] = 0.0f;
        for (int64_t t = 0; t < NT; ++t) {
            const uint32_t* blk = words + m * (N / C) + t * W;
            int64_t z = blk[0];
            if (z > cap) z = cap;
            for (int64_t j = 0; j < z; ++j) {
                uint32_t w = blk[1 + j];
                H[m * N + (w & 0xFFFFu)] = (float)oracle_bf16_to_double((uint16_t)(w >> 16));
            }
        }
    }
}

/* Eq.1 with sigma = relu, fp64:
 *   h_g = relu(x W_g), h_u = x W_u, h = h_u * h_g, y = h W_d.
 * With hidden-major storage, (x W_g)[m,n] = sum_k x[m,k] Wg[n,k] and (h W_d)[m,j] = sum_n h[m,n] Wd[n,j].
 * Y is double [M, K]; H (optional, may be NULL) receives h as double [M, N]. */
void oracle_ffn_dense(const uint16_t* X, const uint16_t* Wg, const uint16_t* Wu, const uint16_t* Wd, int64_t M,
                      int64_t K, int64_t N, double* Y, double* H) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t j = 0; j < K; ++j) Y[m * K + j] = 0.0;
        for (int64_t n = 0; n < N; ++n) {
            double g = 0.0, u = 0.0;
            for (int64_t k = 0; k < K; ++k) {
                double x = oracle_bf16_to_double(X[m * K + k]);
                g += x * oracle_bf16_to_double(Wg[n * K + k]);
                u += x * oracle_bf16_to_double(Wu[n * K + k]);
            }
            double hg = g > 0.0 ? g : 0.0;
            double h = u * hg;
            if (H) H[m * N + n] = h;
            if (h != 0.0)
                for (int64_t j = 0; j < K; ++j) Y[m * K + j] += h * oracle_bf16_to_double(Wd[n * K + j]);
        }
    }
}

/*
 * Eq.3 / Alg.2 over a packed TwELL:
 *   y[m,:] = sum_t sum_{c < h_nz[m,t]} h_v[m, t T/C + c] * (x[m,:] . W_u[n,:]) * W_d[n,:],  n = h_I[...]
 * Only the stored prefix min(h_nz, cap) exists (reading R5).  gate_mode 0: h_v is the stored bf16
 * value (the paper's pipeline, L2 P:994-1002 multiplies by it); gate_mode 1: h_v is replaced by the
 * exact fp64 pre-activation A[m, n] (A must then be given) — the form that equals Eq.1 exactly.
 * Y is double [M, K]. fp64, entries in stored (ascending column) order.
 */
void oracle_ffn_twell(const uint16_t* X, const uint32_t* words, const uint16_t* Wu, const uint16_t* Wd, int64_t M,
                      int64_t K, int64_t N, int T, int C, int gate_mode, const double* A, double* Y) {
    const int64_t NT = N / T, W = T / C, cap = W - 1;
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t j = 0; j < K; ++j) Y[m * K + j] = 0.0;
        for (int64_t t = 0; t < NT; ++t) {
            const uint32_t* blk = words + m * (N / C) + t * W;
            int64_t z = blk[0];
            if (z > cap) z = cap;
            for (int64_t c = 0; c < z; ++c) {
                uint32_t w = blk[1 + c];
                int64_t n = (int64_t)(w & 0xFFFFu);
                double hv = gate_mode == 1 ? A[m * N + n] : oracle_bf16_to_double((uint16_t)(w >> 16));
                double u = 0.0;
                for (int64_t k = 0; k < K; ++k)
                    u += oracle_bf16_to_double(X[m * K + k]) * oracle_bf16_to_double(Wu[n * K + k]);
                double h = hv * u;
                for (int64_t j = 0; j < K; ++j) Y[m * K + j] += h * oracle_bf16_to_double(Wd[n * K + j]);
            }
        }
    }
}

/* fp32-input variants of the gate pre-activation and dense FFN (fp32 mode, reading R19). */
void oracle_gate_preact_f32(const float* X, const float* Wg, int64_t M, int64_t K, int64_t N, double* A) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k) acc += (double)X[m * K + k] * (double)Wg[n * K + k];
            A[m * N + n] = acc;
        }
}

/*
 * fp32 mode (reading R19): Alg.1 lines 7-17 producing the logical SoA outputs of Alg.1
 * (P:88-89): h_v [M, N/C] float, h_I [M, N/C] uint16, h_nz [M, N/T]; capacity T/C (no count word);
 * true count kept (R5).  Returns the number of overflowed (row, tile) blocks.
 */
int64_t oracle_pack_soa(const float* S, int64_t M, int64_t N, int T, int C, float* hv, uint16_t* hi, uint32_t* hnz) {
    const int64_t NT = N / T, W = T / C, cap = W;
    int64_t overflow = 0;
#pragma omp parallel for schedule(static) reduction(+ : overflow)
    for (int64_t r = 0; r < M; ++r) {
        for (int64_t t = 0; t < NT; ++t) {
            const int64_t n0 = t * T;
            int64_t z = 0;
            for (int64_t c = 0; c < T; ++c) {
                float s = S[r * N + n0 + c];
                if (s > 0.0f) {
                    if (z < cap) {
                        hv[r * (N / C) + t * W + z] = s;
                        hi[r * (N / C) + t * W + z] = (uint16_t)(n0 + c);
                    }
                    z += 1;
                }
            }
            hnz[r * NT + t] = (uint32_t)z;
            if (z > cap) overflow += 1;
        }
    }
    return overflow;
}

/* Eq.1 with fp32 inputs, fp64 arithmetic.  Y double [M, K]. */
void oracle_ffn_dense_f32(const float* X, const float* Wg, const float* Wu, const float* Wd, int64_t M, int64_t K,
                          int64_t N, double* Y) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t j = 0; j < K; ++j) Y[m * K + j] = 0.0;
        for (int64_t n = 0; n < N; ++n) {
            double g = 0.0, u = 0.0;
            for (int64_t k = 0; k < K; ++k) {
                g += (double)X[m * K + k] * (double)Wg[n * K + k];
                u += (double)X[m * K + k] * (double)Wu[n * K + k];
            }
            double h = (g > 0.0 ? g : 0.0) * u;
            if (h != 0.0)
                for (int64_t j = 0; j < K; ++j) Y[m * K + j] += h * (double)Wd[n * K + j];
        }
    }
}

/* Eq.3 over the SoA TwELL, fp32 inputs, fp64 arithmetic, gate = stored h_v. */
void oracle_ffn_soa_f32(const float* X, const float* hv, const uint16_t* hi, const uint32_t* hnz, const float* Wu,
                        const float* Wd, int64_t M, int64_t K, int64_t N, int T, int C, double* Y) {
    const int64_t NT = N / T, W = T / C;
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t j = 0; j < K; ++j) Y[m * K + j] = 0.0;
        for (int64_t t = 0; t < NT; ++t) {
            int64_t z = hnz[m * NT + t];
            if (z > W) z = W;
            for (int64_t c = 0; c < z; ++c) {
                const int64_t o = m * (N / C) + t * W + c;
                const int64_t n = hi[o];
                double u = 0.0;
                for (int64_t k = 0; k < K; ++k) u += (double)X[m * K + k] * (double)Wu[n * K + k];
                const double h = (double)hv[o] * u;
                for (int64_t j = 0; j < K; ++j) Y[m * K + j] += h * (double)Wd[n * K + j];
            }
        }
    }
}

/* Non-gated FFN, App.C eq.: h = relu(x W_u), y = h W_d, fp64.  Y double [M, K]. */
void oracle_ffn_nongated_dense(const uint16_t* X, const uint16_t* Wu, const uint16_t* Wd, int64_t M, int64_t K,
                               int64_t N, double* Y) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t j = 0; j < K; ++j) Y[m * K + j] = 0.0;
        for (int64_t n = 0; n < N; ++n) {
            double a = 0.0;
            for (int64_t k = 0; k < K; ++k)
                a += oracle_bf16_to_double(X[m * K + k]) * oracle_bf16_to_double(Wu[n * K + k]);
            if (a > 0.0)
                for (int64_t j = 0; j < K; ++j) Y[m * K + j] += a * oracle_bf16_to_double(Wd[n * K + j]);
        }
    }
}

/* Down projection from a packed TwELL of h (Listing 3 semantics):
 *   y[m,:] = sum over the stored entries (n, h_v) of h_v * W_d[n,:]   (fp64, stored order).
 * gate_mode 1: h_v replaced by the exact A[m, n] (then equals the dense non-gated FFN exactly). */
void oracle_down_twell(const uint32_t* words, const uint16_t* Wd, int64_t M, int64_t K, int64_t N, int T, int C,
                       int gate_mode, const double* A, double* Y) {
    const int64_t NT = N / T, W = T / C, cap = W - 1;
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t j = 0; j < K; ++j) Y[m * K + j] = 0.0;
        for (int64_t t = 0; t < NT; ++t) {
            const uint32_t* blk = words + m * (N / C) + t * W;
            int64_t z = blk[0];
            if (z > cap) z = cap;
            for (int64_t c = 0; c < z; ++c) {
                uint32_t w = blk[1 + c];
                int64_t n = (int64_t)(w & 0xFFFFu);
                double h = gate_mode == 1 ? A[m * N + n] : oracle_bf16_to_double((uint16_t)(w >> 16));
                for (int64_t j = 0; j < K; ++j) Y[m * K + j] += h * oracle_bf16_to_double(Wd[n * K + j]);
            }
        }
    }
}

/*
 * TwELL -> ELL part of the hybrid format with L0/L1 statistics (Listing 4; hybrid P:177-182):
 * row m's stored entries in tile order (ascending columns) fill ell_col/ell_val[m, 0 .. min(nnz, ell_w));
 * row_nnz[m] = stored count; l0l1[0] = sum_m nnz_m / M, l1l1[1] = sum_m sum(values_m) / M (fp64).
 */
void oracle_twell_to_ell(const uint32_t* words, int64_t M, int64_t N, int T, int C, int64_t ell_w,
                         uint16_t* ell_val, int16_t* ell_col, int32_t* row_nnz, double* l0l1) {
    const int64_t NT = N / T, W = T / C, cap = W - 1;
    double l0 = 0.0, l1 = 0.0;
    for (int64_t m = 0; m < M; ++m) {
        int64_t k = 0;
        double vs = 0.0;
        for (int64_t t = 0; t < NT; ++t) {
            const uint32_t* blk = words + m * (N / C) + t * W;
            int64_t z = blk[0];
            if (z > cap) z = cap;
            for (int64_t c = 0; c < z; ++c, ++k) {
                uint32_t w = blk[1 + c];
                vs += oracle_bf16_to_double((uint16_t)(w >> 16));
                if (k < ell_w) {
                    ell_val[m * ell_w + k] = (uint16_t)(w >> 16);
                    ell_col[m * ell_w + k] = (int16_t)(w & 0xFFFFu);
                }
            }
        }
        row_nnz[m] = (int32_t)k;
        l0 += (double)k / (double)M;
        l1 += vs / (double)M;
    }
    l0l1[0] = l0;
    l0l1[1] = l1;
}

/*
 * Hybrid SDDMM, dense -> hybrid (training forward h = h_g (.) x W_u on the gate pattern; Listing 5 P:1316-1378 for
 * the ELL part, Alg.3 P:220-239 and P:1380 "multiplied by a binary mask containing the sparsity pattern" for the
 * dense tail).  ELL rows (row_loc[m] == -1), j < row_nnz[m]:
 *   out_ell[m, j] = g * sum_k A[m, k] B[n, k],  n = (uint16) ell_col[m, j],  g = P_ell[m, j] (gate) or 1;
 * dense-tail slots s < n_dense, m = dense_map[s]:
 *   out_dense[s, n] = P_dense[s, n] != 0 ? g * sum_k A[m, k] B[n, k] : 0,  g = P_dense[s, n] (gate) or 1.
 * Other entries untouched.  A [M, K], B [N, K] (hidden-major weights), P_* bf16; fp64, k ascending.
 */
void oracle_hybrid_sddmm(const uint16_t* A, const uint16_t* B, int64_t M, int64_t K, int64_t N, int64_t ell_w,
                         const int16_t* ell_col, const int32_t* row_nnz, const int32_t* row_loc,
                         const uint16_t* P_ell, int64_t n_dense, const int32_t* dense_map, const uint16_t* P_dense,
                         int gate, double* out_ell, double* out_dense) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        if (row_loc[m] != -1) continue;
        int64_t z = row_nnz[m] < ell_w ? row_nnz[m] : ell_w;
        for (int64_t j = 0; j < z; ++j) {
            int64_t n = (int64_t)(uint16_t)ell_col[m * ell_w + j];
            double s = 0.0;
            for (int64_t k = 0; k < K; ++k) s += oracle_bf16_to_double(A[m * K + k]) * oracle_bf16_to_double(B[n * K + k]);
            double g = gate ? oracle_bf16_to_double(P_ell[m * ell_w + j]) : 1.0;
            out_ell[m * ell_w + j] = g * s;
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < n_dense; ++s) {
        int64_t m = dense_map[s];
        for (int64_t n = 0; n < N; ++n) {
            double p = oracle_bf16_to_double(P_dense[s * N + n]);
            if (p == 0.0) {
                out_dense[s * N + n] = 0.0;
                continue;
            }
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k) acc += oracle_bf16_to_double(A[m * K + k]) * oracle_bf16_to_double(B[n * K + k]);
            out_dense[s * N + n] = (gate ? p : 1.0) * acc;
        }
    }
}

/*
 * Hybrid SpMM, hybrid -> dense (training forward y = h W_d; Listing 6, Alg.3):
 *   ELL rows (row_loc[m] == -1): Y[m, :] = sum_{j < min(row_nnz[m], ell_w)} v[m, j] W[(uint16) ell_col[m, j], :];
 *   dense-tail slots s < n_dense: Y[dense_map[s], :] = sum_n D[s, n] W[n, :];
 *   dropped rows (row_loc[m] == -2, tail full): Y[m, :] = 0.
 * Values v / D in fp64 (so the oracle chain SDDMM -> SpMM stays unrounded), W [N, K] bf16; fp64, n ascending.
 */
void oracle_hybrid_spmm(const double* ell_val, const int16_t* ell_col, const int32_t* row_nnz, const int32_t* row_loc,
                        int64_t M, int64_t ell_w, int64_t n_dense, const int32_t* dense_map, const double* D,
                        const uint16_t* W, int64_t N, int64_t K, double* Y) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t k = 0; k < K; ++k) Y[m * K + k] = 0.0;
        if (row_loc[m] != -1) continue;
        int64_t z = row_nnz[m] < ell_w ? row_nnz[m] : ell_w;
        for (int64_t j = 0; j < z; ++j) {
            int64_t n = (int64_t)(uint16_t)ell_col[m * ell_w + j];
            double v = ell_val[m * ell_w + j];
            for (int64_t k = 0; k < K; ++k) Y[m * K + k] += v * oracle_bf16_to_double(W[n * K + k]);
        }
    }
    for (int64_t s = 0; s < n_dense; ++s) {
        int64_t m = dense_map[s];
        for (int64_t n = 0; n < N; ++n) {
            double v = D[s * N + n];
            if (v == 0.0) continue;
            for (int64_t k = 0; k < K; ++k) Y[m * K + k] += v * oracle_bf16_to_double(W[n * K + k]);
        }
    }
}
