// hybrid_mm.cuh — the training forward on the hybrid format (after sffn_twell_to_hybrid):
//   SDDMM (dense -> hybrid): h = h_g (.) x W_u on the gate pattern — Listing 5 for the ELL rows, the
//         dense tail by a tcgen05 GEMM times the pattern mask (Alg.3);
//   SpMM  (hybrid -> dense): y = h W_d — Listing 6 for the ELL rows, the dense tail by a tcgen05 GEMM
//         whose rows are scattered to their token rows (Alg.3 lines 14-17).
// The CUDA-core ELL kernels follow the paper's mapping (one CTA per row); the dense tails reuse gemm_tc.cuh.
#pragma once
#include "ptx.cuh"

namespace sffn {

constexpr int HMM_WARPS = 4;

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ float dot8_bf16(const uint4& a, const uint4& b) {
    float s = bf16_lo(a.x) * bf16_lo(b.x);
    s = fmaf(bf16_hi(a.x), bf16_hi(b.x), s);
    s = fmaf(bf16_lo(a.y), bf16_lo(b.y), s);
    s = fmaf(bf16_hi(a.y), bf16_hi(b.y), s);
    s = fmaf(bf16_lo(a.z), bf16_lo(b.z), s);
    s = fmaf(bf16_hi(a.z), bf16_hi(b.z), s);
    s = fmaf(bf16_lo(a.w), bf16_lo(b.w), s);
    return fmaf(bf16_hi(a.w), bf16_hi(b.w), s);
}
__device__ __forceinline__ uint16_t f32_to_bf16_bits(float f) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// SDDMM, ELL rows (row_loc == -1): one CTA per row, warps over the row's entries, lanes over K in 16-byte chunks
// (A row and the entry's B row both 128-bit loads), fp32 FMA, warp shuffle reduction (Listing 5);
// out = bf16(g * dot), g = the pattern value (gate) or 1.
__global__ void __launch_bounds__(HMM_WARPS * 32)
    hybrid_sddmm_ell_kernel(const uint4* __restrict__ A, const uint4* __restrict__ B, int K8, int ell_w,
                            const int16_t* __restrict__ ell_col, const int32_t* __restrict__ row_nnz,
                            const int32_t* __restrict__ row_loc, const uint16_t* __restrict__ P_ell, int gate,
                            uint16_t* __restrict__ out_ell) {
    const int64_t m = blockIdx.x;
    if (__ldg(row_loc + m) != -1) return;
    const int z = min(__ldg(row_nnz + m), ell_w);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint4* a = A + m * K8;
    for (int j = warp; j < z; j += HMM_WARPS) {
        const int64_t n = static_cast<uint16_t>(__ldg(ell_col + m * ell_w + j));
        const uint4* b = B + n * K8;
        float acc = 0.f;
#pragma unroll 4
        for (int c = lane; c < K8; c += 32) acc += dot8_bf16(__ldg(a + c), __ldg(b + c));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) {
            const float g = gate ? __uint_as_float(static_cast<uint32_t>(__ldg(P_ell + m * ell_w + j)) << 16) : 1.f;
            out_ell[m * ell_w + j] = f32_to_bf16_bits(g * acc);
        }
    }
}

// SDDMM dense tail: out[s, n] = P[s, n] != 0 ? bf16(g * S[s, n]) : 0 for s < min(*count, D) (S = the fp32 GEMM of
// the gathered A rows with B), g = P (gate) or 1 — the mask of Alg.3's dense portion.
__global__ void hybrid_tail_mask_kernel(const float* __restrict__ S, const uint16_t* __restrict__ P, int64_t N,
                                        const int* __restrict__ count, int D, int gate, uint16_t* __restrict__ out) {
    const int64_t rows = min(D, __ldg(count));
    const int64_t tot = rows * N;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < tot;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t p = __ldg(P + i);
        const float pf = __uint_as_float(p << 16);
        out[i] = pf != 0.f ? f32_to_bf16_bits((gate ? pf : 1.f) * __ldg(S + i)) : uint16_t(0);
    }
}

// SpMM, ELL rows: one CTA per row; each thread owns HMM_CH 8-column chunks of the output row in fp32 registers and
// sweeps the row's entries once, loading 16 bytes of W[col, :] per chunk (Listing 6); bf16 16-byte stores.
// Rows with row_loc == -2 (dropped) are written as zeros; dense-tail rows are left to the tail GEMM.
constexpr int HMM_CH = 4;
__global__ void __launch_bounds__(128)
    hybrid_spmm_ell_kernel(const uint16_t* __restrict__ ell_val, const int16_t* __restrict__ ell_col,
                           const int32_t* __restrict__ row_nnz, const int32_t* __restrict__ row_loc, int ell_w,
                           const uint4* __restrict__ W, int K8, uint4* __restrict__ Y) {
    const int64_t m = blockIdx.x;
    const int loc = __ldg(row_loc + m);
    if (loc >= 0) return;
    uint4* y = Y + m * K8;
    if (loc == -2) {
        for (int c = threadIdx.x; c < K8; c += blockDim.x) y[c] = make_uint4(0, 0, 0, 0);
        return;
    }
    const int z = min(__ldg(row_nnz + m), ell_w);
    for (int c0 = threadIdx.x; c0 < K8; c0 += blockDim.x * HMM_CH) {
        float acc[HMM_CH][8];
#pragma unroll
        for (int q = 0; q < HMM_CH; ++q)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[q][i] = 0.f;
        for (int j = 0; j < z; ++j) {
            const float v = __uint_as_float(static_cast<uint32_t>(__ldg(ell_val + m * ell_w + j)) << 16);
            const int64_t n = static_cast<uint16_t>(__ldg(ell_col + m * ell_w + j));
            const uint4* w = W + n * K8;
#pragma unroll
            for (int q = 0; q < HMM_CH; ++q) {
                const int c = c0 + q * blockDim.x;
                if (c < K8) {
                    const uint4 b = __ldg(w + c);
                    const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        acc[q][2 * i] = fmaf(v, bf16_lo(bw[i]), acc[q][2 * i]);
                        acc[q][2 * i + 1] = fmaf(v, bf16_hi(bw[i]), acc[q][2 * i + 1]);
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < HMM_CH; ++q) {
            const int c = c0 + q * blockDim.x;
            if (c < K8)
                y[c] = make_uint4(pack_bf16x2(acc[q][0], acc[q][1]), pack_bf16x2(acc[q][2], acc[q][3]),
                                  pack_bf16x2(acc[q][4], acc[q][5]), pack_bf16x2(acc[q][6], acc[q][7]));
        }
    }
}

// Training forward through the union tensor-core path (sffn_forward_train): after the union up/down, H_c holds
// h = h_g (.) x W_u (bf16) for every stored (row, unit) at the row's union positions.  Warp per pi position p
// (token row m = perm[p]): the row's compact gate list (ascending units = ascending union positions = the ELL
// order of sffn_twell_to_hybrid) gives the positions; ELL rows: ell_h[m, j] = H_c[p, pos_j] for j < min(nnz, ell_w);
// dense-tail rows (row_loc = s >= 0): dense_h[s, :] = 0, then dense_h[s, unit_j] = H_c[p, pos_j] (unit from the
// block's union list).  Dropped rows (-2) are skipped.
__global__ void union_h_to_hybrid_kernel(const uint16_t* __restrict__ hc, int M, int N, int brows,
                                         const int32_t* __restrict__ perm, const uint32_t* __restrict__ glist,
                                         const uint16_t* __restrict__ coff, int lmax, int nchunk,
                                         const int32_t* __restrict__ ulist, const int32_t* __restrict__ row_nnz,
                                         const int32_t* __restrict__ row_loc, int ell_w, uint16_t* __restrict__ ell_h,
                                         uint16_t* __restrict__ dense_h, const uint32_t* __restrict__ tw, int T, int C,
                                         const int32_t* __restrict__ udense) {
    const int64_t p = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= M) return;
    const int64_t m = __ldg(perm + p);
    const int loc = __ldg(row_loc + m);
    if (loc == -2) return;
    const uint32_t* gl = glist + p * lmax;
    const uint16_t* hrow = hc + p * N;
    if (__ldg(udense + p / brows) != 0) {
        // dense block (identity union, no gate list): walk the row's TwELL tiles in order (lane per tile, warp
        // prefix of the counts = the ELL slot order of sffn_twell_to_hybrid); position = unit
        const int NT = N / T, WPT = T / C, cap = WPT - 1;
        const uint32_t* row = tw + m * (N / C);
        uint16_t* d = loc >= 0 ? dense_h + static_cast<int64_t>(loc) * N : nullptr;
        if (d) {
            for (int c = lane; c < N / 8; c += 32) reinterpret_cast<uint4*>(d)[c] = make_uint4(0, 0, 0, 0);
            __syncwarp();
        }
        int base = 0;
        for (int t0 = 0; t0 < NT; t0 += 32) {
            const int t = t0 + lane;
            const int cnt = t < NT ? min(static_cast<int>(__ldg(row + static_cast<int64_t>(t) * WPT)), cap) : 0;
            int inc = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            const int start = base + inc - cnt;
            for (int e = 0; e < cnt; ++e) {
                const int n = static_cast<int>(__ldg(row + static_cast<int64_t>(t) * WPT + 1 + e) & 0xFFFFu);
                if (d) d[n] = __ldg(hrow + n);
                else if (start + e < ell_w) ell_h[m * ell_w + start + e] = __ldg(hrow + n);
            }
            base += __shfl_sync(0xffffffffu, inc, 31);
        }
        return;
    }
    if (loc == -1) {
        const int z = min(__ldg(row_nnz + m), ell_w);
        for (int j = lane; j < z; j += 32) ell_h[m * ell_w + j] = __ldg(hrow + (__ldg(gl + j) >> 16));
        return;
    }
    uint16_t* d = dense_h + static_cast<int64_t>(loc) * N;
    for (int c = lane; c < N / 8; c += 32) reinterpret_cast<uint4*>(d)[c] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    const int e = __ldg(coff + p * (nchunk + 1) + nchunk);  // stored entries of the row
    const int32_t* ul = ulist + (p / brows) * static_cast<int64_t>(N);
    for (int j = lane; j < e; j += 32) {
        const int pos = static_cast<int>(__ldg(gl + j) >> 16);
        d[__ldg(ul + pos)] = __ldg(hrow + pos);
    }
}

}  // namespace sffn
