// fp32_path.cuh — the fp32 correctness mode (reading R19): fp32 inputs, fp32 accumulation,
// logical (SoA) TwELL of Alg.1's outputs:
//   h_v  float    [M, N/C]   values              (capacity T/C per tile: no count word in the slots)
//   h_I  uint16   [M, N/C]   global column index (shard-local)
//   h_nz uint32   [M, N/T]   true count per (row, tile)
// The gate GEMM cannot use tcgen05 kind::tf32 (10-bit mantissa, ~1e-3 error against a 1e-5 bar), so it
// is a register-blocked SIMT fp32 GEMM; its epilogue compacts each row-tile with warp ballot / popc.
#pragma once
#include "ptx.cuh"

namespace sffn {

constexpr int F32_BM = 64, F32_BN = 256, F32_BK = 16;

// One CTA (256 threads) per 64 x 256 output tile; thread (ty, tx) owns rows 8 ty .. 8 ty + 7 and columns
// tx + 32 j, j < 8 (conflict-free shared-memory reads).  Then warp w compacts rows 8 w .. 8 w + 7.
__global__ void __launch_bounds__(256) pack_f32_kernel(const float* __restrict__ X, const float* __restrict__ Wg, int M,
                                                       int K, int N, int T, int C, float* __restrict__ hv,
                                                       uint16_t* __restrict__ hi, uint32_t* __restrict__ hnz,
                                                       uint32_t* overflow) {
    __shared__ float As[F32_BK][F32_BM + 4];
    __shared__ float Bs[F32_BK][F32_BN + 4];
    extern __shared__ float Cs[];  // [F32_BM][F32_BN + 1]
    const int tid = threadIdx.x, ty = tid >> 5, tx = tid & 31;
    const int m0 = blockIdx.y * F32_BM, n0 = blockIdx.x * F32_BN;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
    for (int k0 = 0; k0 < K; k0 += F32_BK) {
        // A: 64 rows x 16 k -> As[k][r]; B: 256 rows x 16 k -> Bs[k][c]
        for (int i = tid; i < F32_BM * F32_BK; i += 256) {
            const int r = i / F32_BK, k = i % F32_BK;
            As[k][r] = (m0 + r < M && k0 + k < K) ? X[static_cast<int64_t>(m0 + r) * K + k0 + k] : 0.0f;
        }
        for (int i = tid; i < F32_BN * F32_BK; i += 256) {
            const int c = i / F32_BK, k = i % F32_BK;
            Bs[k][c] = (n0 + c < N && k0 + k < K) ? Wg[static_cast<int64_t>(n0 + c) * K + k0 + k] : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < F32_BK; ++k) {
            float a[8], b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = As[k][8 * ty + i];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = Bs[k][tx + 32 * j];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) Cs[(8 * ty + i) * (F32_BN + 1) + tx + 32 * j] = acc[i][j];
    __syncthreads();

    // Alg.1 lines 7-17 per row: warp ballot over 32 columns, slot = running count + popc(mask & lanes below)
    const int W = T / C, cap = W, NT = N / T, lane = tx;
    const uint32_t below = (1u << lane) - 1u;
    for (int rr = 0; rr < 8; ++rr) {
        const int r = 8 * ty + rr, m = m0 + r;
        if (m >= M) break;
        for (int tl = 0; tl < F32_BN / T; ++tl) {
            const int t = n0 / T + tl;
            if (t >= NT) break;
            int z = 0;
            for (int c0 = tl * T; c0 < (tl + 1) * T; c0 += 32) {
                const float v = Cs[r * (F32_BN + 1) + c0 + lane];
                const bool pos = v > 0.0f;  // strict (R1)
                const uint32_t mask = __ballot_sync(0xffffffffu, pos);
                const int slot = z + __popc(mask & below);
                if (pos && slot < cap) {
                    const int64_t o = static_cast<int64_t>(m) * (N / C) + static_cast<int64_t>(t) * W + slot;
                    hv[o] = v;
                    hi[o] = static_cast<uint16_t>(n0 + c0 + lane);
                }
                z += __popc(mask);
            }
            if (lane == 0) {
                hnz[static_cast<int64_t>(m) * NT + t] = static_cast<uint32_t>(z);
                if (z > cap && overflow) atomicAdd(overflow, 1u);
            }
        }
    }
}

// Eq.3 in fp32 from the SoA TwELL: one CTA of 4 warps per row; warp w owns float4 chunks
// [w 32 NCH, (w+1) 32 NCH) of K; x and y stay in registers; per tile, partial dots -> warp reduce ->
// SMEM -> fixed-order sum; axpy with W_d.
template <int NCH>
__global__ void __launch_bounds__(128) updown_f32_kernel(const float4* __restrict__ X, const float* __restrict__ hv,
                                                         const uint16_t* __restrict__ hi,
                                                         const uint32_t* __restrict__ hnz, const float4* __restrict__ Wu,
                                                         const float4* __restrict__ Wd, float4* __restrict__ Y, int M,
                                                         int K, int N, int T, int C) {
    __shared__ float part[2][4][32];
    const int m = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int K4 = K >> 2;
    int ci[NCH];
    bool ok[NCH];
    float4 x[NCH], y[NCH];
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
        ci[j] = warp * 32 * NCH + j * 32 + lane;
        ok[j] = ci[j] < K4;
        x[j] = ok[j] ? X[static_cast<int64_t>(m) * K4 + ci[j]] : make_float4(0, 0, 0, 0);
        y[j] = make_float4(0, 0, 0, 0);
    }
    const int W = T / C, NT = N / T;
    int buf = 0;
    for (int t = 0; t < NT; ++t) {
        const int cnt = min(static_cast<int>(hnz[static_cast<int64_t>(m) * NT + t]), W);
        const int64_t base = static_cast<int64_t>(m) * (N / C) + static_cast<int64_t>(t) * W;
        for (int e0 = 0; e0 < cnt; e0 += 32) {
            const int ne = min(32, cnt - e0);
            for (int e = 0; e < ne; ++e) {
                const int n = hi[base + e0 + e];
                const float4* wr = Wu + static_cast<int64_t>(n) * K4;
                float s = 0.0f;
#pragma unroll
                for (int j = 0; j < NCH; ++j)
                    if (ok[j]) {
                        const float4 w = wr[ci[j]];
                        s = fmaf(x[j].x, w.x, s);
                        s = fmaf(x[j].y, w.y, s);
                        s = fmaf(x[j].z, w.z, s);
                        s = fmaf(x[j].w, w.w, s);
                    }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                if (lane == 0) part[buf][warp][e] = s;
            }
            __syncthreads();
            for (int e = 0; e < ne; ++e) {
                const float u = part[buf][0][e] + part[buf][1][e] + part[buf][2][e] + part[buf][3][e];
                const float h = hv[base + e0 + e] * u;
                const int n = hi[base + e0 + e];
                const float4* wr = Wd + static_cast<int64_t>(n) * K4;
#pragma unroll
                for (int j = 0; j < NCH; ++j)
                    if (ok[j]) {
                        const float4 w = wr[ci[j]];
                        y[j].x = fmaf(h, w.x, y[j].x);
                        y[j].y = fmaf(h, w.y, y[j].y);
                        y[j].z = fmaf(h, w.z, y[j].z);
                        y[j].w = fmaf(h, w.w, y[j].w);
                    }
            }
            buf ^= 1;
        }
    }
#pragma unroll
    for (int j = 0; j < NCH; ++j)
        if (ok[j]) Y[static_cast<int64_t>(m) * K4 + ci[j]] = y[j];
}

}  // namespace sffn
