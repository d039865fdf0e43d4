// updown.cuh — fused sparse up/down projection from packed TwELL (Alg.2, Eq.3).
//
// One CTA of 4 warps per token row m (the paper uses one warp per row, L2 P:881-887; at K = 4096 a
// single warp would need ~190 registers for x and y, so the K dimension is split across 4 warps).
// Warp w owns the 16-byte chunks [w*32*NCH, (w+1)*32*NCH) of the K dimension; lane l holds chunks
// w*32*NCH + j*32 + l, j < NCH (coalesced 512-B warp accesses).  Per TwELL tile (P:1078 packed
// words, one 128-B coalesced read at T/C = 32):
//   up   : each warp computes its partial dot x_m[slice] . W_u[n, slice] for the tile's entries
//          (4 entries in flight per lane: 4*NCH independent 16-B gathers), warp-reduces them with
//          shuffles and parks them in shared memory; one barrier per batch of <= 32 entries;
//   gate : u = sum of the 4 partials in fixed warp order (deterministic), h = h_v * u (h_v = the
//          stored bf16 gate value, reading R10);
//   down : y[slice] += h * W_d[n, slice] with fp32 FMA (the paper rounds products to bf16,
//          L2 P:1016-1019; we keep fp32 products, reading R9).
// Output: bf16 round-to-nearest, 16-B vector stores (L2 P:1055-1073).
#pragma once
#include "ptx.cuh"

namespace sffn {

constexpr int UD_WARPS = 4;

__device__ __forceinline__ void bf16x8_to_f32(const uint4 q, float* f) {
    f[0] = __uint_as_float(q.x << 16);
    f[1] = __uint_as_float(q.x & 0xFFFF0000u);
    f[2] = __uint_as_float(q.y << 16);
    f[3] = __uint_as_float(q.y & 0xFFFF0000u);
    f[4] = __uint_as_float(q.z << 16);
    f[5] = __uint_as_float(q.z & 0xFFFF0000u);
    f[6] = __uint_as_float(q.w << 16);
    f[7] = __uint_as_float(q.w & 0xFFFF0000u);
}

__device__ __forceinline__ uint4 ldg_nc(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int NCH>
__global__ void __launch_bounds__(UD_WARPS * 32)
    updown_kernel(const uint4* __restrict__ X, const uint32_t* __restrict__ tw, const uint4* __restrict__ Wu,
                  const uint4* __restrict__ Wd, uint4* __restrict__ Y, int M, int K, int N, int T, int C) {
    constexpr int EB = 4;  // entries in flight per lane
    __shared__ float part[2][UD_WARPS][32];

    const int m = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int K8 = K >> 3;
    int cidx[NCH];
    bool cok[NCH];
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
        cidx[j] = warp * 32 * NCH + j * 32 + lane;
        cok[j] = cidx[j] < K8;
    }

    float x[NCH * 8], y[NCH * 8];
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
        const uint4 q = cok[j] ? X[static_cast<int64_t>(m) * K8 + cidx[j]] : make_uint4(0, 0, 0, 0);
        bf16x8_to_f32(q, &x[j * 8]);
#pragma unroll
        for (int i = 0; i < 8; ++i) y[j * 8 + i] = 0.0f;
    }

    const int WPT = T / C, cap = WPT - 1, NT = N / T;
    const uint32_t* trow = tw + static_cast<int64_t>(m) * (N / C);
    int buf = 0;
#pragma unroll 1
    for (int t = 0; t < NT; ++t) {
        const uint32_t* blk = trow + t * WPT;
        const int cnt = min(static_cast<int>(__ldg(blk)), cap);
#pragma unroll 1
        for (int e0 = 0; e0 < cnt; e0 += 32) {
            const int ne = min(32, cnt - e0);
            const uint32_t myw = lane < ne ? __ldg(blk + 1 + e0 + lane) : 0u;
            // ---- up: partial dots over this warp's K slice
#pragma unroll 1
            for (int e = 0; e < ne; e += EB) {
                uint4 q[EB][NCH];
#pragma unroll
                for (int i = 0; i < EB; ++i) {
                    const int ee = min(e + i, ne - 1);
                    const uint32_t n = __shfl_sync(0xffffffffu, myw, ee) & 0xFFFFu;
                    const uint4* wr = Wu + static_cast<int64_t>(n) * K8;
#pragma unroll
                    for (int j = 0; j < NCH; ++j) q[i][j] = cok[j] ? ldg_nc(wr + cidx[j]) : make_uint4(0, 0, 0, 0);
                }
                float a[EB];
#pragma unroll
                for (int i = 0; i < EB; ++i) {
                    float s = 0.0f;
#pragma unroll
                    for (int j = 0; j < NCH; ++j) {
                        float w[8];
                        bf16x8_to_f32(q[i][j], w);
#pragma unroll
                        for (int k = 0; k < 8; ++k) s = fmaf(x[j * 8 + k], w[k], s);
                    }
                    a[i] = s;
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                    for (int i = 0; i < EB; ++i) a[i] += __shfl_xor_sync(0xffffffffu, a[i], off);
                if (lane == 0) {
#pragma unroll
                    for (int i = 0; i < EB; ++i)
                        if (e + i < ne) part[buf][warp][e + i] = a[i];
                }
            }
            __syncthreads();
            // ---- gate scaling + down axpy
#pragma unroll 1
            for (int e = 0; e < ne; e += EB) {
                uint4 q[EB][NCH];
                float h[EB];
#pragma unroll
                for (int i = 0; i < EB; ++i) {
                    const int ee = min(e + i, ne - 1);
                    const uint32_t w = __shfl_sync(0xffffffffu, myw, ee);
                    const uint32_t n = w & 0xFFFFu;
                    float u = part[buf][0][ee];
#pragma unroll
                    for (int ww = 1; ww < UD_WARPS; ++ww) u += part[buf][ww][ee];
                    h[i] = (e + i < ne) ? __uint_as_float(w & 0xFFFF0000u) * u : 0.0f;
                    const uint4* wr = Wd + static_cast<int64_t>(n) * K8;
#pragma unroll
                    for (int j = 0; j < NCH; ++j) q[i][j] = cok[j] ? ldg_nc(wr + cidx[j]) : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int i = 0; i < EB; ++i) {
#pragma unroll
                    for (int j = 0; j < NCH; ++j) {
                        float w[8];
                        bf16x8_to_f32(q[i][j], w);
#pragma unroll
                        for (int k = 0; k < 8; ++k) y[j * 8 + k] = fmaf(h[i], w[k], y[j * 8 + k]);
                    }
                }
            }
            buf ^= 1;
        }
    }
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
        if (cok[j]) {
            uint4 o;
            o.x = pack_bf16x2(y[j * 8 + 0], y[j * 8 + 1]);
            o.y = pack_bf16x2(y[j * 8 + 2], y[j * 8 + 3]);
            o.z = pack_bf16x2(y[j * 8 + 4], y[j * 8 + 5]);
            o.w = pack_bf16x2(y[j * 8 + 6], y[j * 8 + 7]);
            Y[static_cast<int64_t>(m) * K8 + cidx[j]] = o;
        }
    }
}

// TwELL -> dense bf16 (verification).  One warp per (row, tile).
__global__ void unpack_kernel(const uint32_t* __restrict__ tw, int M, int N, int T, int C, int64_t col_offset,
                              int64_t ld, __nv_bfloat16* __restrict__ out) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int NT = N / T;
    if (gw >= static_cast<int64_t>(M) * NT) return;
    const int m = static_cast<int>(gw / NT), t = static_cast<int>(gw % NT);
    const int WPT = T / C, cap = WPT - 1;
    __nv_bfloat16* orow = out + static_cast<int64_t>(m) * ld + col_offset;
    for (int c = lane; c < T; c += 32) orow[t * T + c] = __ushort_as_bfloat16(0);
    __syncwarp();
    const uint32_t* blk = tw + static_cast<int64_t>(m) * (N / C) + t * WPT;
    const int cnt = min(static_cast<int>(blk[0]), cap);
    for (int e = lane; e < cnt; e += 32) {
        const uint32_t w = blk[1 + e];
        orow[w & 0xFFFFu] = __ushort_as_bfloat16(static_cast<unsigned short>(w >> 16));
    }
}

// out[c, r] = in[r, c], bf16, 32x32 tiles through shared memory.
__global__ void transpose_bf16_kernel(const __nv_bfloat16* __restrict__ in, int64_t rows, int64_t cols,
                                      __nv_bfloat16* __restrict__ out) {
    __shared__ __nv_bfloat16 tile[32][34];
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][i];
    }
}

}  // namespace sffn

namespace sffn {

// Non-gated down projection from TwELL (App.C eq. P:1751-1756, y = h W_d with h = relu(x W_u) stored in
// TwELL; the paper's Listing 3).  One CTA of 4 warps per row; warp w owns a contiguous K
// slice of the output (the paper's SPLIT_OUT_DIM idea) and walks every stored entry
// independently — no cross-warp reduction: y[slice] += h_v * W_d[n, slice] in fp32 FMA.
template <int NCH>
__global__ void __launch_bounds__(UD_WARPS * 32)
    down_kernel(const uint32_t* __restrict__ tw, const uint4* __restrict__ Wd, uint4* __restrict__ Y, int M, int K,
                int N, int T, int C) {
    constexpr int EB = 4;
    const int m = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int K8 = K >> 3;
    int cidx[NCH];
    bool cok[NCH];
    float y[NCH * 8];
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
        cidx[j] = warp * 32 * NCH + j * 32 + lane;
        cok[j] = cidx[j] < K8;
#pragma unroll
        for (int i = 0; i < 8; ++i) y[j * 8 + i] = 0.0f;
    }
    const int WPT = T / C, cap = WPT - 1, NT = N / T;
    const uint32_t* trow = tw + static_cast<int64_t>(m) * (N / C);
#pragma unroll 1
    for (int t = 0; t < NT; ++t) {
        const uint32_t* blk = trow + t * WPT;
        const int cnt = min(static_cast<int>(__ldg(blk)), cap);
#pragma unroll 1
        for (int e0 = 0; e0 < cnt; e0 += 32) {
            const int ne = min(32, cnt - e0);
            const uint32_t myw = lane < ne ? __ldg(blk + 1 + e0 + lane) : 0u;
#pragma unroll 1
            for (int e = 0; e < ne; e += EB) {
                uint4 q[EB][NCH];
                float h[EB];
#pragma unroll
                for (int i = 0; i < EB; ++i) {
                    const int ee = min(e + i, ne - 1);
                    const uint32_t w = __shfl_sync(0xffffffffu, myw, ee);
                    h[i] = (e + i < ne) ? __uint_as_float(w & 0xFFFF0000u) : 0.0f;
                    const uint4* wr = Wd + static_cast<int64_t>(w & 0xFFFFu) * K8;
#pragma unroll
                    for (int j = 0; j < NCH; ++j) q[i][j] = cok[j] ? ldg_nc(wr + cidx[j]) : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int i = 0; i < EB; ++i)
#pragma unroll
                    for (int j = 0; j < NCH; ++j) {
                        float w[8];
                        bf16x8_to_f32(q[i][j], w);
#pragma unroll
                        for (int k = 0; k < 8; ++k) y[j * 8 + k] = fmaf(h[i], w[k], y[j * 8 + k]);
                    }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
        if (cok[j]) {
            uint4 o;
            o.x = pack_bf16x2(y[j * 8 + 0], y[j * 8 + 1]);
            o.y = pack_bf16x2(y[j * 8 + 2], y[j * 8 + 3]);
            o.z = pack_bf16x2(y[j * 8 + 4], y[j * 8 + 5]);
            o.w = pack_bf16x2(y[j * 8 + 6], y[j * 8 + 7]);
            Y[static_cast<int64_t>(m) * K8 + cidx[j]] = o;
        }
    }
}

}  // namespace sffn
