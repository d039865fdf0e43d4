// union.cuh — block-union metadata for the tensor-core sparse up/down.
//
// For every block b of 128 consecutive token rows (the tcgen05 M tile), the union U_b of the hidden units
// that are active (stored in the TwELL) for at least one row of the block, in ascending order:
//   ulist [NB, N]      int32  U_b, then padding up to ulen[b] (a multiple of 64, >= 64) with unit 0
//   ulen  [NB]         int32  padded length
//   umask [NB, N/32]   uint32 bit n%32 of word n/32 set iff n in U_b
//   uwoff [NB, N/32]   int32  number of union members in words < w  (position of n in U_b =
//                             uwoff[n/32] + popc(umask[n/32] & ((1 << n%32) - 1)))
//   chunk_off [NB + 1] int32  exclusive prefix of ceil(ulen / 256): the up-GEMM work list
// Deterministic: bit sets are order-independent and the positions come from prefix sums.
#pragma once
#include "ptx.cuh"

namespace sffn {

struct UnionMeta {
    int32_t* ulist;
    int32_t* ulen;
    uint32_t* umask;
    int32_t* uwoff;
    int32_t* chunk_off;
    int32_t* utot;  // [NB] un-padded union sizes
};

constexpr int UB_THREADS = 512;

// One CTA per block of 128 rows.  Dynamic smem: N/32 uint32 masks + N/32 int32 offsets + scan scratch.
__global__ void __launch_bounds__(UB_THREADS) union_build_kernel(const uint32_t* __restrict__ tw, int M, int N, int T,
                                                                  int C, UnionMeta um) {
    extern __shared__ uint32_t ub_smem[];
    const int NW = N >> 5;
    uint32_t* mask = ub_smem;                                  // [NW]
    int32_t* woff = reinterpret_cast<int32_t*>(ub_smem + NW);  // [NW]
    int32_t* wsum = woff + NW;                                 // [UB_THREADS / 32]
    const int b = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = UB_THREADS / 32;
    for (int w = threadIdx.x; w < NW; w += UB_THREADS) mask[w] = 0u;
    __syncthreads();

    // OR the stored indices of the block's rows (warp per (row, tile), coalesced reads of the tile's words)
    const int NT = N / T, WPT = T / C, cap = WPT - 1;
    const int rows = min(128, M - b * 128);
    const int pairs = rows * NT;
    for (int pidx = warp; pidx < pairs; pidx += nwarps) {
        const int r = pidx / NT, t = pidx - r * NT;
        const uint32_t* blk = tw + static_cast<int64_t>(b * 128 + r) * (N / C) + static_cast<int64_t>(t) * WPT;
        const int cnt = min(static_cast<int>(__ldg(blk)), cap);
        for (int e = lane; e < cnt; e += 32) {
            const uint32_t n = __ldg(blk + 1 + e) & 0xFFFFu;
            atomicOr(&mask[n >> 5], 1u << (n & 31));
        }
    }
    __syncthreads();

    // exclusive scan of popc(mask[w]) over w (each thread owns a contiguous segment)
    const int seg = (NW + UB_THREADS - 1) / UB_THREADS;
    const int w0 = threadIdx.x * seg, w1 = min(NW, w0 + seg);
    int local = 0;
    for (int w = w0; w < w1; ++w) local += __popc(mask[w]);
    int incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int v = lane < nwarps ? wsum[lane] : 0;
        int s = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += u;
        }
        if (lane < nwarps) wsum[lane] = s - v;  // exclusive warp offsets
        if (lane == nwarps - 1) wsum[nwarps] = s;  // total
    }
    __syncthreads();
    int run = wsum[warp] + incl - local;
    for (int w = w0; w < w1; ++w) {
        woff[w] = run;
        run += __popc(mask[w]);
    }
    __syncthreads();
    const int total = wsum[nwarps];
    const int padded = max(64, (total + 63) & ~63);

    int32_t* ul = um.ulist + static_cast<int64_t>(b) * N;
    for (int w = threadIdx.x; w < NW; w += UB_THREADS) {
        uint32_t m = mask[w];
        int pos = woff[w];
        um.umask[static_cast<int64_t>(b) * NW + w] = m;
        um.uwoff[static_cast<int64_t>(b) * NW + w] = pos;
        while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            ul[pos++] = (w << 5) + bit;
        }
    }
    for (int j = total + threadIdx.x; j < padded; j += UB_THREADS) ul[j] = 0;
    if (threadIdx.x == 0) {
        um.ulen[b] = padded;
        um.utot[b] = total;
    }
}

// chunk_off[b] = sum_{b' < b} ceil(ulen[b'] / 256);  chunk_off[NB] = total.  One CTA.
__global__ void __launch_bounds__(1024) union_scan_kernel(UnionMeta um, int NB) {
    __shared__ int wsum[33];
    __shared__ int carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < NB; base += 1024) {
        const int i = base + threadIdx.x;
        const int v = i < NB ? (um.ulen[i] + 255) / 256 : 0;
        int s = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += u;
        }
        if (lane == 31) wsum[warp] = s;
        __syncthreads();
        if (warp == 0) {
            int x = wsum[lane];
            int y = x;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, y, off);
                if (lane >= off) y += u;
            }
            wsum[lane] = y - x;
            if (lane == 31) wsum[32] = y;
        }
        __syncthreads();
        if (i < NB) um.chunk_off[i] = carry + wsum[warp] + s - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += wsum[32];
        __syncthreads();
    }
    if (threadIdx.x == 0) um.chunk_off[NB] = carry;
}

}  // namespace sffn
