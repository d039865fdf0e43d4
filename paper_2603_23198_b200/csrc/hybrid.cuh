// hybrid.cuh — overflow-exact inference: the paper's hybrid format idea (rows
// routed to a compact sparse representation or to a dense backup; backup rows sized "one-eighth of the token
// batch") applied to inference.  Rows whose TwELL has any overflowed tile (count > T/C - 1,
// reading R5) are collected, recomputed with the dense tcgen05 FFN (all positives, exact), and written over
// the sparse result.  No host synchronization: the backup row count lives on the device and the dense GEMMs
// read it (GemmArgs::m_dev).
#pragma once
#include "ptx.cuh"

namespace sffn {

// rows with an overflowed tile -> list[atomic slot] (capacity R); *count = total such rows (may exceed R)
__global__ void ov_rows_kernel(const uint32_t* __restrict__ tw, int M, int N, int T, int C, int* __restrict__ count,
                               int32_t* __restrict__ list, int R) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= M) return;
    const int NT = N / T, WPT = T / C, cap = WPT - 1;
    const uint32_t* row = tw + gw * (N / C);
    bool ov = false;
    for (int t = lane; t < NT; t += 32) ov |= static_cast<int>(__ldg(row + static_cast<int64_t>(t) * WPT)) > cap;
    if (__any_sync(0xffffffffu, ov) && lane == 0) {
        const int slot = atomicAdd(count, 1);
        if (slot < R) list[slot] = static_cast<int32_t>(gw);
    }
}

// dst[i, :] = src[list[i], :] (gather) or dst[list[i], :] = src[i, :] (scatter), i < min(*count, R); warp per row
template <bool GATHER>
__global__ void move_rows_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, const int32_t* __restrict__ list,
                                 const int* __restrict__ count, int R, int K8) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= min(R, __ldg(count))) return;
    const int64_t r = __ldg(list + gw);
    const uint4* s = src + (GATHER ? r : gw) * K8;
    uint4* d = dst + (GATHER ? gw : r) * K8;
    for (int c = lane; c < K8; c += 32) d[c] = __ldg(s + c);
}

}  // namespace sffn

namespace sffn {

// TwELL -> hybrid format (the training entry; Listing 4, hybrid format P:177-182).
// Warp per row; lane t handles TwELL tiles t, t+32, ...; an exclusive warp prefix scan of the stored counts
// gives each tile's offset in the row's ELL storage (ascending columns).  Rows whose stored count exceeds
// ELL_W keep their true count in row_nnz, are routed to the dense tail (slot by atomic, capacity D; the
// row is densified there) and row_loc[m] = slot; otherwise row_loc[m] = -1 (the paper's h_b).
// L0 / L1 statistics (Listing 4): sum over rows of nnz / M and of sum(values) / M, one double atomic per warp.
__global__ void twell_to_hybrid_kernel(const uint32_t* __restrict__ tw, int M, int N, int T, int C, int ell_w,
                                       uint16_t* __restrict__ ell_val, int16_t* __restrict__ ell_col,
                                       int32_t* __restrict__ row_nnz, int32_t* __restrict__ row_loc, int D,
                                       uint16_t* __restrict__ dense_rows, int32_t* __restrict__ dense_map,
                                       int* __restrict__ dense_count, double* __restrict__ l0l1) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= M) return;
    const int NT = N / T, WPT = T / C, cap = WPT - 1;
    const uint32_t* row = tw + gw * (N / C);
    // pass 1: total stored count and value sum
    int total = 0;
    float vsum = 0.0f;
    for (int t = lane; t < NT; t += 32) {
        const uint32_t* blk = row + static_cast<int64_t>(t) * WPT;
        const int cnt = min(static_cast<int>(__ldg(blk)), cap);
        total += cnt;
        for (int e = 0; e < cnt; ++e) vsum += __uint_as_float(__ldg(blk + 1 + e) & 0xFFFF0000u);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        total += __shfl_xor_sync(0xffffffffu, total, off);
        vsum += __shfl_xor_sync(0xffffffffu, vsum, off);
    }
    int slot = -1;
    if (lane == 0) {
        row_nnz[gw] = total;
        if (total > ell_w) {
            const int s = atomicAdd(dense_count, 1);
            slot = s < D ? s : -2;  // -2: dense tail full (row keeps only its first ELL_W entries)
            if (s < D) dense_map[s] = static_cast<int32_t>(gw);
        }
        row_loc[gw] = slot;
        if (l0l1) {
            atomicAdd(l0l1, static_cast<double>(total) / M);
            atomicAdd(l0l1 + 1, static_cast<double>(vsum) / M);
        }
    }
    slot = __shfl_sync(0xffffffffu, slot, 0);
    // pass 2: ELL compaction in 32-tile rounds (exclusive scan of the stored counts across lanes)
    int base = 0;
    for (int t0 = 0; t0 < NT; t0 += 32) {
        const int t = t0 + lane;
        const uint32_t* blk = row + static_cast<int64_t>(t) * WPT;
        const int cnt = t < NT ? min(static_cast<int>(__ldg(blk)), cap) : 0;
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += v;
        }
        const int start = base + incl - cnt;
        for (int e = 0; e < cnt && start + e < ell_w; ++e) {
            const uint32_t w = __ldg(blk + 1 + e);
            ell_val[gw * ell_w + start + e] = static_cast<uint16_t>(w >> 16);
            ell_col[gw * ell_w + start + e] = static_cast<int16_t>(w & 0xFFFFu);
        }
        base += __shfl_sync(0xffffffffu, incl, 31);
    }
    // dense tail: densify the row
    if (slot >= 0) {
        uint16_t* drow = dense_rows + static_cast<int64_t>(slot) * N;
        for (int n = lane; n < N; n += 32) drow[n] = 0;
        __syncwarp();
        for (int t = lane; t < NT; t += 32) {
            const uint32_t* blk = row + static_cast<int64_t>(t) * WPT;
            const int cnt = min(static_cast<int>(__ldg(blk)), cap);
            for (int e = 0; e < cnt; ++e) {
                const uint32_t w = __ldg(blk + 1 + e);
                drow[w & 0xFFFFu] = static_cast<uint16_t>(w >> 16);
            }
        }
    }
}

}  // namespace sffn
