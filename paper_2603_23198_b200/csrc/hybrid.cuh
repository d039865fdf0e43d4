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
