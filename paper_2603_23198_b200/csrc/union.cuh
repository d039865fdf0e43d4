// union.cuh — block-union metadata for the tensor-core sparse up/down.
//
// For every block b of 128 consecutive token rows (the tcgen05 M tile), the union U_b of the hidden units
// that are active (stored in the TwELL) for at least one row of the block, in ascending order:
//   ulist [NB, N]      int32  U_b, then padding up to ulen[b] (a multiple of 64, >= 64) with unit 0
//   ulen  [NB]         int32  padded length
//   umask [NB, N/32]   uint32 bit n%32 of word n/32 set iff n in U_b
//   uwoff [NB, N/32]   int32  number of union members in words < w  (position of n in U_b =
//                             uwoff[n/32] + popc(umask[n/32] & ((1 << n%32) - 1)))
//   tiles     [..]     int32  up-GEMM work list (b << 8 | chunk c), ordered group of 16 blocks -> c -> b
//                             so concurrently running tiles share X rows and neighbouring W_u rows
// Deterministic: bit sets are order-independent and the positions come from prefix sums.
#pragma once
#include "ptx.cuh"

namespace sffn {

struct UnionMeta {
    int32_t* ulist;
    int32_t* ulen;
    uint32_t* umask;
    int32_t* uwoff;
    int32_t* chunk_off;  // [1]: number of UP tiles
    int32_t* utot;       // [NB] un-padded union sizes
    int32_t* tiles;      // [NB * ceil(N/256)]: UP work list, (b << 8) | chunk, grouped raster
    int* counters;       // [2] dynamic tile-scheduler counters of the UP and DOWN GEMMs
    uint32_t* glist;     // [NB*128, lmax] per (pi-ordered) row: (union position << 16) | bf16 gate, ascending
    uint16_t* coff;      // [NB*128, nchunk + 1] per row: entries before union chunk c (256 positions per chunk)
    int lmax, nchunk;
};

constexpr int UNION_GROUP_UP = 8;    // token blocks whose up-GEMM tiles run together (L2 working set)
constexpr int UNION_GROUP_DOWN = 16;  // token blocks whose down-GEMM tiles run together

constexpr int UB_THREADS = 512;

// Visit every stored entry (n, word) of one packed TwELL row: warp-cooperative, lane-ordered.
// Fast path (4 <= T/C <= 32): 16-byte loads, each warp instruction covers 128 words; a lane's 4 words lie in
// one tile whose count word sits in the lane holding the tile's first word (shuffle).  Generic path otherwise.
template <class F>
__device__ __forceinline__ void for_each_row_entry(const uint32_t* __restrict__ row, int RW, int NT, int WPT, int cap,
                                                   int lane, F&& f) {
    if (WPT >= 4 && WPT <= 32) {
        const uint4* r4 = reinterpret_cast<const uint4*>(row);
        const int RW4 = RW >> 2;
        for (int g0 = 0; g0 < RW4; g0 += 64) {
            uint4 v[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) v[u] = (g0 + 32 * u + lane < RW4) ? __ldg(r4 + g0 + 32 * u + lane) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int w0 = 4 * (g0 + 32 * u + lane);  // first word of this lane
                const int s0 = w0 % WPT;                 // slot of v.x
                const int src = lane - (s0 >> 2);
                const int cnt = min(static_cast<int>(__shfl_sync(0xffffffffu, v[u].x, src)), cap);
                if (w0 < RW) {
                    const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int sl = s0 + q;
                        if (sl >= 1 && sl <= cnt) f(w[q]);
                    }
                }
            }
        }
    } else {
        for (int t = 0; t < NT; ++t) {
            const uint32_t* blk = row + static_cast<int64_t>(t) * WPT;
            const int cnt = min(static_cast<int>(__ldg(blk)), cap);
            for (int e = lane; e < cnt; e += 32) f(__ldg(blk + 1 + e));
        }
    }
}

// One CTA per block of 128 rows.  Dynamic smem: N/32 uint32 masks + N/32 int32 offsets + scan scratch.
__global__ void __launch_bounds__(UB_THREADS) union_build_kernel(const uint32_t* __restrict__ tw, int M, int N, int T,
                                                                  int C, UnionMeta um, const int32_t* __restrict__ perm) {
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

    // OR the stored indices of the block's rows.  Warp per row, lanes over consecutive words (coalesced);
    // when a tile's words fit a 32-word group (T/C <= 32) the count is taken from the owning lane by shuffle.
    const int NT = N / T, WPT = T / C, cap = WPT - 1, RW = N / C;
    const int rows = min(128, M - b * 128);
    for (int r = warp; r < rows; r += nwarps) {
        const uint32_t* row = tw + static_cast<int64_t>(__ldg(perm + b * 128 + r)) * RW;
        for_each_row_entry(row, RW, NT, WPT, cap, lane, [&](uint32_t w) {
            const uint32_t n = w & 0xFFFFu;
            atomicOr(&mask[n >> 5], 1u << (n & 31));
        });
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

// G_b: the stored gate values in union coordinates, H_c[b*128 + r, j] (bf16), zero elsewhere; the up-GEMM
// epilogue multiplies this tile in place by X_b W_u[U_b]^T.  One CTA (256 threads) per 8 rows of a block.
constexpr int GS_ROWS = 8;
__global__ void __launch_bounds__(256) union_gate_scatter_kernel(const uint32_t* __restrict__ tw, int M, int N, int T,
                                                                 int C, UnionMeta um, uint16_t* __restrict__ hc,
                                                                 const int32_t* __restrict__ perm) {
    const int b = blockIdx.x / (128 / GS_ROWS);
    const int r0 = (blockIdx.x % (128 / GS_ROWS)) * GS_ROWS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp w handles row r0 + w
    const int NW = N >> 5, NT = N / T, WPT = T / C, cap = WPT - 1, RW = N / C;
    const int padded = __ldg(um.ulen + b);
    const uint32_t* msk = um.umask + static_cast<int64_t>(b) * NW;
    const int32_t* wof = um.uwoff + static_cast<int64_t>(b) * NW;
    const int r = r0 + warp;
    uint16_t* hrow = hc + (static_cast<int64_t>(b) * 128 + r) * N;
    for (int c = lane; c < padded / 8; c += 32) *reinterpret_cast<uint4*>(hrow + 8 * c) = make_uint4(0, 0, 0, 0);
    __syncwarp();
    if (b * 128 + r >= M) return;
    const uint32_t* row = tw + static_cast<int64_t>(__ldg(perm + b * 128 + r)) * RW;
    for_each_row_entry(row, RW, NT, WPT, cap, lane, [&](uint32_t w) {
        const int n = static_cast<int>(w & 0xFFFFu);
        const int j = __ldg(wof + (n >> 5)) + __popc(__ldg(msk + (n >> 5)) & ((1u << (n & 31)) - 1u));
        hrow[j] = static_cast<uint16_t>(w >> 16);
    });
}

// Compact gate lists for the UP epilogue (instead of materialising G in H_c): warp per pi-ordered row i;
// the row's stored entries in ascending neuron order = ascending union position; warp ballot/popc
// compaction; then coff[i][c] = #entries with position < 256 c (lower bounds, lanes over chunks).
__global__ void union_gate_list_kernel(const uint32_t* __restrict__ tw, int M, int N, int T, int C, UnionMeta um,
                                       const int32_t* __restrict__ perm) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int NB = (M + 127) / 128;
    if (i >= static_cast<int64_t>(NB) * 128) return;
    const int b = static_cast<int>(i >> 7);
    const int NW = N >> 5, NT = N / T, WPT = T / C, cap = WPT - 1, RW = N / C;
    const uint32_t* msk = um.umask + static_cast<int64_t>(b) * NW;
    const int32_t* wof = um.uwoff + static_cast<int64_t>(b) * NW;
    uint32_t* gl = um.glist + i * um.lmax;
    int base = 0;
    if (i < M) {
        const uint32_t* row = tw + static_cast<int64_t>(__ldg(perm + i)) * RW;
        // visit the row in word order; compact with ballot/popc in lane order (ascending)
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
            for (int e = 0; e < cnt; ++e) {
                const uint32_t w = __ldg(blk + 1 + e);
                const int n = static_cast<int>(w & 0xFFFFu);
                const int j = __ldg(wof + (n >> 5)) + __popc(__ldg(msk + (n >> 5)) & ((1u << (n & 31)) - 1u));
                gl[start + e] = (static_cast<uint32_t>(j) << 16) | (w >> 16);
            }
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncwarp();
    uint16_t* co = um.coff + i * (um.nchunk + 1);
    for (int c = lane; c <= um.nchunk; c += 32) {
        int lo = 0, hi = base;  // first entry with position >= 256 c
        const uint32_t key = static_cast<uint32_t>(256 * c) << 16;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (gl[mid] < key) lo = mid + 1; else hi = mid;
        }
        co[c] = static_cast<uint16_t>(lo);
    }
}

// Row permutation pi (Alg.2 iterates m in pi(0..M-1); descending-nnz order): within each
// window of PERM_W consecutive rows (one 2048-token sequence), rows sorted by stored non-zeros
// descending, ties by row index -> unique keys, deterministic.  Blocks of 128 never straddle windows.
constexpr int PERM_W = 2048;

// stored non-zeros per row (warp per row; lanes stride over the row's count words)
__global__ void row_nnz_kernel(const uint32_t* __restrict__ tw, int M, int N, int T, int C, int* __restrict__ nnz) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= M) return;
    const int NT = N / T, WPT = T / C, cap = WPT - 1;
    const uint32_t* row = tw + gw * (N / C);
    int s = 0;
    for (int t = lane; t < NT; t += 32) s += min(static_cast<int>(__ldg(row + static_cast<int64_t>(t) * WPT)), cap);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) nnz[gw] = s;
}

__global__ void __launch_bounds__(1024) union_perm_kernel(const int* __restrict__ nnz, int M, int32_t* __restrict__ perm) {
    __shared__ unsigned long long keys[PERM_W];
    const int w0 = blockIdx.x * PERM_W;
    const int rows = min(PERM_W, M - w0);
    for (int i = threadIdx.x; i < PERM_W; i += 1024) {
        unsigned long long key = ~0ull;  // padding sorts last
        if (i < rows)
            key = (static_cast<unsigned long long>(0x7FFFFFFF - __ldg(nnz + w0 + i)) << 32) | static_cast<unsigned>(w0 + i);
        keys[i] = key;
    }
    __syncthreads();
    for (int k = 2; k <= PERM_W; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < PERM_W; i += 1024) {
                const int l = i ^ j;
                if (l > i) {
                    const unsigned long long a = keys[i], c = keys[l];
                    const bool up = (i & k) == 0;
                    if ((a > c) == up) {
                        keys[i] = c;
                        keys[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < rows; i += 1024) perm[w0 + i] = static_cast<int32_t>(keys[i] & 0xFFFFFFFFu);
}

// Xp[i, :] = X[perm[i], :]  (warp per row, 16-byte vectors)
__global__ void permute_rows_kernel(const uint4* __restrict__ X, const int32_t* __restrict__ perm, int M, int K8,
                                    uint4* __restrict__ Xp) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= M) return;
    const uint4* src = X + static_cast<int64_t>(__ldg(perm + gw)) * K8;
    uint4* dst = Xp + gw * K8;
    for (int c = lane; c < K8; c += 32) dst[c] = __ldg(src + c);
}

// UP work list: for each group of UNION_GROUP blocks, chunk-major then block: tiles[] = (b << 8) | c.
// One CTA; thread per group; chunk_off[0] = total tiles.
__global__ void __launch_bounds__(1024) union_scan_kernel(UnionMeta um, int NB, int UNION_GROUP) {
    __shared__ int wsum[33];
    __shared__ int carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NG = (NB + UNION_GROUP - 1) / UNION_GROUP;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < NG; base += 1024) {
        const int g = base + threadIdx.x;
        int tot = 0, maxc = 0;
        if (g < NG) {
            for (int b = g * UNION_GROUP; b < min(NB, (g + 1) * UNION_GROUP); ++b) {
                const int c = (um.ulen[b] + 255) / 256;
                tot += c;
                maxc = max(maxc, c);
            }
        }
        int s = tot;
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
        if (g < NG) {
            int pos = carry + wsum[warp] + s - tot;
            const int b0 = g * UNION_GROUP, b1 = min(NB, (g + 1) * UNION_GROUP);
            for (int c = 0; c < maxc; ++c)
                for (int b = b0; b < b1; ++b)
                    if (c < (um.ulen[b] + 255) / 256) um.tiles[pos++] = (b << 8) | c;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += wsum[32];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        um.chunk_off[0] = carry;
        um.counters[0] = 0;
        um.counters[1] = 0;
    }
}

}  // namespace sffn
