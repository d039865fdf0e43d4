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
    int32_t* udense;     // [NB] 1: dense block (identity union; weight tiles by TMA, gates read from the TwELL)
    int32_t* tiles;      // [NB * ceil(N/256)]: UP work list, (b << 8) | chunk, grouped raster
    int* counters;       // [2] dynamic tile-scheduler counters of the UP and DOWN GEMMs
    uint32_t* glist;     // [NB*128, lmax] per (pi-ordered) row: (union position << 16) | bf16 gate, ascending
    uint16_t* coff;      // [NB*128, nchunk + 1] per row: entries before union chunk c (256 positions per chunk)
    int lmax, nchunk;
    int brows;           // token rows per union block: 128 (one tcgen05 M tile) or 256 (a CTA pair's M=256 tile)
};

constexpr int UNION_GROUP_UP = 8;    // token blocks whose up-GEMM tiles run together (L2 working set)
constexpr int UNION_GROUP_DOWN = 4;   // token blocks whose down-GEMM tiles run together (4 vs 16: -0.9% forward, -2% e2e)
constexpr int UNION_GROUP_MAX = 16;   // largest UP group the work-list builder supports

constexpr int UB_THREADS = 512;

// Visit every stored entry of one packed TwELL row, lane per tile (ascending tiles over lanes): the count word and
// the first three entries come in one 16-byte load, further entries 16 bytes at a time only when the tile holds
// them, so a row of mostly short tiles costs one 32-byte sector per tile instead of the full T/C words.
// f(word, tile, e) gets the e-th stored entry (0-based) of tile `tile`.  Requires a 16-byte aligned row.
template <class F>
__device__ __forceinline__ void for_each_tile_entry(const uint32_t* __restrict__ row, int NT, int WPT, int cap,
                                                    int t, F&& f) {
    const uint32_t* blk = row + static_cast<int64_t>(t) * WPT;
    if ((WPT & 3) == 0) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(blk));
        const int cnt = min(static_cast<int>(a.x), cap);
        if (cnt >= 1) f(a.y, 0);
        if (cnt >= 2) f(a.z, 1);
        if (cnt >= 3) f(a.w, 2);
        for (int s = 4; s <= cnt; s += 4) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(blk + s));
            f(v.x, s - 1);
            if (s + 1 <= cnt) f(v.y, s);
            if (s + 2 <= cnt) f(v.z, s + 1);
            if (s + 3 <= cnt) f(v.w, s + 2);
        }
    } else {
        const int cnt = min(static_cast<int>(__ldg(blk)), cap);
        for (int e = 0; e < cnt; ++e) f(__ldg(blk + 1 + e), e);
    }
}
// Visit every stored entry (n, word) of one packed TwELL row: warp-cooperative, lane-ordered.
// Fast path (4 <= T/C <= 32): 16-byte loads, each warp instruction covers 128 words; a lane's 4 words lie in
// one tile whose count word sits in the lane holding the tile's first word (shuffle).  Generic path otherwise.
template <class F>
__device__ __forceinline__ void for_each_row_entry(const uint32_t* __restrict__ row, int RW, int NT, int WPT, int cap,
                                                   int lane, F&& f) {
    if (WPT >= 4 && WPT <= 32) {
        const uint4* r4 = reinterpret_cast<const uint4*>(row);
        const int RW4 = RW >> 2;
        constexpr int U = 8;  // 8 x 512 bytes of the row in flight per warp
        for (int g0 = 0; g0 < RW4; g0 += 32 * U) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = (g0 + 32 * u + lane < RW4) ? __ldg(r4 + g0 + 32 * u + lane) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
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
        // lane per tile (T/C > 32: long tiles, mostly empty; T/C < 4): independent per-lane chains instead of one
        // dependent count -> entries round trip per tile for the whole warp
        for (int t = lane; t < NT; t += 32) for_each_tile_entry(row, NT, WPT, cap, t, [&](uint32_t w, int) { f(w); });
    }
}

__device__ __forceinline__ int tile_count(const uint32_t* __restrict__ row, int WPT, int cap, int t) {
    return min(static_cast<int>(__ldg(row + static_cast<int64_t>(t) * WPT)), cap);
}

// UP work list (the former union_scan kernel, now run by the last block CTA of union_meta_kernel): for each group
// of `group` blocks, chunk-major then block: tiles[] = (b << 8) | c; chunk_off[0] = total tiles; zeroes the two
// dynamic tile-scheduler counters.  NTH threads (thread ids 0..NTH-1, all in full warps), scratch = NTH/32 + 1 ints of
// shared memory; `sync` is a barrier over exactly those threads (__syncthreads or a named barrier).
struct SyncAll {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
template <int NTH, class Sync = SyncAll>
__device__ void union_scan_body(UnionMeta um, int NB, int group, int* wsum, Sync sync = Sync()) {
    constexpr int NWP = NTH / 32;
    constexpr int MAXG = UNION_GROUP_MAX;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    group = max(1, min(group, MAXG));
    const int NG = (NB + group - 1) / group;
    int carry = 0;
    for (int base = 0; base < NG; base += NTH) {
        const int g = base + static_cast<int>(threadIdx.x);
        const int b0 = g * group;
        int nchk[MAXG];  // chunks of each block of the group (registers: no dependent loads in the write loop)
        int tot = 0, maxc = 0;
#pragma unroll
        for (int j = 0; j < MAXG; ++j) {
            const int bb = b0 + j;
            nchk[j] = (g < NG && j < group && bb < NB) ? (__ldcg(um.ulen + bb) + 255) / 256 : 0;
            tot += nchk[j];
            maxc = max(maxc, nchk[j]);
        }
        int sc = tot;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, sc, off);
            if (lane >= off) sc += u;
        }
        if (lane == 31) wsum[warp] = sc;
        sync();
        if (warp == 0) {
            const int x = lane < NWP ? wsum[lane] : 0;
            int y = x;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, y, off);
                if (lane >= off) y += u;
            }
            if (lane < NWP) wsum[lane] = y - x;
            if (lane == 31) wsum[NWP] = y;
        }
        sync();
        int pos = carry + wsum[warp] + sc - tot;
        for (int c = 0; c < maxc; ++c)
#pragma unroll
            for (int j = 0; j < MAXG; ++j)
                if (c < nchk[j]) um.tiles[pos++] = ((b0 + j) << 8) | c;
        carry += wsum[NWP];
        sync();
    }
    if (threadIdx.x == 0) {
        um.chunk_off[0] = carry;
        um.counters[0] = 0;
        um.counters[1] = 0;
    }
}

// Union metadata of one block of brows pi-ordered rows, `split` CTAs (UB_THREADS) per block (split = 1 when
// there are already enough blocks to fill the GPU, up to META_SPLIT_MAX for small M):
//   1. each CTA ORs the stored indices of its brows/META_SPLIT rows into a SMEM bitmask (warp per row,
//      coalesced row reads, 8 x 512 B in flight per warp) and (split > 1) merges it into the block's global umask
//      (atomicOr of the non-zero words; umask and the counters were zeroed by union_rank_kernel);
//   2. the last CTA of the block (per-block counter) reloads the merged mask, prefix sums -> sorted U_b
//      (padded to a multiple of 64 with unit 0), uwoff / ulen / utot;
//   3. the last block to finish (global counter) builds the UP work list.
// Splitting a block's rows over several CTAs shortens the per-CTA chain of dependent row reads, which
// bounded the kernel (one CTA per block took ~57 us at any M).  Dynamic SMEM: 2 N/32 words + (UB_THREADS/32
// + 1) scan ints.
constexpr int META_SPLIT_MAX = 8;
__global__ void __launch_bounds__(UB_THREADS) union_meta_kernel(const uint32_t* __restrict__ tw, int M, int N, int T,
                                                                 int C, UnionMeta um, const int32_t* __restrict__ perm,
                                                                 int* bctr, int up_group, int split,
                                                                 int dense_units, const int* __restrict__ rnnz,
                                                                 int64_t dense_nnz) {
    extern __shared__ uint32_t ub_smem[];
    constexpr int NWP = UB_THREADS / 32;
    const int NW = N >> 5;
    uint32_t* mask = ub_smem;                                  // [NW]
    int32_t* woff = reinterpret_cast<int32_t*>(ub_smem + NW);  // [NW]
    int32_t* wsum = woff + NW;                                 // [NWP + 1]
    __shared__ int s_last;
    __shared__ int s_prow[256];
    const int b = blockIdx.x / split, part = blockIdx.x % split;
    const int NB = gridDim.x / split;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int BR = um.brows, PR = BR / split;
    const int r0 = part * PR;
    const int rows = max(0, min(PR, M - b * BR - r0));
    for (int w = threadIdx.x; w < NW; w += UB_THREADS) mask[w] = 0u;
    for (int r = threadIdx.x; r < rows; r += UB_THREADS)
        s_prow[r] = __ldg(perm + static_cast<int64_t>(b) * BR + r0 + r);
    // shortcut for dense-ish blocks: when the block's rows hold >= dense_nnz stored entries in total (a
    // multiple of N), its union is (close to) all N units: skip the OR pass and make the block dense
    __shared__ int s_bsum;
    if (threadIdx.x == 0) s_bsum = 0;
    __syncthreads();
    {
        const int brows = min(BR, M - b * BR);
        int v = 0;
        for (int r = threadIdx.x; r < brows; r += UB_THREADS)
            v += __ldg(rnnz + __ldg(perm + static_cast<int64_t>(b) * BR + r));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0 && v) atomicAdd(&s_bsum, v);
    }
    __syncthreads();
    const bool dense_block = static_cast<int64_t>(s_bsum) >= dense_nnz;

    const int NT = N / T, WPT = T / C, cap = WPT - 1, RW = N / C;
    for (int r = warp; r < (dense_block ? 0 : rows); r += NWP) {
        const uint32_t* row = tw + static_cast<int64_t>(s_prow[r]) * RW;
        for_each_row_entry(row, RW, NT, WPT, cap, lane, [&](uint32_t w) {
            const uint32_t n = w & 0xFFFFu;
            atomicOr(&mask[n >> 5], 1u << (n & 31));
        });
    }
    __syncthreads();
    uint32_t* gmask = um.umask + static_cast<int64_t>(b) * NW;
    if (split > 1) {
        for (int w = threadIdx.x; w < NW; w += UB_THREADS)
            if (mask[w] && !dense_block) atomicOr(gmask + w, mask[w]);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(bctr + b, 1) == split - 1;
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        for (int w = threadIdx.x; w < NW; w += UB_THREADS) mask[w] = dense_block ? 0xFFFFFFFFu : __ldcg(gmask + w);
        __syncthreads();
    } else {
        for (int w = threadIdx.x; w < NW; w += UB_THREADS) {
            if (dense_block) mask[w] = 0xFFFFFFFFu;
            gmask[w] = mask[w];
        }
        __syncthreads();
    }

    // exclusive scan of popc(mask[w]) over w (each thread owns a contiguous segment); a block whose union
    // reaches dense_units is made dense (all N units, identity list): the union GEMMs then load its weight
    // tiles by TMA instead of gathering (cheaper than gathering most of the rows anyway)
    for (int pass = 0; pass < 2; ++pass) {
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
        int v = lane < NWP ? wsum[lane] : 0;
        int sc = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, sc, off);
            if (lane >= off) sc += u;
        }
        if (lane < NWP) wsum[lane] = sc - v;  // exclusive warp offsets
        if (lane == NWP - 1) wsum[NWP] = sc;  // total
    }
    __syncthreads();
    int run = wsum[warp] + incl - local;
    for (int w = w0; w < w1; ++w) {
        woff[w] = run;
        run += __popc(mask[w]);
    }
    __syncthreads();
    if (pass == 0 && wsum[NWP] >= dense_units && wsum[NWP] < N) {
        __syncthreads();
        for (int w = threadIdx.x; w < NW; w += UB_THREADS) mask[w] = 0xFFFFFFFFu;
        __syncthreads();
        continue;
    }
    break;
    }
    const int total = wsum[NWP];
    const int padded = max(64, (total + 63) & ~63);
    if (total == N)  // dense (forced or natural): the gate lists read the all-ones mask
        for (int w = threadIdx.x; w < NW; w += UB_THREADS) gmask[w] = mask[w];

    int32_t* ul = um.ulist + static_cast<int64_t>(b) * N;
    for (int w = threadIdx.x; w < NW; w += UB_THREADS) {
        uint32_t m = mask[w];
        int pos = woff[w];
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
        um.udense[b] = (dense_units <= N && total == N) ? 1 : 0;  // only when the dense (TMA) path is enabled
    }

    // the last CTA builds the UP work list from every block's ulen
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(bctr + NB, 1) == NB - 1;
    __syncthreads();
    if (s_last) {
        __threadfence();
        union_scan_body<UB_THREADS>(um, NB, up_group, wsum);
    }
}

// Compact gate lists for the UP epilogue (instead of materialising G in H_c): warp per pi-ordered row i (8 per
// CTA); the row's stored entries in ascending neuron order = ascending union position (lane per tile, warp prefix
// of the tile counts); position = uwoff + popc(umask prefix); coff[i][c] = entries with position < 256 c, from
// per-warp SMEM chunk counters.  Dynamic SMEM: 8 x (nchunk + 1) ints.
// The same warp also copies its row of X into pi order (Xp[i] = X[perm[i]], the UP GEMM's TMA-loaded A operand;
// formerly a separate permute_rows_kernel): the HBM-bound copy overlaps the latency-bound gate-list reads.
constexpr int GL_COPY_U = 4;  // 16-byte X loads in flight per lane
__global__ void __launch_bounds__(256) union_gate_list_kernel(const uint32_t* __restrict__ tw, int M, int N, int T,
                                                              int C, UnionMeta um, const int32_t* __restrict__ perm,
                                                              const uint4* __restrict__ X, int K8,
                                                              uint4* __restrict__ Xp) {
    extern __shared__ int32_t gl_smem[];
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int BR = um.brows;
    const int NB = (M + BR - 1) / BR;
    if (i >= static_cast<int64_t>(NB) * BR) return;
    const int b = static_cast<int>(i / BR);
    const int nch = um.nchunk;
    int32_t* cc = gl_smem + warp * (nch + 1);
    for (int c = lane; c <= nch; c += 32) cc[c] = 0;
    __syncwarp();
    const int NW = N >> 5, NT = N / T, WPT = T / C, cap = WPT - 1, RW = N / C;
    const uint32_t* msk = um.umask + static_cast<int64_t>(b) * NW;
    const int32_t* wof = um.uwoff + static_cast<int64_t>(b) * NW;
    uint32_t* gl = um.glist + i * um.lmax;
    const int64_t src_row = i < M ? static_cast<int64_t>(__ldg(perm + i)) : -1;
    if (src_row >= 0 && Xp) {
        const uint4* src = X + src_row * K8;
        uint4* dst = Xp + i * K8;
        for (int c0 = 0; c0 < K8; c0 += 32 * GL_COPY_U) {
            uint4 v[GL_COPY_U];
#pragma unroll
            for (int u = 0; u < GL_COPY_U; ++u) {
                const int c = c0 + 32 * u + lane;
                if (c < K8) v[u] = __ldcs(src + c);
            }
#pragma unroll
            for (int u = 0; u < GL_COPY_U; ++u) {
                const int c = c0 + 32 * u + lane;
                if (c < K8) dst[c] = v[u];
            }
        }
    }
    const bool dense = __ldg(um.udense + b) != 0;  // identity union: the UP epilogue reads the TwELL directly
    if (dense) return;
    auto emit = [&](uint32_t w, int idx) {
        const int n = static_cast<int>(w & 0xFFFFu);
        const int j = dense ? n : __ldg(wof + (n >> 5)) + __popc(__ldg(msk + (n >> 5)) & ((1u << (n & 31)) - 1u));
        gl[idx] = (static_cast<uint32_t>(j) << 16) | (w >> 16);
        atomicAdd(&cc[j >> 8], 1);
    };
    if (i < M) {
        const uint32_t* row = tw + src_row * RW;
        // lane per tile (ascending): measured faster here than coalesced whole-row reads (the row's
        // first-touch DRAM read happened in union_meta_kernel; these sector reads mostly hit L2)
        int base = 0;
        for (int t0 = 0; t0 < NT; t0 += 32) {
            const int t = t0 + lane;
            const int cnt = t < NT ? tile_count(row, WPT, cap, t) : 0;
            int inc = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += v;
            }
            const int start = base + inc - cnt;
            if (t < NT) for_each_tile_entry(row, NT, WPT, cap, t, [&](uint32_t w, int e) { emit(w, start + e); });
            base += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    __syncwarp();
    uint16_t* co = um.coff + i * (nch + 1);
    int carry = 0;
    for (int c0 = 0; c0 <= nch; c0 += 32) {
        const int c = c0 + lane;
        const int v = c <= nch ? cc[c] : 0;
        int inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += u;
        }
        if (c <= nch) co[c] = static_cast<uint16_t>(carry + inc - v);
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
}

// G_b: the stored gate values in union coordinates, H_c[b*128 + r, j] (bf16), zero elsewhere; the up-GEMM
// epilogue multiplies this tile in place by X_b W_u[U_b]^T.  One CTA (256 threads) per 8 rows of a block.
constexpr int GS_ROWS = 8;
__global__ void __launch_bounds__(256) union_gate_scatter_kernel(const uint32_t* __restrict__ tw, int M, int N, int T,
                                                                 int C, UnionMeta um, uint16_t* __restrict__ hc,
                                                                 const int32_t* __restrict__ perm) {
    const int BR = um.brows;
    const int b = blockIdx.x / (BR / GS_ROWS);
    const int r0 = (blockIdx.x % (BR / GS_ROWS)) * GS_ROWS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp w handles row r0 + w
    const int NW = N >> 5, NT = N / T, WPT = T / C, cap = WPT - 1, RW = N / C;
    const int padded = __ldg(um.ulen + b);
    const uint32_t* msk = um.umask + static_cast<int64_t>(b) * NW;
    const int32_t* wof = um.uwoff + static_cast<int64_t>(b) * NW;
    const int r = r0 + warp;
    uint16_t* hrow = hc + (static_cast<int64_t>(b) * BR + r) * N;
    for (int c = lane; c < padded / 8; c += 32) *reinterpret_cast<uint4*>(hrow + 8 * c) = make_uint4(0, 0, 0, 0);
    __syncwarp();
    if (static_cast<int64_t>(b) * BR + r >= M) return;
    const uint32_t* row = tw + static_cast<int64_t>(__ldg(perm + static_cast<int64_t>(b) * BR + r)) * RW;
    for_each_row_entry(row, RW, NT, WPT, cap, lane, [&](uint32_t w) {
        const int n = static_cast<int>(w & 0xFFFFu);
        const int j = __ldg(wof + (n >> 5)) + __popc(__ldg(msk + (n >> 5)) & ((1u << (n & 31)) - 1u));
        hrow[j] = static_cast<uint16_t>(w >> 16);
    });
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

// pi: stable descending order of stored non-zeros within each window, i.e. row i of a window goes to position
//   #{ j in window : nnz_j > nnz_i  or  (nnz_j == nnz_i and j < i) }.
// One CTA (PERM_THREADS) per window: the window's packed keys (nnz << 11) | (2047 - j) — unique, so the order is
// total and deterministic — bitonic-sorted descending (66 compare-exchange stages; padding rows get -1 and sort
// last), then perm[w0 + p] = w0 + (2047 - (key_p & 2047)).  (The former ranking kernel compared every row with
// all 2048 keys: 4 M comparisons per window.)
// The grid also zeroes union_meta_kernel's merged masks and counters.
constexpr int PERM_THREADS = PERM_W / 2;
static_assert(PERM_W == 2048, "rank keys pack the window index in 11 bits");
__global__ void __launch_bounds__(PERM_THREADS) union_rank_kernel(const int* __restrict__ nnz, int M,
                                                                 int32_t* __restrict__ perm,
                                                                 uint32_t* __restrict__ zero_a, int64_t na,
                                                                 int* __restrict__ zero_b, int nb) {
    {  // zero union_meta_kernel's merged masks and counters (it runs after this kernel on the same stream)
        const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
        for (int64_t i = t; i < na; i += nt) zero_a[i] = 0u;
        for (int64_t i = t; i < nb; i += nt) zero_b[i] = 0;
    }
    // thread t holds the keys at positions t and t + 1024; a compare-exchange of positions p < q = p ^ j keeps the
    // larger key at p in descending blocks ((p & k) == 0) and the smaller one otherwise.  Partners within a warp
    // (j < 32) by shuffle, j = 1024 in registers, the rest through double-buffered SMEM (one barrier per stage).
    __shared__ int key[2][PERM_W];
    const int w0 = blockIdx.x * PERM_W;
    const int rows = min(PERM_W, M - w0);
    const int t = threadIdx.x;
    int v[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const int i = t + s * PERM_THREADS;
        v[s] = i < rows ? (__ldg(nnz + w0 + i) << 11) | (PERM_W - 1 - i) : -1;
    }
    auto cx = [](int p, int j, int k, int mine, int other) {
        const bool desc = (p & k) == 0, lower = (p & j) == 0;
        return (desc == lower) ? max(mine, other) : min(mine, other);
    };
    int buf = 0;
    for (int k = 2; k <= PERM_W; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == PERM_THREADS) {  // partner: the thread's other key
                const int a = v[0], c = v[1];
                v[0] = cx(t, j, k, a, c);
                v[1] = cx(t + PERM_THREADS, j, k, c, a);
            } else if (j >= 32) {
                key[buf][t] = v[0];
                key[buf][t + PERM_THREADS] = v[1];
                __syncthreads();
                const int o0 = key[buf][t ^ j], o1 = key[buf][(t + PERM_THREADS) ^ j];
                v[0] = cx(t, j, k, v[0], o0);
                v[1] = cx(t + PERM_THREADS, j, k, v[1], o1);
                buf ^= 1;
            } else {
#pragma unroll
                for (int s = 0; s < 2; ++s) v[s] = cx(t + s * PERM_THREADS, j, k, v[s], __shfl_xor_sync(0xffffffffu, v[s], j));
            }
        }
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const int p = t + s * PERM_THREADS;
        if (p < rows) perm[w0 + p] = w0 + (PERM_W - 1 - (v[s] & (PERM_W - 1)));
    }
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

}  // namespace sffn
