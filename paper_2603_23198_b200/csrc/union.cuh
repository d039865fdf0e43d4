// union.cuh — block-union metadata layout and helpers for the tensor-core sparse up/down (
// the metadata itself is built by prep.cuh).
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

// token blocks whose up-GEMM tiles run together: min(NB / 8, the blocks whose X rows fill 32 MB), clamped to [8, 32].
// With the fraction-ordered work list the group's X tiles are the L2 working set that grows with the group (ncu,
// profiles/r02/s3/ncu_up_group_order.txt: UP fastest at 32 blocks for 7B (1 MB of X per block), 16 for 70B (2 MB), within
// 1.3% for 1B); interleaved A/B without the ordering: 32 vs 8 was 1.2-2% faster at 7B / 70B, and 8 stays best for
// the 4096-row chunks of the host pipeline (NB = 32)
__host__ __device__ constexpr int union_group_up(int64_t NB, int64_t K) {
    const int64_t by_x = (int64_t(32) << 20) / (128 * K * 2);
    const int64_t g = NB / 8 < by_x ? NB / 8 : by_x;
    return g < 8 ? 8 : (g > 32 ? 32 : static_cast<int>(g));
}
constexpr int UNION_GROUP_DOWN = 4;   // token blocks whose down-GEMM tiles run together (4 vs 16: -0.9% forward, -2% e2e)
constexpr int UNION_GROUP_MAX = 64;   // largest UP group the work-list builder supports

// CTAs per union block of the prep kernel when M is small (a power of two dividing the block rows)
constexpr int META_SPLIT_MAX = 8;

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

// UP work list (run by the last block builder of the prep kernel): for each group
// of `group` blocks, chunk-major then block: tiles[] = (b << 8) | c; chunk_off[0] = total tiles; zeroes the two
// dynamic tile-scheduler counters.  NTH threads (thread ids 0..NTH-1, all in full warps), scratch wsum = NTH/32 + 1
// and goff = NTH ints of shared memory; `sync` is a barrier over exactly those threads (__syncthreads or a named
// barrier).
struct SyncAll {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
template <int NTH, class Sync = SyncAll>
__device__ void union_scan_body(UnionMeta um, int NB, int group, int* wsum, int* goff, Sync sync = Sync(),
                                bool order_by_fraction = false, bool snake = false) {
    constexpr int NWP = NTH / 32;
    constexpr int MAXG = UNION_GROUP_MAX;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    group = max(1, min(group, MAXG));
    const int NG = (NB + group - 1) / group;
    int carry = 0;
    for (int base = 0; base < NG; base += NTH) {
        const int g = base + static_cast<int>(threadIdx.x);
        const int b0 = g * group;
        int tot = 0;  // tiles of this thread's group (16 independent loads in flight per batch)
        if (g < NG)
            for (int j0 = 0; j0 < group; j0 += 16) {
                int l[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int bb = b0 + j0 + j;
                    l[j] = (j0 + j < group && bb < NB) ? (__ldcg(um.ulen + bb) + 255) / 256 : 0;
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) tot += l[j];
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
        goff[threadIdx.x] = carry + wsum[warp] + sc - tot;  // first tile of this thread's group
        sync();
        // warp w writes groups w, w + NWP, ... of this round: lane j (and j + 32) holds block j's chunk count, one
        // ballot per chunk index places the group's blocks that have that chunk (chunk-major, block ascending)
        const unsigned lt = (1u << lane) - 1u;
        for (int i = warp; i < NTH && base + i < NG; i += NWP) {
            const int gi = base + i;
            int p = goff[i];
            const int bi = gi * group;
            const int n0 = (lane < group && bi + lane < NB) ? (__ldcg(um.ulen + bi + lane) + 255) / 256 : 0;
            const int n1 = (lane + 32 < group && bi + lane + 32 < NB) ? (__ldcg(um.ulen + bi + lane + 32) + 255) / 256 : 0;
            const int mc = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(max(n0, n1))));
            if (!order_by_fraction) {
                for (int c = 0; c < mc; ++c) {
                    const unsigned m0 = __ballot_sync(0xffffffffu, c < n0), m1 = __ballot_sync(0xffffffffu, c < n1);
                    if (c < n0) um.tiles[p + __popc(m0 & lt)] = ((bi + lane) << 8) | c;
                    if (c < n1) um.tiles[p + __popc(m0) + __popc(m1 & lt)] = ((bi + lane + 32) << 8) | c;
                    p += __popc(m0) + __popc(m1);
                }
            } else {
                // slot s emits chunk floor(s * n / mc) of a block with n chunks when it changes: every block's chunks
                // advance at the same rate through its union, so concurrent tiles cover similar unit ranges (the
                // union of a block is spread evenly over N) and share gathered weight rows in L2
                // snake (default; SFFN_UP_SNAKE=0 disables): odd groups walk their unions backwards, so a group starts
                // on the unit range the previous group ended on (ncu: UP DRAM -5-7%, time -0.1% 7B / -0.4% 70B)
                const bool rev = snake && (gi & 1);
                for (int s_ = 0; s_ < mc; ++s_) {
                    const int t = rev ? mc - 1 - s_ : s_, tp = rev ? t + 1 : t - 1;
                    const int c0 = t * n0 / mc, c1 = t * n1 / mc;
                    const bool e0 = n0 > 0 && (s_ == 0 || c0 != tp * n0 / mc);
                    const bool e1 = n1 > 0 && (s_ == 0 || c1 != tp * n1 / mc);
                    const unsigned m0 = __ballot_sync(0xffffffffu, e0), m1 = __ballot_sync(0xffffffffu, e1);
                    if (e0) um.tiles[p + __popc(m0 & lt)] = ((bi + lane) << 8) | c0;
                    if (e1) um.tiles[p + __popc(m0) + __popc(m1 & lt)] = ((bi + lane + 32) << 8) | c1;
                    p += __popc(m0) + __popc(m1);
                }
            }
        }
        carry += wsum[NWP];
        sync();
    }
    if (threadIdx.x == 0) {
        um.chunk_off[0] = carry;
        um.counters[0] = 0;
        um.counters[1] = 0;
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

}  // namespace sffn
