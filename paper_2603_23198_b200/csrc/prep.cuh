// prep.cuh — the union path's metadata in ONE launch (DESIGN.md §7 K2 "prep"): row order pi, block unions, the UP
// work list, the compact gate lists and X in pi order.  Replaces union_rank_kernel + union_meta_kernel +
// union_gate_list_kernel of round 1 (three launches, each re-reading its inputs).
//
// One CTA (PREP_THREADS) per (block of BR pi-ordered rows, part), `split` parts per block for small M.  Per CTA:
//   1. pi (Alg.2 iterates m in pi(0..M-1); descending stored non-zeros per 2048-row window): every CTA
//      bitonic-sorts its window's 2048 unique keys (nnz << 11 | 2047 - j) itself — 16 (x split) identical sorts per
//      window, no cross-CTA wait — and keeps the rows at its block's positions; writes perm for its rows;
//   2. warp 15 lane 0 streams the CTA's rows of X into pi order (Xp) with 1-D bulk copies (TMA engine, 8 KB pieces
//      through an 8-slot SMEM ring), asynchronous to everything below;
//   3. warps 0-14: OR of the rows' stored indices into a SMEM bitmask; split > 1: merged into
//      the block's global mask (atomicOr), the last part builds;
//   4. the builder: prefix sums -> sorted U_b (padded to a multiple of 64 with unit 0), uwoff / ulen / utot / udense;
//      releases the block (flag) for the other parts; the last builder overall writes the UP work list;
//   5. warps 0-14: the gate lists of the CTA's rows from the block's mask in SMEM (gated forward only).
// Counters (logical CTA ids, per-block arrivals and flags, builders) are zeroed by the caller's memset that also
// zeroes the gate GEMM's row counts.  Logical CTA ids come from an atomic counter, so a part that waits for its
// block's builder never waits for a CTA that has not started (the builder is the last part to arrive).
#pragma once
#include "union.cuh"

namespace sffn {

constexpr int PREP_THREADS = 512;
constexpr int PREP_WORK = PREP_THREADS - 32;  // warps 0-14: OR / build / gate lists; warp 15: X copy
constexpr int PREP_NW = PREP_WORK / 32;
constexpr int PREP_SLOTS = 8, PREP_PIECE = 8192;  // X copy ring: 8 slots of `piece` bytes (8 KB standalone)
constexpr int PREP_U = 2;   // TwELL tiles per lane per row in flight (56 tiles per row at N = 14336, T = 256)
constexpr int PREP_RR = 2;  // rows per warp in flight in the OR pass
constexpr int PREP_UD = 1;  // dense path: tiles per lane in flight (4 x 16 bytes each)
constexpr int PREP_DENSE_ROW = 3;  // mean stored entries per tile above which a block's rows take the one-row dense path
struct PrepCtr {         // int offsets into the prep counter block (zeroed by the caller)
    static constexpr int lid = 0, built = 1, arrive = 2;  // arrive[NB], then flag[NB]
};

__device__ __forceinline__ void prep_sync() { asm volatile("bar.sync 1, %0;" ::"n"(PREP_WORK) : "memory"); }
// optional per-CTA phase timestamps (globaltimer, ns): trace[8 * lid + k], k = 0 start, 1 sorted, 2 OR pass done,
// 3 union built, 4 gate lists done, 5 X copy done (tools only; null in production)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
struct PrepSync {
    __device__ __forceinline__ void operator()() const { prep_sync(); }
};
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }

// dynamic SMEM: ring PREP_SLOTS x piece (the sort's keys, 2 x 2048 ints, live in it before the X copy starts: piece
// >= 2 KB) | mask NW | woff NW | gate-list chunk counters PREP_NW x (nchunk + 1) | wsum | work-list group offsets
inline size_t prep_smem_bytes(int N, int nchunk, int piece = PREP_PIECE) {
    return 1024 + static_cast<size_t>(PREP_SLOTS) * piece + 2 * (N / 32) * 4 + PREP_NW * (nchunk + 1) * 4 + 64 * 4 +
           PREP_WORK * 4;
}
// static SMEM of the prep kernel (mbarriers, per-row tables, scalars), for the host's co-residency budget
constexpr int PREP_STATIC_SMEM = PREP_SLOTS * 8 + 2 * 256 * 4 + 16;
// loads of what the gate GEMM wrote (TwELL, row counts): read-only path standalone; L2 (coherent) when the prep
// kernel runs concurrently with the gate GEMM (OV), whose writes it observes through the window counters
template <bool OV, class Tp>
__device__ __forceinline__ Tp pld(const Tp* p) {
    if constexpr (OV) return __ldcg(p);
    else return __ldg(p);
}

// Parts (CTAs) per block: the base split (small M) times a boost for the densest blocks of each 2048-row window —
// the rows are in descending stored-nnz order, so a window's first blocks carry 2-3x the entries of its median block
// and set the kernel's span (per-CTA phase trace, DESIGN.md §7 "prep").  boost 0: uniform; 1: x2 for window positions
// 0-1; 2: x4 for position 0, x2 for 1-2.  The host picks the strongest boost whose CTAs fit in one wave.
__host__ __device__ inline int prep_parts(int bw, int base, int boost) {
    const int m = boost == 2 ? (bw == 0 ? 4 : (bw < 3 ? 2 : 1)) : (boost == 1 ? (bw < 2 ? 2 : 1) : 1);
    return min(META_SPLIT_MAX, base * m);
}
// logical CTA lid -> (block b, part); returns the block's part count (0 past the end).  Order: window position
// major (every window's densest block first, the sparsest last), then window, then part — the heavy CTAs start in
// the first wave and a block's parts have consecutive ids (a waiting part never waits for an unstarted builder).
__host__ __device__ inline int prep_map(int lid, int NB, int WB, int base, int boost, int* b, int* part) {
    const int NWIN = (NB + WB - 1) / WB;
    int rem = lid;
    for (int bw = 0; bw < WB; ++bw) {
        const int nw = NWIN - 1 + (((NWIN - 1) * WB + bw < NB) ? 1 : 0);  // windows that have position bw
        const int sp = prep_parts(bw, base, boost);
        if (rem < nw * sp) {
            *b = (rem / sp) * WB + bw;
            *part = rem % sp;
            return sp;
        }
        rem -= nw * sp;
    }
    *b = -1;
    *part = 0;
    return 0;
}
// Overlapped prep (OV): window-major ids (window w's CTAs start before window w+1's, so the CTAs resident beside the
// gate GEMM are those of the windows it finishes first), each window's blocks in position order; the windows of the
// gate GEMM's last raster group (w >= tail_w0: they complete when the GEMM ends and are then the critical path) get
// tail_split parts per block, the others prep_parts(bw, base, boost)
__host__ __device__ inline int prep_map_ov(int lid, int NB, int WB, int base, int boost, int tail_w0, int tail_split,
                                           int* b, int* part) {
    const int NWIN = (NB + WB - 1) / WB;
    int rem = lid;
    for (int w = 0; w < NWIN; ++w) {
        const int nbw = min(WB, NB - w * WB);
        int wp = 0;
        for (int bw = 0; bw < nbw; ++bw) wp += w >= tail_w0 ? tail_split : prep_parts(bw, base, boost);
        if (rem >= wp) {
            rem -= wp;
            continue;
        }
        for (int bw = 0; bw < nbw; ++bw) {
            const int sp = w >= tail_w0 ? tail_split : prep_parts(bw, base, boost);
            if (rem < sp) {
                *b = w * WB + bw;
                *part = rem;
                return sp;
            }
            rem -= sp;
        }
    }
    *b = -1;
    *part = 0;
    return 0;
}
inline int prep_ctas_ov(int NB, int WB, int base, int boost, int tail_w0, int tail_split) {
    int n = 0;
    for (int b = 0; b < NB; ++b) n += (b / WB) >= tail_w0 ? tail_split : prep_parts(b % WB, base, boost);
    return n;
}
inline int prep_ctas(int NB, int WB, int base, int boost) {
    int n = 0;
    const int NWIN = (NB + WB - 1) / WB;
    for (int bw = 0; bw < WB; ++bw) n += (NWIN - 1 + (((NWIN - 1) * WB + bw < NB) ? 1 : 0)) * prep_parts(bw, base, boost);
    return n;
}

// OV: launched as a programmatic dependent of the gate GEMM (which must have been given win_done); every CTA waits
// for its window's count before reading the window's row counts and TwELL rows
struct PrepOv {
    const int* win_done;  // per 2048-row window: epilogue warp-tiles done (gate GEMM), null standalone
    int win_n;            // gate GEMM N-tiles (a window is complete at ceil(rows / 32) * win_n)
    int tail_w0, tail_split;
};
template <bool OV>
__global__ void __launch_bounds__(PREP_THREADS, 2) union_prep_kernel(
    const uint32_t* __restrict__ tw, int M, int N, int T, int C, UnionMeta um, int32_t* __restrict__ perm,
    const int* __restrict__ rnnz, int* __restrict__ pctr, int up_group, int split_base, int split_boost, int piece,
    PrepOv ov, int dense_units, int64_t dense_nnz,
    const uint8_t* __restrict__ X, int64_t row_bytes, uint8_t* __restrict__ Xp, int gate_lists,
    unsigned long long* trace) {
    extern __shared__ uint8_t prep_raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(prep_raw) + 1023) & ~uintptr_t(1023));
    int* key = reinterpret_cast<int*>(ring);  // [2][2048], in the ring until the X copy starts (after the OR pass)
    const int NW = N >> 5;
    uint32_t* mask = reinterpret_cast<uint32_t*>(ring + PREP_SLOTS * piece);  // [NW]
    int32_t* woff = reinterpret_cast<int32_t*>(mask + NW);                // [NW]
    int32_t* ccnt = woff + NW;                                            // [PREP_NW][nchunk + 1]
    int32_t* wsum = ccnt + PREP_NW * (um.nchunk + 1);                     // [PREP_NW + 1]
    int32_t* goff = wsum + 64;                                            // [PREP_WORK] work-list group offsets
    __shared__ uint64_t full[PREP_SLOTS];
    __shared__ int s_prow[256], s_rcnt[256];
    __shared__ int s_lid, s_last, s_bsum;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
    const int BR = um.brows;
    const int NB = (M + BR - 1) / BR;

    if (t == 0) {
        s_lid = atomicAdd(pctr + PrepCtr::lid, 1);
        s_bsum = 0;
        for (int i = 0; i < PREP_SLOTS; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int lid = s_lid;
    if (trace && t == 0) trace[8 * lid] = gtimer();
    int b, part;
    const int split = OV ? prep_map_ov(lid, NB, PERM_W / BR, split_base, split_boost, ov.tail_w0, ov.tail_split, &b, &part)
                         : prep_map(lid, NB, PERM_W / BR, split_base, split_boost, &b, &part);
    if (split == 0) return;  // more CTAs than prep_ctas() (launch error): uniform across the CTA, nothing to do
    const int PR = BR / split;
    if constexpr (OV) {
        // the window's TwELL rows and row counts are complete once every epilogue warp-tile of its rows has signalled
        // (gate GEMM: TMA store waited, fenced, then the atomic); acquire, then L2 loads (pld<true>)
        if (t == 0) {
            const int w = (b * BR) / PERM_W;
            const int need = ((min(PERM_W, M - w * PERM_W) + 31) / 32) * ov.win_n;
            int v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ov.win_done + w) : "memory");
                if (v >= need) break;
                __nanosleep(500);
            }
        }
        __syncthreads();
    }
    // part `part` owns the block rows part, part + split, part + 2 split, ...: the rows are in descending-nnz order,
    // so interleaving balances the parts' work (contiguous ranges gave part 0 the densest rows and made every
    // other part wait for it at the merge)
    auto prow = [&](int r) -> int64_t { return static_cast<int64_t>(b) * BR + static_cast<int64_t>(r) * split + part; };
    const int w0 = (b * BR) / PERM_W * PERM_W;                    // window start row
    const int pb = b * BR - w0;                                   // block start position within the window
    const int wrows = min(PERM_W, M - w0);
    const int rows = max(0, min(PR, (M - b * BR - part + split - 1) / split));  // real rows of this part

    // ---------------------------------------------------------------- 1. pi: bitonic sort of the window (descending)
    // thread t holds positions 4t .. 4t+3: partners at distance j = 1, 2 in registers, 4..64 in the warp (shuffle),
    // >= 128 through SMEM (10 of the 66 stages; one barrier each, double-buffered); every loop is unrolled so the
    // register indices are static
    int v[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int i = 4 * t + s;
        v[s] = i < wrows ? (pld<OV>(rnnz + w0 + i) << 11) | (PERM_W - 1 - i) : -1;
    }
    {
        auto cx = [](int p, int j, int k, int mine, int other) {
            const bool desc = (p & k) == 0, lower = (p & j) == 0;
            return (desc == lower) ? max(mine, other) : min(mine, other);
        };
        int4* kb4 = reinterpret_cast<int4*>(key);
        int buf = 0;
#pragma unroll
        for (int k = 2; k <= PERM_W; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                if (j <= 2) {
                    int nv[4];
#pragma unroll
                    for (int s = 0; s < 4; ++s) nv[s] = cx(4 * t + s, j, k, v[s], v[s ^ j]);
#pragma unroll
                    for (int s = 0; s < 4; ++s) v[s] = nv[s];
                } else if (j <= 64) {
#pragma unroll
                    for (int s = 0; s < 4; ++s)
                        v[s] = cx(4 * t + s, j, k, v[s], __shfl_xor_sync(0xffffffffu, v[s], j >> 2));
                } else {
                    int4* kb = kb4 + buf * (PERM_W / 4);
                    kb[t] = make_int4(v[0], v[1], v[2], v[3]);
                    __syncthreads();
                    const int4 o = kb[t ^ (j >> 2)];
                    v[0] = cx(4 * t + 0, j, k, v[0], o.x);
                    v[1] = cx(4 * t + 1, j, k, v[1], o.y);
                    v[2] = cx(4 * t + 2, j, k, v[2], o.z);
                    v[3] = cx(4 * t + 3, j, k, v[3], o.w);
                    buf ^= 1;
                }
            }
        }
    }
    // this part's rows (block positions part, part + split, ...) and the block's stored-entry sum (dense shortcut)
    int bs = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int p = 4 * t + s;
        if (v[s] >= 0 && p >= pb && p < pb + BR) {
            bs += v[s] >> 11;
            const int br = p - pb;
            const int r = (br % split == part) ? br / split : -1;
            if (r >= 0 && r < PR) {
                const int row = w0 + (PERM_W - 1 - (v[s] & (PERM_W - 1)));
                s_prow[r] = row;
                s_rcnt[r] = v[s] >> 11;  // stored entries of the row (the gate GEMM's count)
                perm[prow(r)] = row;
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) bs += __shfl_xor_sync(0xffffffffu, bs, off);
    if (lane == 0 && bs) atomicAdd(&s_bsum, bs);
    __syncthreads();
    const bool dense_block = static_cast<int64_t>(s_bsum) >= dense_nnz;
    if (trace && t == 0) trace[8 * lid + 1] = gtimer();

    if (warp == PREP_NW) {
        // ------------------------------------------------------------ 2. X rows into pi order (bulk copies)
        // start after this CTA's OR pass (the latency-bound TwELL reads run on a quiet DRAM; the copy then overlaps the
        // union build and the gate lists)
        asm volatile("bar.sync 2, %0;" ::"n"(PREP_THREADS) : "memory");
        if (lane == 0 && Xp && rows > 0) {
            constexpr int LA = PREP_SLOTS - 2;  // loads in flight; the slot reused next was stored 2 pieces ago
            const uint64_t pol = policy_evict_first();  // X is read once here
            const int per_row = static_cast<int>((row_bytes + piece - 1) / piece);
            const int n = rows * per_row;
            auto piece_at = [&](int i, const uint8_t*& src, uint8_t*& dst, uint32_t& bytes) {
                const int r = i / per_row, q = i % per_row;
                const int64_t off = static_cast<int64_t>(q) * piece;
                bytes = static_cast<uint32_t>((row_bytes - off < piece ? row_bytes - off : static_cast<int64_t>(piece)));
                src = X + static_cast<int64_t>(s_prow[r]) * row_bytes + off;
                dst = Xp + prow(r) * row_bytes + off;
            };
            auto load = [&](int i) {
                const uint8_t* src;
                uint8_t* dst;
                uint32_t bytes;
                piece_at(i, src, dst, bytes);
                const int sl = i % PREP_SLOTS;
                mbar_arrive_expect_tx(&full[sl], bytes);
                bulk_g2s(ring + sl * piece, src, bytes, &full[sl], pol);
            };
            for (int i = 0; i < min(n, LA); ++i) load(i);
            for (int i = 0; i < n; ++i) {
                const int sl = i % PREP_SLOTS;
                // relaxed: the data is only read by the async proxy (the bulk store); an acquire wait would
                // invalidate the SM's L1 under the other warps' TwELL reads
                mbar_wait_relaxed(&full[sl], static_cast<uint32_t>((i / PREP_SLOTS) & 1));
                const uint8_t* src;
                uint8_t* dst;
                uint32_t bytes;
                piece_at(i, src, dst, bytes);
                if constexpr (OV) {
                    // beside the gate GEMM: keep its X / W_g tiles in L2 (X_pi is re-read only after the GEMM)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                                     dst),
                                 "r"(smem_u32(ring + sl * piece)), "r"(bytes), "l"(pol)
                                 : "memory");
                } else {
                    bulk_s2g(dst, ring + sl * piece, bytes);
                }
                bulk_commit();
                if (i + LA < n) {
                    bulk_wait_read<PREP_SLOTS - LA>();  // the store of piece i + LA - PREP_SLOTS has read its slot
                    load(i + LA);
                }
            }
            bulk_wait0();
        }
        if (trace && lane == 0) trace[8 * lid + 5] = gtimer();
        return;
    }

    // -------------------------------------------------------------------- 3. OR of the part's rows (warps 0-14)
    const int NT = N / T, WPT = T / C, cap = WPT - 1, RW = N / C;
    for (int w = t; w < NW; w += PREP_WORK) mask[w] = 0u;
    prep_sync();
    // lane per tile, PREP_U tiles in flight per lane (count + first three entries in one 16-byte load); the warp
    // prefix of the tile counts gives each entry its place in the row's ascending list, stashed raw (unit | gate)
    // in the row's gate list and turned into union positions in step 5 (no second pass over the TwELL)
    // Dense rows (the first blocks of each window: several stored entries per tile) would need dependent loads past
    // entry 6 of most tiles; rows with more than PREP_DENSE_ROW entries per tile on average take a one-row path that
    // loads count + 15 entries of every tile up front (4 x 16 bytes per lane and tile), the others the two-row path.
    const bool dense_rows = (WPT & 3) == 0 && WPT >= 16 && !dense_block &&
                            static_cast<int64_t>(s_bsum) > static_cast<int64_t>(PREP_DENSE_ROW) * NT * BR;
    for (int r = warp; r < (dense_rows ? rows : 0); r += PREP_NW) {
        const uint32_t* row = tw + static_cast<int64_t>(s_prow[r]) * RW;
        uint32_t* glr = um.glist + prow(r) * um.lmax;
        int base = 0;
        for (int t0 = 0; t0 < NT; t0 += 32 * PREP_UD) {
            uint4 a[PREP_UD][4];
#pragma unroll
            for (int u = 0; u < PREP_UD; ++u) {
                const int tt = t0 + 32 * u + lane;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    a[u][q] = make_uint4(0, 0, 0, 0);
                    if (tt < NT) a[u][q] = pld<OV>(reinterpret_cast<const uint4*>(row + static_cast<int64_t>(tt) * WPT + 4 * q));
                }
            }
#pragma unroll
            for (int u = 0; u < PREP_UD; ++u) {
                const int tt = t0 + 32 * u + lane;
                const int cnt = tt < NT ? min(static_cast<int>(a[u][0].x), cap) : 0;
                int inc = cnt;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int x = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += x;
                }
                uint32_t* dst = glr + base + inc - cnt;
                auto put = [&](uint32_t w, int e) {
                    const uint32_t n = w & 0xFFFFu;
                    atomicOr(&mask[n >> 5], 1u << (n & 31));
                    dst[e] = w;
                };
                // entries 0..14 from the four registers (word 1 + e of the tile), the rest by further loads
#pragma unroll
                for (int e = 0; e < 15; ++e) {
                    const int wi = 1 + e;
                    const uint4& q4 = a[u][wi >> 2];
                    const uint32_t w = (wi & 3) == 0 ? q4.x : (wi & 3) == 1 ? q4.y : (wi & 3) == 2 ? q4.z : q4.w;
                    if (e < cnt) put(w, e);
                }
                if (tt < NT)
                    for (int e4 = 16; e4 <= cnt; e4 += 4) {
                        const uint4 v4 = pld<OV>(reinterpret_cast<const uint4*>(row + static_cast<int64_t>(tt) * WPT + e4));
                        put(v4.x, e4 - 1);
                        if (e4 + 1 <= cnt) put(v4.y, e4);
                        if (e4 + 2 <= cnt) put(v4.z, e4 + 1);
                        if (e4 + 3 <= cnt) put(v4.w, e4 + 2);
                    }
                base += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
    }
    // PREP_RR rows per warp in flight (their tile loads issued together)
    for (int r = warp; r < ((dense_block || dense_rows) ? 0 : rows); r += PREP_RR * PREP_NW) {
        const uint32_t* rowp[PREP_RR];
        uint32_t* glp[PREP_RR];
        int base[PREP_RR];
#pragma unroll
        for (int q = 0; q < PREP_RR; ++q) {
            const int rq = r + q * PREP_NW;
            rowp[q] = rq < rows ? tw + static_cast<int64_t>(s_prow[rq]) * RW : nullptr;
            glp[q] = um.glist + prow(rq) * um.lmax;
            base[q] = 0;
        }
        for (int t0 = 0; t0 < NT; t0 += 32 * PREP_U) {
            // count + entries 0..6 (two 16-byte loads) issued for every tile up front: most tiles need nothing more
            uint4 a[PREP_RR][PREP_U], a2[PREP_RR][PREP_U];
#pragma unroll
            for (int q = 0; q < PREP_RR; ++q)
#pragma unroll
                for (int u = 0; u < PREP_U; ++u) {
                    const int tt = t0 + 32 * u + lane;
                    a[q][u] = make_uint4(0, 0, 0, 0);
                    a2[q][u] = make_uint4(0, 0, 0, 0);
                    if (tt < NT && rowp[q]) {
                        const uint32_t* blk = rowp[q] + static_cast<int64_t>(tt) * WPT;
                        if ((WPT & 3) == 0) {
                            a[q][u] = pld<OV>(reinterpret_cast<const uint4*>(blk));
                            if (WPT >= 8) a2[q][u] = pld<OV>(reinterpret_cast<const uint4*>(blk + 4));
                        } else {
                            a[q][u].x = pld<OV>(blk);
                        }
                    }
                }
#pragma unroll
            for (int q = 0; q < PREP_RR; ++q)
#pragma unroll
                for (int u = 0; u < PREP_U; ++u) {
                    const int tt = t0 + 32 * u + lane;
                    const int cnt = min(static_cast<int>(a[q][u].x), cap);
                    int inc = cnt;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const int x = __shfl_up_sync(0xffffffffu, inc, d);
                        if (lane >= d) inc += x;
                    }
                    uint32_t* dst = glp[q] + base[q] + inc - cnt;
                    auto put = [&](uint32_t w, int e) {
                        const uint32_t n = w & 0xFFFFu;
                        atomicOr(&mask[n >> 5], 1u << (n & 31));
                        dst[e] = w;
                    };
                    if (tt < NT && rowp[q]) {
                        const uint32_t* blk = rowp[q] + static_cast<int64_t>(tt) * WPT;
                        if ((WPT & 3) == 0) {
                            if (cnt >= 1) put(a[q][u].y, 0);
                            if (cnt >= 2) put(a[q][u].z, 1);
                            if (cnt >= 3) put(a[q][u].w, 2);
                            if (cnt >= 4) put(a2[q][u].x, 3);
                            if (cnt >= 5) put(a2[q][u].y, 4);
                            if (cnt >= 6) put(a2[q][u].z, 5);
                            if (cnt >= 7) put(a2[q][u].w, 6);
                            for (int e4 = 8; e4 <= cnt; e4 += 4) {
                                const uint4 v4 = pld<OV>(reinterpret_cast<const uint4*>(blk + e4));
                                put(v4.x, e4 - 1);
                                if (e4 + 1 <= cnt) put(v4.y, e4);
                                if (e4 + 2 <= cnt) put(v4.z, e4 + 1);
                                if (e4 + 3 <= cnt) put(v4.w, e4 + 2);
                            }
                        } else {
                            for (int e = 0; e < cnt; ++e) put(pld<OV>(blk + 1 + e), e);
                        }
                    }
                    base[q] += __shfl_sync(0xffffffffu, inc, 31);
                }
        }
    }
    prep_sync();
    asm volatile("bar.arrive 2, %0;" ::"n"(PREP_THREADS) : "memory");  // release the X copy (warp 15)
    if (trace && t == 0) trace[8 * lid + 2] = gtimer();
    uint32_t* gmask = um.umask + static_cast<int64_t>(b) * NW;
    int* flag = pctr + PrepCtr::arrive + NB + b;
    bool builder = true;
    if (split > 1) {
        for (int w = t; w < NW; w += PREP_WORK)
            if (mask[w] && !dense_block) atomicOr(gmask + w, mask[w]);
        __threadfence();
        prep_sync();
        if (t == 0) s_last = atomicAdd(pctr + PrepCtr::arrive + b, 1) == split - 1;
        prep_sync();
        builder = s_last != 0;
        if (builder) {
            __threadfence();
            for (int w = t; w < NW; w += PREP_WORK) mask[w] = dense_block ? 0xFFFFFFFFu : __ldcg(gmask + w);
            prep_sync();
        }
    } else {
        if (dense_block)
            for (int w = t; w < NW; w += PREP_WORK) mask[w] = 0xFFFFFFFFu;
        prep_sync();
    }

    if (builder) {
        // ---------------------------------------------------------------- 4. U_b
        for (int pass = 0; pass < 2; ++pass) {
            const int seg = (NW + PREP_WORK - 1) / PREP_WORK;
            const int wa = t * seg, wb = min(NW, wa + seg);
            int local = 0;
            for (int w = wa; w < wb; ++w) local += __popc(mask[w]);
            int incl = local;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += u;
            }
            if (lane == 31) wsum[warp] = incl;
            prep_sync();
            if (warp == 0) {
                const int x = lane < PREP_NW ? wsum[lane] : 0;
                int sc = x;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, sc, off);
                    if (lane >= off) sc += u;
                }
                if (lane < PREP_NW) wsum[lane] = sc - x;
                if (lane == PREP_NW - 1) wsum[PREP_NW] = sc;
            }
            prep_sync();
            int run = wsum[warp] + incl - local;
            for (int w = wa; w < wb; ++w) {
                woff[w] = run;
                run += __popc(mask[w]);
            }
            prep_sync();
            if (pass == 0 && wsum[PREP_NW] >= dense_units && wsum[PREP_NW] < N) {
                for (int w = t; w < NW; w += PREP_WORK) mask[w] = 0xFFFFFFFFu;
                prep_sync();
                continue;
            }
            break;
        }
        const int total = wsum[PREP_NW];
        const int padded = max(64, (total + 63) & ~63);
        int32_t* ul = um.ulist + static_cast<int64_t>(b) * N;
        for (int w = t; w < NW; w += PREP_WORK) {
            uint32_t m = mask[w];
            int pos = woff[w];
            gmask[w] = m;
            um.uwoff[static_cast<int64_t>(b) * NW + w] = pos;
            while (m) {
                const int bit = __ffs(m) - 1;
                m &= m - 1;
                ul[pos++] = (w << 5) + bit;
            }
        }
        for (int j = total + t; j < padded; j += PREP_WORK) ul[j] = 0;
        if (t == 0) {
            um.ulen[b] = padded;
            um.utot[b] = total;
            um.udense[b] = (dense_units <= N && total == N) ? 1 : 0;
        }
        __threadfence();
        prep_sync();
        if (t == 0) {
            if (split > 1) atomicExch(flag, 1);  // release the other parts of the block (after the fence)
            s_last = atomicAdd(pctr + PrepCtr::built, 1) == NB - 1;
        }
        prep_sync();
        if (s_last) {  // the last block built: the UP work list from every block's ulen
            __threadfence();
            const int ug = up_group & 0xFFFF, uflags = up_group >> 16;  // flags: 1 fraction order, 2 snake
            union_scan_body<PREP_WORK>(um, NB, ug, wsum, goff, PrepSync(), (uflags & 1) != 0, (uflags & 2) != 0);
        }
    } else {
        // wait for the block's builder (it is running: it arrived after this part), then its mask and offsets
        if (t == 0) {
            while (atomicAdd(flag, 0) == 0) __nanosleep(200);
            __threadfence();
        }
        prep_sync();
        for (int w = t; w < NW; w += PREP_WORK) {
            mask[w] = __ldcg(gmask + w);
            woff[w] = __ldcg(um.uwoff + static_cast<int64_t>(b) * NW + w);
        }
        prep_sync();
    }

    if (trace && t == 0) trace[8 * lid + 3] = gtimer();
    if (!gate_lists) return;  // non-gated variant: the union only (H_c is scattered from the TwELL by another kernel)
    // -------------------------------------------------------------------- 5. gate lists of the part's rows
    const bool udense = __ldcg(um.udense + b) != 0;  // identity union: the UP epilogue reads the TwELL directly
    const int nch = um.nchunk;
    int32_t* cc = ccnt + warp * (nch + 1);
    for (int r = warp; r < PR; r += PREP_NW) {
        const int64_t i = prow(r);  // pi-ordered row
        for (int c = lane; c <= nch; c += 32) cc[c] = 0;
        __syncwarp();
        if (r < rows && !udense) {
            // the stashed (unit | gate) words -> (union position << 16 | gate), ascending either way; written by
            // this warp in step 3 (plain loads: not the read-only path)
            uint32_t* gl = um.glist + i * um.lmax;
            const int n_r = s_rcnt[r];
            constexpr int B5 = 8;  // loads in flight per lane
            for (int e0 = 0; e0 < n_r; e0 += 32 * B5) {
                uint32_t w[B5];
#pragma unroll
                for (int q = 0; q < B5; ++q) {
                    const int e = e0 + 32 * q + lane;
                    w[q] = e < n_r ? __ldcg(gl + e) : 0u;
                }
#pragma unroll
                for (int q = 0; q < B5; ++q) {
                    const int e = e0 + 32 * q + lane;
                    if (e < n_r) {
                        const int n = static_cast<int>(w[q] & 0xFFFFu);
                        const int j = woff[n >> 5] + __popc(mask[n >> 5] & ((1u << (n & 31)) - 1u));
                        gl[e] = (static_cast<uint32_t>(j) << 16) | (w[q] >> 16);
                        atomicAdd(&cc[j >> 8], 1);
                    }
                }
            }
        }
        __syncwarp();
        if (!udense) {
            uint16_t* co = um.coff + i * (nch + 1);
            int carry = 0;
            for (int c0 = 0; c0 <= nch; c0 += 32) {
                const int c = c0 + lane;
                const int x = c <= nch ? cc[c] : 0;
                int inc = x;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += u;
                }
                if (c <= nch) co[c] = static_cast<uint16_t>(carry + inc - x);
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
        __syncwarp();
    }
    if (trace) {
        prep_sync();
        if (t == 0) trace[8 * lid + 4] = gtimer();
    }
}

}  // namespace sffn
