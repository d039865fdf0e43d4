// gemm_union_pair.cuh — CTA-pair (cluster of 2, tcgen05 cta_group::2) variant of the union up/down GEMMs
// (gemm_union.cuh).  Union blocks are 256 token rows (UnionMeta::brows == 256): one pair tile is M = 256 rows
// (128 per CTA, each CTA's A rows by TMA) x N = up to 256 union positions (UP) / 256 output columns (DOWN), and
// each CTA gathers only HALF of the B operand (N/2 weight rows / columns), the leader issuing M=256 MMAs that read
// both CTAs' shared memory.  Per SM this halves the gathered bytes per MMA FLOP and cuts the operand stream from
// 48 KB to 32 KB per k-block (same MMA work), at the price of unions over 256 rows instead of 128.
//
// Cross-CTA protocol (both CTAs run identical role loops over the same tile sequence):
//   tile ring   : the leader's warp 0 claims tiles (atomic counter) and publishes each into BOTH CTAs' SMEM ring
//                 (st.shared::cluster + remote mbarrier arrive); every reader of both CTAs releases a slot by
//                 arriving on the LEADER's sempty barrier.
//   operands    : A tiles by TMA (.cta_group::2: completion on the leader's full barrier, expect_tx by the leader
//                 for both CTAs); B rows by 16-byte cp.async into the CTA's own SMEM, completion on a CTA-local
//                 gfull barrier (cp.async.mbarrier.arrive.noinc), relayed by one thread per CTA (warp 3) to the
//                 leader's full barrier after a generic->async proxy fence.
//   stage reuse : tcgen05.commit multicast arrives on both CTAs' empty barriers.
//   accumulators: commit multicast on both CTAs' tfull; every epilogue warp of both CTAs arrives on the leader's
//                 tempty.
#pragma once
#include "gemm_union.cuh"

namespace sffn {


constexpr int UGP_B_BYTES = GEMM_B_BYTES / 2;                 // this CTA's half of the B tile (16 KB)
constexpr int UGP_STAGE = GEMM_A_BYTES + UGP_B_BYTES;         // 32 KB
constexpr int UGP_STAGES = 6;
constexpr int UGP_SMEM = 1024 + UGP_STAGES * UGP_STAGE + 4 * UG_EWB + 1024;
constexpr int UGP_READERS = 2 * (UG_GW + 6);  // per CTA: gather warps + 4 epilogue + relay + (leader MMA | peer A producer)
static_assert(UGP_SMEM <= GEMM_SMEM_LIMIT, "pair union GEMM shared memory");

template <bool UP>
__global__ void __launch_bounds__(UG_THREADS, 1)
    union_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ CUtensorMap tmOut, const UnionArgs args) {
    constexpr int S = UGP_STAGES;
    constexpr int BM2 = 2 * GEMM_BM;  // rows per pair tile
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stA = smem;
    uint8_t* stB = smem + S * GEMM_A_BYTES;
    uint8_t* epi = stB + S * UGP_B_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(epi + 4 * UG_EWB);  // [S] leader: A bytes + 2 relay arrivals
    uint64_t* gfull = full + S;                                        // [S] local: cp.async completion
    uint64_t* empty = gfull + S;                                       // [S]
    uint64_t* tfull = empty + S;                                       // [2]
    uint64_t* tempty = tfull + 2;                                      // [2] leader
    uint64_t* sfull = tempty + 2;                                      // [UG_RING]
    uint64_t* sempty = sfull + UG_RING;                                // [UG_RING] leader
    int* sched = reinterpret_cast<int*>(sempty + UG_RING);             // [UG_RING]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sched + UG_RING);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int N = args.N;
    const int NB = args.NB;
    const int num_tiles = UP ? __ldg(args.um.chunk_off) : NB * args.NJ;
    const int nk_up = (args.K + GEMM_BK - 1) / GEMM_BK;
    const uint32_t rank = cluster_ctarank();

    if (threadIdx.x == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmOut);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 3);  // leader producer (expect_tx) + the two CTAs' relays
            mbar_init(&gfull[i], UG_GATHER);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8);
        }
        for (int i = 0; i < UG_RING; ++i) {
            mbar_init(&sfull[i], 1);
            mbar_init(&sempty[i], UGP_READERS);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
    tc_fence_before();
    cluster_sync();  // barriers of both CTAs initialised before any remote arrive / store
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t full_leader = mapa_shared(full, 0);
    const uint32_t sempty_leader = mapa_shared(sempty, 0);
    const uint32_t tempty_leader = mapa_shared(tempty, 0);

    auto next_tile = [&](int& ridx, uint32_t& rphase, bool arrive_lane) -> int {
        mbar_wait_cluster(&sfull[ridx], rphase);
        const int t = *reinterpret_cast<volatile int*>(&sched[ridx]);
        if (arrive_lane) mbar_arrive_cluster(sempty_leader + 8u * static_cast<uint32_t>(ridx));
        if (++ridx == UG_RING) {
            ridx = 0;
            rphase ^= 1;
        }
        return t;
    };
    auto tile_info = [&](int tile, int& b, int& cj, int& len) {
        if (UP) {
            const int v = __ldg(args.um.tiles + tile);
            b = v >> 8;
            cj = v & 255;
            len = min(256, __ldg(args.um.ulen + b) - 256 * cj);
        } else {
            const int G = args.group;
            const int per = G * args.NJ;
            const int grp = tile / per;
            const int gb = min(G, NB - grp * G);
            const int in = tile - grp * per;
            b = grp * G + in % gb;
            cj = in / gb;
            len = __ldg(args.um.ulen + b);
        }
    };

    if (warp == 0) {
        // ------------------------------------------------------------ tile claims (leader) + A operand by TMA
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            int widx = 0;
            uint32_t wphase = 0;
            int ridx = 0;
            uint32_t rphase = 0;
            for (;;) {
                int tile;
                if (rank == 0) {
                    mbar_wait_cluster(&sempty[widx], wphase ^ 1);
                    tile = atomicAdd(args.counter, 1);
                    if (tile >= num_tiles) tile = -1;
                    sched[widx] = tile;
                    st_cluster_u32(mapa_shared(&sched[widx], 1), static_cast<uint32_t>(tile));
                    mbar_arrive(&sfull[widx]);
                    mbar_arrive_cluster(mapa_shared(&sfull[widx], 1));
                    if (++widx == UG_RING) {
                        widx = 0;
                        wphase ^= 1;
                    }
                } else {
                    tile = next_tile(ridx, rphase, true);
                }
                if (tile < 0) break;
                int b, cj, len;
                tile_info(tile, b, cj, len);
                const int nk = UP ? nk_up : len / GEMM_BK;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait_relaxed(&empty[stage], phase ^ 1);
                    if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * GEMM_A_BYTES);
                    tma_load_2d_pair(stA + stage * GEMM_A_BYTES, &tmA, full_leader + 8u * static_cast<uint32_t>(stage),
                                     kb * GEMM_BK, b * BM2 + static_cast<int>(rank) * GEMM_BM, pol);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 3) {
        // ------------------------------------------------------------ relay: local gather completion -> leader
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int ridx = 0;
            uint32_t rphase = 0;
            for (;;) {
                const int tile = next_tile(ridx, rphase, true);
                if (tile < 0) break;
                int b, cj, len;
                tile_info(tile, b, cj, len);
                const int nk = UP ? nk_up : len / GEMM_BK;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait_relaxed(&gfull[stage], phase);  // per stage: no L1 invalidation
                    fence_async_smem();  // cp.async (generic proxy) writes -> tensor-core reads (async proxy)
                    mbar_arrive_remote(full_leader + 8u * static_cast<uint32_t>(stage));
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp >= 8) {
        // ------------------------------------------------------------ B operand: this CTA's half, gathered
        const int gw = warp - 8;
        const int c8 = lane & 7;
        int stage = 0;
        uint32_t phase = 0;
        int ridx = 0;
        uint32_t rphase = 0;
        for (;;) {
            const int tile = next_tile(ridx, rphase, lane == 0);
            if (tile < 0) break;
            int b, cj, len;
            tile_info(tile, b, cj, len);
            const int32_t* ul = args.um.ulist + static_cast<int64_t>(b) * N;
            if (UP) {
                // rows rr = 4 UG_GW i + 4 gw + sub of this CTA's half (half = len/2 chunk positions)
                constexpr int NP = 128 / (4 * UG_GW);
                const int sub = lane >> 3;
                const int half = len >> 1;
                const int p0 = 256 * cj + static_cast<int>(rank) * half;
                int nidx[NP];
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const int rr = 4 * UG_GW * i + 4 * gw + sub;
                    nidx[i] = rr < half ? __ldg(ul + p0 + rr) : -1;
                }
                for (int kb = 0; kb < nk_up; ++kb) {
                    mbar_wait_relaxed(&empty[stage], phase ^ 1);
                    const uint32_t dst = smem_u32(stB + stage * UGP_B_BYTES);
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        const int rr = 4 * UG_GW * i + 4 * gw + sub;
                        if (nidx[i] >= 0)
                            cp_async16(dst + rr * 128 + ((c8 ^ (rr & 7)) << 4),
                                       args.wsrc + static_cast<int64_t>(nidx[i]) * args.K + kb * GEMM_BK + 8 * c8, 16);
                    }
                    cp_async_arrive_noinc(&gfull[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            } else {
                // k-block row r = 16 i + 2 gw + rsub, MN atom a (columns 256 cj + 128 rank + 64 a + 8 c8)
                constexpr int NP = 64 / (2 * UG_GW);
                const int a = (lane >> 3) & 1, rsub = lane >> 4;
                const int nk = len / GEMM_BK;
                const int col = cj * 256 + static_cast<int>(rank) * 128 + a * 64 + 8 * c8;
                const bool in = col < args.K;
                // union indices two k-blocks ahead (an L2 round trip is about one k-block of MMA time)
                int nidx[NP], n1[NP];
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    nidx[i] = __ldg(ul + 2 * UG_GW * i + 2 * gw + rsub);
                    n1[i] = __ldg(ul + (nk > 1 ? GEMM_BK : 0) + 2 * UG_GW * i + 2 * gw + rsub);
                }
                for (int kb = 0; kb < nk; ++kb) {
                    int nxt[NP];
                    const int kn = kb + 2 < nk ? kb + 2 : nk - 1;
#pragma unroll
                    for (int i = 0; i < NP; ++i) nxt[i] = __ldg(ul + kn * GEMM_BK + 2 * UG_GW * i + 2 * gw + rsub);
                    mbar_wait_relaxed(&empty[stage], phase ^ 1);
                    const uint32_t dst = smem_u32(stB + stage * UGP_B_BYTES) + a * 8192;
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        const int r = 2 * UG_GW * i + 2 * gw + rsub;
                        cp_async16(dst + r * 128 + ((c8 ^ (r & 7)) << 4),
                                   args.wsrc + static_cast<int64_t>(nidx[i]) * args.K + (in ? col : 0), in ? 16 : 0);
                    }
                    cp_async_arrive_noinc(&gfull[stage]);
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        nidx[i] = n1[i];
                        n1[i] = nxt[i];
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (leader only)
        if (lane == 0 && rank == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            int ridx = 0;
            uint32_t rphase = 0;
            for (;;) {
                const int tile = next_tile(ridx, rphase, true);
                if (tile < 0) break;
                int b, cj, len;
                tile_info(tile, b, cj, len);
                const int nk = UP ? nk_up : len / GEMM_BK;
                const uint32_t idesc = UP ? umma_idesc_bf16(BM2, len) : (umma_idesc_bf16(BM2, 256) | (1u << 16));
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + static_cast<uint32_t>(acc * GEMM_BN);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait_relaxed(&full[stage], phase);  // per stage: no L1 invalidation
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(stA + stage * GEMM_A_BYTES);
                    const uint32_t b0 = smem_u32(stB + stage * UGP_B_BYTES);
#pragma unroll
                    for (int k = 0; k < GEMM_BK / 16; ++k) {
                        const uint64_t bd = UP ? umma_desc_sw128(b0 + k * 32) : umma_desc_sw128_mn(b0 + k * 2048, 8192, 1024);
                        umma_f16_pair(d, umma_desc_sw128(a0 + k * 32), bd, idesc, (kb | k) != 0);
                    }
                    umma_commit_pair(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_pair(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue (both CTAs, own 128 rows)
        const int ew = warp - 4;
        uint8_t* stg = epi + ew * UG_EWB;
        int acc = 0;
        uint32_t acc_phase = 0;
        int ridx = 0;
        uint32_t rphase = 0;
        for (;;) {
            const int tile = next_tile(ridx, rphase, lane == 0);
            if (tile < 0) break;
            int b, cj, len;
            tile_info(tile, b, cj, len);
            const int row0 = b * BM2 + static_cast<int>(rank) * GEMM_BM + ew * 32;
            // UP: this row's gate entries of the chunk, loaded before waiting for the accumulator
            int e0 = 0, e1 = 0;
            const uint32_t* gl = nullptr;
            uint32_t gpre[UG_GPRE];
            if constexpr (UP) {
                const int64_t prow = static_cast<int64_t>(row0) + lane;  // pi-ordered row (H_c row)
                gl = args.um.glist + prow * args.um.lmax;
                const uint16_t* co = args.um.coff + prow * (args.um.nchunk + 1);
                e0 = __ldg(co + cj);
                e1 = __ldg(co + cj + 1);
#pragma unroll
                for (int i = 0; i < UG_GPRE; ++i) gpre[i] = e0 + i < e1 ? __ldg(gl + e0 + i) : 0u;
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t tb = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * GEMM_BN);
            const uint32_t release = tempty_leader + 8u * static_cast<uint32_t>(acc);
            if constexpr (UP) {
                const int p0 = 256 * cj;
#pragma unroll 1
                for (int h = 0; h < 2 && 128 * h < len; ++h) {
                    const int nbox = min(2, (len - 128 * h) / 64);
                    if (lane == 0) bulk_wait_read0();
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < 2; ++q)
#pragma unroll
                        for (int c16 = 0; c16 < 8; ++c16)
                            *reinterpret_cast<uint4*>(stg + q * 4096 + lane * 128 + ((c16 ^ (lane & 7)) << 4)) =
                                make_uint4(0, 0, 0, 0);  // XOR: conflict-free 16-byte stores
                    auto put_g = [&](uint32_t w) {
                        const int j = static_cast<int>(w >> 16) - p0 - 128 * h;
                        if (j >= 0 && j < 128)
                            *reinterpret_cast<uint16_t*>(stg + (j >> 6) * 4096 + sw128_off(lane, j & 63)) =
                                static_cast<uint16_t>(w & 0xFFFFu);
                    };
#pragma unroll
                    for (int i = 0; i < UG_GPRE; ++i)
                        if (e0 + i < e1) put_g(gpre[i]);
                    for (int e = e0 + UG_GPRE; e < e1; ++e) put_g(__ldg(gl + e));
#pragma unroll 1
                    for (int q32 = 0; q32 < 2 * nbox; ++q32) {
                        uint32_t v[32];
                        tmem_ld32(tb + 128 * h + 32 * q32, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int p = 0; p < 16; ++p) {
                            const int c = 32 * q32 + 2 * p;
                            uint32_t* sp = reinterpret_cast<uint32_t*>(stg + (c >> 6) * 4096 + sw128_off(lane, c & 63));
                            const uint32_t gg = *sp;
                            if (gg) {
                                const float g0 = __uint_as_float(gg << 16), g1 = __uint_as_float(gg & 0xFFFF0000u);
                                const float h0 = (gg & 0xFFFFu) ? g0 * __uint_as_float(v[2 * p]) : 0.0f;
                                const float h1 = (gg >> 16) ? g1 * __uint_as_float(v[2 * p + 1]) : 0.0f;
                                *sp = pack_bf16x2(h0, h1);
                            }
                        }
                    }
                    if (h == 1 || 128 * (h + 1) >= len) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(release);
                    }
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        for (int q = 0; q < nbox; ++q) tma_store_2d(&tmOut, stg + q * 4096, p0 + 128 * h + 64 * q, row0);
                        bulk_commit();
                    }
                }
            } else {
                // DOWN: rows were processed in pi order; row i of the tile goes to Y[perm[row0 + i]].  Stage
                // 32 rows x 128 columns (bf16) per half in SMEM (conflict-free rotated 16-byte stores), then the
                // warp writes two rows per instruction with coalesced 16-byte global stores (LSU, not per-row
                // bulk copies: those were 256 small TMA requests per tile competing with the A-tile loads).
                uint32_t* srow = reinterpret_cast<uint32_t*>(stg) + lane * 64;
                const int prow_l = row0 + lane;
                const int64_t yrow_l = prow_l < args.M ? static_cast<int64_t>(__ldg(args.perm + prow_l)) : -1;
#pragma unroll 1
                for (int half = 0; half < 2; ++half) {
                    const int c0 = cj * 256 + half * 128;
                    const int nc = min(128, args.K - c0);
#pragma unroll 1
                    for (int ch = 0; ch < 4; ++ch) {
                        uint32_t v[32];
                        tmem_ld32(tb + half * 128 + ch * 32, v);
                        tmem_wait_ld();
                        st_row32_bf16(srow + ch * 16, v, lane);
                    }
                    if (half == 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(release);
                    }
                    __syncwarp();
                    const int chunk = lane & 15;
#pragma unroll 4
                    for (int it = 0; it < 16; ++it) {
                        const int r = 2 * it + (lane >> 4);
                        const int64_t yrow = __shfl_sync(0xffffffffu, yrow_l, r);
                        const uint4 val = *reinterpret_cast<const uint4*>(stg + r * 256 + chunk * 16);
                        if (yrow >= 0 && chunk * 8 < nc)
                            *reinterpret_cast<uint4*>(args.Y + yrow * args.K + c0 + chunk * 8) = val;
                    }
                    __syncwarp();  // staging rows read before the next half overwrites them
                }
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (UP) {
            if (lane == 0) bulk_wait0();
        }
    }

    __syncwarp();
    tc_fence_before();
    cluster_sync();  // remote arrivals / stores and the leader's MMAs into the peer's TMEM are finished
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair(tmem_base, 512);
    }
}

}  // namespace sffn
