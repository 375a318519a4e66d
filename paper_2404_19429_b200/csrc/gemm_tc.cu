// gemm_tc.cu -- the expert GEMMs on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// "Each expert processes the C received tokens": per expert an FFN,
// whose token count per (expert, chunk) is irregular and known only on the device after the
// gate (fig:proposed_partition).  One persistent, warp-specialised kernel serves all
// six expert GEMMs of a fwd+bwd step:
//   M-grouped (rows = tokens of a group, 128-row aligned):      fc1 (act epilogue: H and
//     act'(A)), fc2, dfc2 (epilogue multiplies act'(A)), dfc1
//   K-grouped (reduction over a group's token rows, fp32 out):  dW2 = dO^T H, dW1 = dA^T X
// Operands are TMA-loaded with 128-byte swizzle into a shared-memory ring; a single elected
// thread issues tcgen05.mma (kind::f16, bf16 in, fp32 accumulate) into one of two TMEM
// accumulators (BN fp32 columns each), so the epilogue drains tile i while the tensor core
// computes tile i+1.  With CG = 2 a cluster of two CTAs (one TPC) computes a 256 x BN tile
// with tcgen05.mma.cta_group::2: each CTA loads its own 128 rows of A and half of B, the
// leader CTA issues the MMAs and commits to both CTAs' barriers (halves the operand traffic
// per SM).  Operands may be K-major or MN-major (the dX GEMMs read W1/W2 and the dW GEMMs
// read both activations transposed in place -- no transposition pass over HBM).
// bf16 epilogues stage each warp's 32x32 sub-tile in 64B-swizzled shared memory and write it
// with TMA bulk-tensor stores; the act'(A) operand of dfc2 arrives by TMA the same way.
//
// Roles (384 threads):  warp 0 TMA producer | warp 1 MMA issuer | warp 2 TMEM allocator |
//                       warp 3 idle | warps 4-11 epilogue (TMEM lanes 32*(w%4), column half
//                       (w-4)/4).
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace lancet {
namespace tc {

constexpr int BM = 128, BK = 64, UMMA_K = 16;
constexpr int kThreads = 384;            // 4 control warps + 8 epilogue warps
constexpr int kEpiWarps = 8;
constexpr int kMaxGroups = 128;                 // group tables cached in shared memory
constexpr uint32_t A_STAGE = BM * BK * 2;                 // 16 KiB
constexpr uint32_t kWarpStage = 4096;                     // per epilogue warp: out0 | (out1 or act'(A))
constexpr uint32_t kBarBytes = 256;                       // mbarriers + TMEM address
constexpr size_t kSmemLimit = 232448;                     // 227 KiB opt-in per block

template <int BN, bool A_MN, int CG>
struct Cfg {
    static constexpr bool kStaged = !A_MN;                // M-grouped: bf16 out via TMA store
                                                          // (K-grouped: fp32 out, also TMA)
    static constexpr uint32_t B_STAGE = BN * BK * 2 / CG; // this CTA's share of B
    static constexpr size_t kEpi = (size_t)kEpiWarps * kWarpStage;
    static constexpr size_t kFixed = 1024 + kEpi + kBarBytes + sizeof(int) * (3 * kMaxGroups + 1);
    static constexpr int STAGES_FIT = (int)((kSmemLimit - kFixed) / (A_STAGE + B_STAGE));
#ifdef LANCET_EXP_STAGES
    static constexpr int STAGES = STAGES_FIT > LANCET_EXP_STAGES ? LANCET_EXP_STAGES : STAGES_FIT;
#else
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
#endif
    static constexpr size_t kRing = (size_t)STAGES * (A_STAGE + B_STAGE);
    static constexpr size_t kSmem = kFixed + kRing;
};

struct Params {
    int mode, n_groups, gpw, n_weights, epi, act, accumulate;
    int M, N, K;
    const int* grp_rows;
    const int* grp_off;
    void* C;
    long ldc, c_group_stride;
    ChunkSync cs;
};

// ---- device-side chunk pipeline (ChunkSync, push mode) ----------------------------------
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// producer: every rank's rows of chunk ch have landed (then the TMA loads may read them)
__device__ __forceinline__ void chunk_wait(const ChunkSync& cs, int ch) {
    const uint32_t want = cs.seq[0];
    const uint32_t* f = cs.wait_flags + (long)ch * cs.wait_chunk_stride;
    const unsigned long long t0 = gtimer();
    for (int r = 0; r < cs.ranks; ++r) {
        unsigned ns = 32;
        while (ld_acquire_sys_u32(f + r) < want) {
            if (*reinterpret_cast<volatile uint32_t*>(cs.err) != 0) return;
            if (gtimer() - t0 > cs.timeout_ns) {
                atomicCAS(cs.err, 0u, cs.err_code | ((uint32_t)(ch & 0xFFFF) << 8) | (uint32_t)r);
                return;
            }
            __nanosleep(ns);
            if (ns < 512) ns *= 2;
        }
    }
    // the rows were written by other agents (generic proxy); the TMA loads are async proxy
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
template <int BN, bool A_MN, bool B_MN, int CG>
__device__ __forceinline__ constexpr uint32_t instr_desc() {
    // c_format F32 [4,6) | a_format BF16 [7,10) | b_format BF16 [10,13) | a_major [15] |
    // b_major [16] | N>>3 [17,23) | M>>4 [24,29)   (M = 128 per CTA, 256 per CTA pair)
    return (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16) |
           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((BM * CG) >> 4) << 24);
}

__device__ __forceinline__ void decode_tile(int tile, const int* tstart, int ng, int ntn, int& g, int& mt, int& nt) {
    int lo = 0, hi = ng - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tstart[mid] <= tile) lo = mid;
        else hi = mid - 1;
    }
    g = lo;
    const int local = tile - tstart[g];
    mt = local / ntn;
    nt = local % ntn;
}

// byte offset of 16-byte chunk j of row r in a [32 rows][64 B] box stored with SWIZZLE_64B
__device__ __forceinline__ uint32_t sw64(int r, int j) { return r * 64 + ((j ^ ((r >> 1) & 3)) << 4); }

template <int BN, bool A_MN, bool B_MN, int CG, int MC>
__global__ void __launch_bounds__(kThreads, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
               const __grid_constant__ CUtensorMap tmX, Params p)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    using CF = Cfg<BN, A_MN, CG>;
    constexpr int STAGES = CF::STAGES;
    constexpr uint32_t B_STAGE = CF::B_STAGE;
    constexpr uint32_t TMEM_COLS = 2 * BN;
    constexpr int BNC = BN / CG;                          // B rows (N) loaded by this CTA
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_STAGE;
    uint8_t* sEpi = smem + CF::kRing;
    uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + CF::kEpi);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* abar = tempty + 2;                       // [kEpiWarps] aux-load barriers
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(abar + kEpiWarps);
    int* tstart = reinterpret_cast<int*>(sEpi + CF::kEpi + kBarBytes);   // [n_groups + 1]
    int* srows = tstart + kMaxGroups + 1;              // group tables cached from global memory
    int* soff = srows + kMaxGroups;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // MC pairs of a cluster share one A tile (TMA multicast) and compute MC adjacent N tiles:
    // "super tiles" of MC * BN columns; pair pp takes n tile ntp * MC + pp
    // ragged N / K / M: the tile counts round up; TMA zero-fills the loads past the tensor and
    // clips the stores to it, so the extra rows / columns never reach memory
    const int ntn = ceil_div(p.N, BN * MC);
    const uint32_t crank = CG * MC > 1 ? cta_rank() : 0;
    const uint32_t rank = CG == 2 ? (crank & 1) : 0;    // CTA within the pair
    const int pp = (int)(crank / CG);                   // pair within the cluster
    const uint32_t lead_rank = crank - rank;            // cluster rank of the pair leader
    const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pp));
    const bool leader = rank == 0;
    const int cluster = blockIdx.x / (CG * MC), n_clusters = gridDim.x / (CG * MC);
    constexpr int MT = BM * CG;                        // rows of A per (pair) tile

    if (threadIdx.x == 0) {
        int acc = 0;
        for (int g = 0; g < p.n_groups; ++g) {
            tstart[g] = acc;
            srows[g] = p.grp_rows[g];
            soff[g] = p.grp_off[g];
            const int mt = p.mode == GEMM_M_GROUPED ? ceil_div(srows[g], MT) : ceil_div(p.M, MT);
            acc += mt * ntn;
        }
        tstart[p.n_groups] = acc;
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        tma_prefetch(&tmC);
        if (CF::kStaged) {
            if (p.epi == EPI_ACT) tma_prefetch(&tmC2);
            if (p.epi == EPI_DACT) tma_prefetch(&tmX);
        }
    }
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], MC); }
        for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], kEpiWarps * CG); }
        for (int i = 0; i < kEpiWarps; ++i) mbar_init(&abar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        if constexpr (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    tc_fence_before();
    if constexpr (CG * MC > 1) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int total = tstart[p.n_groups];

    if (warp == 0) {
        // ===================== TMA producer (each CTA loads its own rows) =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int ready_c = -1;
            for (int tile = cluster; tile < total; tile += n_clusters) {
                int g, mt, nt;
                decode_tile(tile, tstart, p.n_groups, ntn, g, mt, nt);
                if (p.cs.wait_flags && g / p.cs.gpc > ready_c) {     // chunk pipeline: rows landed?
                    ready_c = g / p.cs.gpc;
                    chunk_wait(p.cs, ready_c);
                }
                const int nb = (nt * MC + pp) * BN + (int)rank * BNC;   // this CTA's B rows / columns
                int num_kb, arow, brow;
                if (p.mode == GEMM_M_GROUPED) {
                    num_kb = ceil_div(p.K, BK);
                    arow = soff[g] + mt * MT + (int)rank * BM;
                    brow = ((g / p.gpw) % p.n_weights) * (B_MN ? p.K : p.N);
                } else {
                    num_kb = round_up(srows[g], kRowAlign) / BK;
                    arow = soff[g];
                    brow = soff[g];
                }
                const int m0 = mt * MT + (int)rank * BM;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_expect_tx(&full[stage], CG * (A_STAGE + B_STAGE));
                    uint8_t* a_dst = sA + stage * A_STAGE;
                    uint8_t* b_dst = sB + stage * B_STAGE;
#define LOAD(map, dst, c0, c1)                                                               \
    do {                                                                                     \
        if constexpr (CG == 1) tma_load_2d(map, &full[stage], dst, c0, c1);                  \
        else tma_load_2d_pair(map, &full[stage], dst, c0, c1);                               \
    } while (0)
                    if constexpr (MC == 2) {
                        // this CTA loads 64 of its 128 A rows and multicasts them to the CTA
                        // with the same rank in the other pair (which loads the other 64)
                        const uint16_t mc_mask = (uint16_t)((1u << rank) | (1u << (CG + rank)));
                        if (A_MN) tma_load_2d_pair_mc(&tmA, &full[stage], a_dst + pp * 8192, m0 + 64 * pp, arow + kb * BK, mc_mask);
                        else tma_load_2d_pair_mc(&tmA, &full[stage], a_dst + pp * 8192, kb * BK, arow + 64 * pp, mc_mask);
                    } else if (A_MN) {
#pragma unroll
                        for (int i = 0; i < BM / 64; ++i) LOAD(&tmA, a_dst + i * 8192, m0 + 64 * i, arow + kb * BK);
                    } else {
                        LOAD(&tmA, a_dst, kb * BK, arow);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int i = 0; i < BNC / 64; ++i) LOAD(&tmB, b_dst + i * 8192, nb + 64 * i, brow + kb * BK);
                    } else {
                        LOAD(&tmB, b_dst, kb * BK, brow + nb);
                    }
#undef LOAD
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (one thread of the leader CTA) =====================
        if (lane == 0 && leader) {
            constexpr uint32_t idesc = instr_desc<BN, A_MN, B_MN, CG>();
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = cluster; tile < total; tile += n_clusters, ++it) {
                int g, mt, nt;
                decode_tile(tile, tstart, p.n_groups, ntn, g, mt, nt);
                const int num_kb = p.mode == GEMM_M_GROUPED ? ceil_div(p.K, BK) : round_up(srows[g], kRowAlign) / BK;
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sA + stage * A_STAGE);
                    const uint32_t b_base = smem_u32(sB + stage * B_STAGE);
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k)
                        tc_mma<CG>(tmem_d, operand_desc<A_MN>(a_base, k), operand_desc<B_MN>(b_base, k), idesc,
                                   (kb | k) != 0 ? 1u : 0u);
                    // the stage is free once BOTH pairs have read it (its A half came from each)
                    tc_commit<CG>(&empty[stage], MC == 2 ? (uint16_t)0xF : pair_mask);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                tc_commit<CG>(&tfull[acc], pair_mask);
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue: 8 warps per CTA =====================
        // warp w may only touch TMEM lanes 32*(w%4)..; warps w and w+4 split the columns
        const int q = warp & 3;
        const int ew = warp - 4;
        const int half = ew >> 2;
        const int cc0 = half * (BN / 64), cc1 = cc0 + BN / 64;
        // staging (2 KiB = one 32x32 bf16 box, SWIZZLE_64B): out0 | out1 (ACT) or act'(A) (DACT)
        uint8_t* sO0 = sEpi + ew * kWarpStage;
        uint8_t* sO1 = sO0 + 2048;
        uint8_t* sX = sO0 + 2048;
        uint64_t* xbar = &abar[ew];
        uint32_t xphase = 0;
        int it = 0;
        for (int tile = cluster; tile < total; tile += n_clusters, ++it) {
            int g, mt, nt;
            decode_tile(tile, tstart, p.n_groups, ntn, g, mt, nt);
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            const bool has_k = p.mode == GEMM_M_GROUPED ? (p.K > 0) : (srows[g] > 0);
            const int n0 = (nt * MC + pp) * BN;
            if constexpr (CF::kStaged) {
                const int mrow = mt * MT + (int)rank * BM;                // first row of this CTA
                const int row0 = soff[g] + mrow + q * 32;                 // this warp's 32 rows
                // a pair tile may extend past the group's 128-aligned rows: skip that half
                const bool live = mrow < round_up(srows[g], kRowAlign);
                const bool dact = p.epi == EPI_DACT;
                if (live && dact && lane == 0) {                          // prefetch act'(A)
                    mbar_expect_tx(xbar, 2048);
                    tma_load_2d(&tmX, xbar, sX, n0 + cc0 * 32, row0);
                }
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
#ifdef LANCET_EXP_NO_EPI
                if (false) {
#else
                if (live) {
#endif
                    // chunk cc of this warp's columns: TMEM -> epilogue math -> staging -> TMA
                    auto chunk = [&](int cc, uint32_t (&v)[32]) {
                        if (!has_k) {                                   // uniform: empty reduction
#pragma unroll
                            for (int i = 0; i < 32; ++i) v[i] = 0u;
                        }
                        float f[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
                        if (dact) {
                            mbar_wait(xbar, xphase);
                            xphase ^= 1;
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                float a8[8];
                                unpack16<bf16>(*reinterpret_cast<const uint4*>(sX + sw64(lane, j)), a8);
#pragma unroll
                                for (int i = 0; i < 8; i += 2) {
                                    const float2 r = __fmul2_rn(make_float2(f[8 * j + i], f[8 * j + i + 1]),
                                                                make_float2(a8[i], a8[i + 1]));
                                    f[8 * j + i] = r.x;
                                    f[8 * j + i + 1] = r.y;
                                }
                            }
                            __syncwarp();
                        }
                        // the previous chunk's TMA stores must have read the staging buffers
#ifndef LANCET_EXP_NO_WAIT
                        if (lane == 0) bulk_wait_read0();
#endif
                        __syncwarp();
                        if (dact && cc + 1 < cc1 && lane == 0) {          // act'(A) of the next chunk
                            mbar_expect_tx(xbar, 2048);
                            tma_load_2d(&tmX, xbar, sX, n0 + (cc + 1) * 32, row0);
                        }
                        if (p.epi == EPI_ACT) {
                            float h[32], gr[32];
                            if (p.act == ACT_RELU) {                        // uniform branch
#pragma unroll
                                for (int i = 0; i < 32; ++i) {
                                    h[i] = f[i] > 0.f ? f[i] : 0.f;
                                    gr[i] = f[i] > 0.f ? 1.f : 0.f;
                                }
                            } else {
#pragma unroll
                                for (int i = 0; i < 32; i += 2) {
                                    float2 h2, g2;
// LANCET_EXP_*: experiment switches for A/B builds only (LANCET_BUILD_DEFS, DESIGN.md §7's
// power experiment); the library is never built with them.
#ifdef LANCET_EXP_NO_MATH
                                    h2 = make_float2(f[i], f[i + 1]); g2 = h2;
#else
                                    gelu_fwd_grad_fast2(make_float2(f[i], f[i + 1]), h2, g2);
#endif
                                    h[i] = h2.x; h[i + 1] = h2.y;
                                    gr[i] = g2.x; gr[i + 1] = g2.y;
                                }
                            }
#ifdef LANCET_EXP_NO_STS
                            {
                                uint32_t acc_ = 0;
#pragma unroll
                                for (int j = 0; j < 4; ++j) { const uint4 a_ = pack16<bf16>(h + 8 * j), b_ = pack16<bf16>(gr + 8 * j); acc_ ^= a_.x ^ a_.y ^ a_.z ^ a_.w ^ b_.x ^ b_.y ^ b_.z ^ b_.w; }
                                if (acc_ == 0x12345678u && lane == 40) *reinterpret_cast<uint32_t*>(sO0) = acc_;
                            }
#else
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                *reinterpret_cast<uint4*>(sO0 + sw64(lane, j)) = pack16<bf16>(h + 8 * j);
                                *reinterpret_cast<uint4*>(sO1 + sw64(lane, j)) = pack16<bf16>(gr + 8 * j);
                            }
#endif
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                *reinterpret_cast<uint4*>(sO0 + sw64(lane, j)) = pack16<bf16>(f + 8 * j);
                        }
                        fence_proxy_async();
                        __syncwarp();
                        if (lane == 0) {
#ifndef LANCET_EXP_NO_STORE
                            tma_store_2d(&tmC, sO0, n0 + cc * 32, row0);
#ifndef LANCET_EXP_NO_G
                            if (p.epi == EPI_ACT) tma_store_2d(&tmC2, sO1, n0 + cc * 32, row0);
#endif
#endif
                            bulk_commit();
                        }
                    };
                    // TMEM loads one chunk ahead of the math (cc1 - cc0 is even)
                    const uint32_t tbase = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
                    uint32_t va[32], vb[32];
#ifdef LANCET_EXP_NO_TMEM
#define TLD(addr, v) do { for (int i_ = 0; i_ < 32; ++i_) v[i_] = __float_as_uint((float)(lane + i_) * 0.01f + (float)(addr & 255)); } while (0)
#define TWAIT(v) do {} while (0)
#else
#define TLD(addr, v) tmem_ld32_issue(addr, v)
#define TWAIT(v) tmem_wait_ld(v)
#endif
                    TLD(tbase + cc0 * 32, va);
                    TWAIT(va);
#pragma unroll 1
                    for (int cc = cc0; cc < cc1; cc += 2) {
                        TLD(tbase + (cc + 1) * 32, vb);
                        chunk(cc, va);
                        TWAIT(vb);
                        if (cc + 2 < cc1) TLD(tbase + (cc + 2) * 32, va);
                        chunk(cc + 1, vb);
                        if (cc + 2 < cc1) TWAIT(va);
                    }
#undef TLD
#undef TWAIT
                }
            } else {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                // fp32 dW tile rows of this warp in the [n_groups][M][N] view of C (3D: a tile
                // past a ragged M is clipped at the group's end, never spills into the next)
                const int crow = mt * MT + (int)rank * BM + q * 32;
                uint8_t* sF = sEpi + ew * kWarpStage;            // 32 x 32 fp32 box, SWIZZLE_128B
#pragma unroll 1
                for (int cc = cc0; cc < cc1; ++cc) {
                    uint32_t v[32];
                    tmem_ld32(tmem_base + acc * BN + cc * 32 + ((uint32_t)(q * 32) << 16), v);
                    if (!has_k) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = 0u;
                    }
                    // the previous chunk's TMA store must have read the staging box
                    if (lane == 0) bulk_wait_read0();
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        *reinterpret_cast<uint4*>(sF + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                            make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        // accumulate: TMA reduce-add (old + new, one rounding: same as a
                        // read-add-write), else a plain store
                        if (p.accumulate) tma_reduce_add_3d(&tmC, sF, n0 + cc * 32, crow, g);
                        else tma_store_3d(&tmC, sF, n0 + cc * 32, crow, g);
                        bulk_commit();
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 1 || leader) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(&tempty[acc], lead_rank); // the leader's MMA waits on it
            }
        }
        if (lane == 0) bulk_wait0();
    }
    tc_fence_before();
    if constexpr (CG * MC > 1) cluster_sync();
    else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if constexpr (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}

template <int BN, bool A_MN, bool B_MN, int CG, int MC>
static int launch_cfg(const GemmArgs& a, int num_sms, cudaStream_t s)
{
    using CF = Cfg<BN, A_MN, CG>;
    static_assert(CF::STAGES >= 3, "shared-memory ring too shallow");
    static_assert(CF::kSmem <= kSmemLimit, "shared memory over the per-block limit");
    CUtensorMap ta, tb, tcm, tc2, tx;
    memset(&tcm, 0, sizeof(tcm));
    memset(&tc2, 0, sizeof(tc2));
    memset(&tx, 0, sizeof(tx));
    bool ok;
    if (A_MN) ok = make_map(&ta, a.A, a.M, a.a_rows, a.lda, 64, 64);
    else ok = make_map(&ta, a.A, a.K, a.a_rows, a.lda, 64, BM / MC);
    if (B_MN) ok = ok && make_map(&tb, a.B, a.N, a.b_rows, a.ldb, 64, 64);
    else ok = ok && make_map(&tb, a.B, a.K, a.b_rows, a.ldb, 64, BN / CG);
    if (CF::kStaged) {
        ok = ok && make_map(&tcm, a.C, a.N, a.c_rows, a.ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        if (a.epi == EPI_ACT) ok = ok && make_map(&tc2, a.C2, a.N, a.c_rows, a.ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        if (a.epi == EPI_DACT) ok = ok && make_map(&tx, a.aux, a.N, a.c_rows, a.ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    } else {   // fp32 C [n_groups][M][N] (3D, group stride c_group_stride)
        ok = ok && make_map3_f32(&tcm, a.C, a.N, a.M, a.n_groups, a.ldc, a.c_group_stride, 32, 32);
    }
    if (!ok) return -1;
    Params p{a.mode, a.n_groups, a.gpw, a.n_weights > 0 ? a.n_weights : (1 << 30), a.epi, a.act, a.accumulate,
             a.M, a.N, a.K, a.grp_rows, a.grp_off, a.C, a.ldc, a.c_group_stride, a.cs};
    constexpr size_t smem = CF::kSmem;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tc_gemm_kernel<BN, A_MN, B_MN, CG, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    // persistent grid: at most one CTA per SM (pairs on one TPC when CG == 2), never more
    // (pair) tiles than the upper bound of tiles
    long max_tiles;
    if (a.mode == GEMM_M_GROUPED) max_tiles = (long)ceil_div(a.max_rows, BM * CG) * a.n_groups * ceil_div(a.N, BN * MC);
    else max_tiles = (long)ceil_div(a.M, BM * CG) * ceil_div(a.N, BN * MC) * a.n_groups;
    // clusters of 4 cannot tile every GPC: cap the persistent grid at what is co-resident
    static int max_active = -1;
    if (max_active < 0) {
        cudaLaunchConfig_t q{};
        q.gridDim = dim3(num_sms);
        q.blockDim = dim3(kThreads);
        q.dynamicSmemBytes = smem;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = CG * MC;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        q.attrs = qa;
        q.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, tc_gemm_kernel<BN, A_MN, B_MN, CG, MC>, &q) != cudaSuccess || n <= 0)
            n = num_sms / (CG * MC);
        max_active = n;
    }
    const int clusters = (int)std::max<long>(1, std::min<long>(std::min(num_sms / (CG * MC), max_active), max_tiles));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(clusters * CG * MC);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = CG * MC;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = g_pdl ? 2 : 1;
    if (cudaLaunchKernelEx(&cfg, tc_gemm_kernel<BN, A_MN, B_MN, CG, MC>, ta, tb, tcm, tc2, tx, p) != cudaSuccess)
        return -1;
    return 1;
}

template <int BN, bool A_MN, bool B_MN>
static int launch_cg(const GemmArgs& a, int num_sms, cudaStream_t s)
{
    // CTA pairs need 256-row (pair) tiles: always possible for M-grouped GEMMs (a pair tile's
    // upper half past a group is computed but not stored), for K-grouped when M % 256 == 0
    const bool pair = a.mode == GEMM_M_GROUPED || a.M % (2 * BM) == 0;
    if (!pair) return launch_cfg<BN, A_MN, B_MN, 1, 1>(a, num_sms, s);
    // two pairs share each A tile (multicast) when the N tiles pair up
    if (a.multicast && a.N % (2 * BN) == 0) return launch_cfg<BN, A_MN, B_MN, 2, 2>(a, num_sms, s);
    return launch_cfg<BN, A_MN, B_MN, 2, 1>(a, num_sms, s);
}

}  // namespace tc

// Any N, K (M-grouped) and M (K-grouped) -- ragged tiles are zero-filled / clipped by TMA; the
// TMA constraints remain: 16-byte aligned base pointers and row strides (d, f multiples of 8,
// checked at creation), at most kMaxGroups groups per launch (run_gemm splits larger tables).
bool gemm_tc_supported(const GemmArgs& a)
{
    if (a.n_groups > tc::kMaxGroups || a.n_groups <= 0) return false;
    if (a.N <= 0 || a.K <= 0 && a.mode == GEMM_M_GROUPED) return false;
    if (a.mode == GEMM_M_GROUPED) {
        if (a.a_mn) return false;
        if (a.epi == EPI_F32) return false;
        if (a.c_rows <= 0 || a.ldc % 8 || a.lda % 8 || a.ldb % 8) return false;
    } else {
        if (!a.a_mn || !a.b_mn) return false;
        if (a.epi != EPI_F32 || a.M <= 0) return false;
        if (a.ldc % 4 || a.c_group_stride % 4 || a.lda % 8 || a.ldb % 8) return false;
    }
    return a.a_rows > 0 && a.b_rows > 0;
}

int launch_gemm_tc(const GemmArgs& a, int num_sms, cudaStream_t s)
{
    if (!gemm_tc_supported(a)) return -1;
    const bool bn256 = a.N % 256 == 0;           // else 128-column tiles (ragged N included)
    if (!a.a_mn && !a.b_mn) return bn256 ? tc::launch_cg<256, false, false>(a, num_sms, s)
                                         : tc::launch_cg<128, false, false>(a, num_sms, s);
    if (!a.a_mn && a.b_mn) return bn256 ? tc::launch_cg<256, false, true>(a, num_sms, s)
                                        : tc::launch_cg<128, false, true>(a, num_sms, s);
    return bn256 ? tc::launch_cg<256, true, true>(a, num_sms, s) : tc::launch_cg<128, true, true>(a, num_sms, s);
}

}  // namespace lancet
