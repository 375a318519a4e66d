// attention_bwd.cu -- backward of the block's causal self-attention on the tcgen05 tensor cores,
// and the block's LayerNorm backward.
//
// With s = q k^T / sqrt(hd), P = softmax_causal(s) (recomputed exactly from the forward's row
// normaliser: P = exp2(s log2e - lse2)), O = P V and dO the gradient of O:
//     D_q = sum_c dO[q][c] O[q][c]            (attn_bwd_d_kernel)
//     dP  = dO V^T,  dS = P (dP - D_q)
//     dV  = P^T dO,  dK = dS^T Q / sqrt(hd)   (attn_bwd_kv_kernel: one CTA per key tile, loop over
//                                              the query tiles at or after it)
//     dQ  = dS K / sqrt(hd)                   (attn_bwd_q_kernel: one CTA per query tile, loop over
//                                              the key tiles at or before it)
// Two kernels instead of one with atomic dQ accumulation: every output is written once by one
// CTA (deterministic, no fp32 reduce traffic) at the price of recomputing S and dP in the dQ pass.
// P^T and dS^T are written by the elementwise warps (thread = key row) as K-major operands of
// the dV / dK MMAs; the same dS^T buffer would be the MN-major A operand of dQ = dS K, the
// K / Q / dO tiles are the MN-major B operands of dQ, dK and dV straight from their TMA boxes.
// Roles (384 threads): warp 0 TMA producer | warp 1 MMA issuer | warp 2 TMEM allocator |
// warps 4-11 elementwise (TMEM lane quadrant warp % 4, column half (warp - 4) / 4).
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace lancet {
namespace attnb {

using namespace lancet::tc;

constexpr int HD = 128, TQ = 128, TK = 128;
constexpr int kThreads = 384;
constexpr uint32_t TILE = 128 * 128 * 2;           // 32 KiB
constexpr uint32_t BOX = 128 * 64 * 2;             // a [128 rows][64] K-major box
constexpr size_t kSmemKV = 1024 + 6 * (size_t)TILE + 256;
constexpr size_t kSmemQ = 1024 + 7 * (size_t)TILE + 256;
constexpr uint32_t TMEM_COLS = 512;

__device__ __forceinline__ constexpr uint32_t idesc(bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(128 >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}
// K-major [128 rows][128 K] operand in two SW128 boxes: K step kk (16 wide)
__device__ __forceinline__ uint64_t kmaj(uint32_t base, int kk) {
    return make_desc(base + (kk >> 2) * BOX + (kk & 3) * 32, 16, 1024);
}
// the same two boxes read as an MN-major operand (rows = K, 64-wide MN blocks one box apart)
__device__ __forceinline__ uint64_t mnmaj(uint32_t base, int kk) {
    return make_desc(base + kk * 2048, BOX, 1024);
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 64 bf16 (one thread's half row) into a K-major SW128 box row
__device__ __forceinline__ void st_row64(uint8_t* box_row, int r, const float* v) {
#pragma unroll
    for (int c16 = 0; c16 < 8; ++c16) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            __nv_bfloat162 hv = __floats2bfloat162_rn(v[c16 * 8 + 2 * q], v[c16 * 8 + 2 * q + 1]);
            w[q] = *reinterpret_cast<uint32_t*>(&hv);
        }
        st_v4(box_row + ((c16 ^ (r & 7)) << 4), make_uint4(w[0], w[1], w[2], w[3]));
    }
}
__device__ __forceinline__ void ld64(uint32_t taddr, float* out) {
    uint32_t a[32], b[32];
    tmem_ld32_issue(taddr, a);
    tmem_ld32_issue(taddr + 32, b);
    tmem_wait_ld(a);
    tmem_wait_ld(b);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        out[i] = __uint_as_float(a[i]);
        out[32 + i] = __uint_as_float(b[i]);
    }
}
__device__ __forceinline__ void store64_bf16(bf16* dst, const float* v, float scale) {
#pragma unroll
    for (int c8 = 0; c8 < 8; ++c8) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            __nv_bfloat162 hv = __floats2bfloat162_rn(v[c8 * 8 + 2 * q] * scale, v[c8 * 8 + 2 * q + 1] * scale);
            w[q] = *reinterpret_cast<uint32_t*>(&hv);
        }
        st_v4(dst + c8 * 8, make_uint4(w[0], w[1], w[2], w[3]));
    }
}

// D[h][t] = sum_c dO[t][h*128 + c] * O[t][h*128 + c]: one warp per (token, head)
__global__ void __launch_bounds__(256)
attn_bwd_d_kernel(const bf16* __restrict__ dO, const bf16* __restrict__ O, float* __restrict__ D, int tok0,
                  int rows, int H, int d, int T_all)
{
    pdl_wait();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows * H) return;
    const int t = tok0 + w / H, h = w % H;
    const size_t off = (size_t)t * d + h * HD + lane * 4;
    const uint2 a = *reinterpret_cast<const uint2*>(dO + off), b = *reinterpret_cast<const uint2*>(O + off);
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float2 fa = __bfloat1622float2(a2[i]), fb = __bfloat1622float2(b2[i]);
        s += fa.x * fb.x + fa.y * fb.y;
    }
    s = warp_sum(s);
    if (lane == 0) D[(size_t)h * T_all + t] = s;
}

// dK, dV of key tile j: CTA -> (key tile, head, sequence), the longest (first key tiles) first.
__global__ void __launch_bounds__(kThreads, 1)
attn_bwd_kv_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDO,
                   const float* __restrict__ lse, const float* __restrict__ Dv, bf16* __restrict__ dqkv, int tok0,
                   int S, int H, int d, int T_all, float scale_log2, float scale)
{
    pdl_wait();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sK = smem, *sV = smem + TILE, *sQ = smem + 2 * TILE, *sDO = smem + 3 * TILE;
    uint8_t *sP = smem + 4 * TILE, *sDS = smem + 5 * TILE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * TILE);
    uint64_t *kv_full = bars, *qd_full = bars + 1, *qd_empty = bars + 2, *s_full = bars + 3, *s_empty = bars + 4;
    uint64_t *p_full = bars + 5, *p_empty = bars + 6, *acc_full = bars + 7;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = S / TK;
    const int bh = gridDim.x / nk;
    const int j = (int)blockIdx.x / bh;                 // key tile: j = 0 has the most query tiles
    const int rem = (int)blockIdx.x % bh;
    const int h = rem % H, row0 = tok0 + (rem / H) * S;
    const int m = nk - j;                                // query tiles i = j .. nk-1

    if (warp == 1 && lane == 0) {
        mbar_init(kv_full, 1); mbar_init(qd_full, 1); mbar_init(qd_empty, 1); mbar_init(s_full, 1);
        mbar_init(s_empty, 8); mbar_init(p_full, 8); mbar_init(p_empty, 1); mbar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const int qc = h * HD, kc = d + h * HD, vc = 2 * d + h * HD;
            mbar_expect_tx(kv_full, 2 * TILE);
            tma_load_2d(&tmQKV, kv_full, sK, kc, row0 + j * TK);
            tma_load_2d(&tmQKV, kv_full, sK + BOX, kc + 64, row0 + j * TK);
            tma_load_2d(&tmQKV, kv_full, sV, vc, row0 + j * TK);
            tma_load_2d(&tmQKV, kv_full, sV + BOX, vc + 64, row0 + j * TK);
            for (int it = 0; it < m; ++it) {
                const int qrow = row0 + (j + it) * TQ;
                mbar_wait(qd_empty, (it & 1) ^ 1);
                mbar_expect_tx(qd_full, 2 * TILE);
                tma_load_2d(&tmQKV, qd_full, sQ, qc, qrow);
                tma_load_2d(&tmQKV, qd_full, sQ + BOX, qc + 64, qrow);
                tma_load_2d(&tmDO, qd_full, sDO, h * HD, qrow);
                tma_load_2d(&tmDO, qd_full, sDO + BOX, h * HD + 64, qrow);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t k_a = smem_u32(sK), v_a = smem_u32(sV), q_a = smem_u32(sQ), do_a = smem_u32(sDO);
            const uint32_t p_a = smem_u32(sP), ds_a = smem_u32(sDS);
            mbar_wait(kv_full, 0);
            for (int it = 0; it < m; ++it) {
                mbar_wait(qd_full, it & 1);
                mbar_wait(s_empty, (it & 1) ^ 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)          // S^T = K Q^T  (keys x queries)
                    tc_mma<1>(tmem, kmaj(k_a, kk), kmaj(q_a, kk), idesc(false), kk > 0);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)          // dP^T = V dO^T
                    tc_mma<1>(tmem + 128, kmaj(v_a, kk), kmaj(do_a, kk), idesc(false), kk > 0);
                tc_commit<1>(s_full);
                mbar_wait(p_full, it & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)          // dV += P^T dO   (dO as MN-major B)
                    tc_mma<1>(tmem + 256, kmaj(p_a, kk), mnmaj(do_a, kk), idesc(true), (it > 0 || kk > 0));
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)          // dK += dS^T Q   (Q as MN-major B)
                    tc_mma<1>(tmem + 384, kmaj(ds_a, kk), mnmaj(q_a, kk), idesc(true), (it > 0 || kk > 0));
                tc_commit<1>(p_empty);
                tc_commit<1>(qd_empty);
            }
            tc_commit<1>(acc_full);
        }
    } else if (warp >= 4) {
        const int quad = warp & 3, half = (warp - 4) >> 2;
        const int r = quad * 32 + lane;                 // key row
        const int kpos = j * TK + r;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        float st[64], dp[64];
        for (int it = 0; it < m; ++it) {
            const int i = j + it;
            const int qtok = row0 + i * TQ + 64 * half;  // first query token of this half
            mbar_wait(s_full, it & 1);
            tc_fence_after();
            ld64(tmem + lane_off + 64 * half, st);
            ld64(tmem + lane_off + 128 + 64 * half, dp);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_empty);
            const float* lq = lse + (size_t)h * T_all + qtok;
            const float* dq = Dv + (size_t)h * T_all + qtok;
            if (i == j) {                               // diagonal tile: key after query -> P = 0
#pragma unroll
                for (int c = 0; c < 64; ++c)
                    if (i * TQ + 64 * half + c < kpos) st[c] = -INFINITY;
            }
#pragma unroll
            for (int c = 0; c < 64; ++c) {
                const float l2 = __ldg(lq + c), dd = __ldg(dq + c);
                const float p = ex2(fmaf(st[c], scale_log2, -l2));
                st[c] = p;
                dp[c] = p * (dp[c] - dd);
            }
            mbar_wait(p_empty, (it & 1) ^ 1);
            st_row64(sP + half * BOX + r * 128, r, st);
            st_row64(sDS + half * BOX + r * 128, r, dp);
            fence_proxy_async();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
        }
        mbar_wait(acc_full, 0);
        tc_fence_after();
        ld64(tmem + lane_off + 256 + 64 * half, st);     // dV
        ld64(tmem + lane_off + 384 + 64 * half, dp);     // dK
        const long tok = (long)row0 + j * TK + r;
        store64_bf16(dqkv + tok * 3 * d + 2 * d + h * HD + 64 * half, st, 1.f);
        store64_bf16(dqkv + tok * 3 * d + d + h * HD + 64 * half, dp, scale);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// dQ of query tile i: CTA -> (query tile, head, sequence), the longest (last query tiles) first.
__global__ void __launch_bounds__(kThreads, 1)
attn_bwd_q_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDO,
                  const float* __restrict__ lse, const float* __restrict__ Dv, bf16* __restrict__ dqkv, int tok0,
                  int S, int H, int d, int T_all, float scale_log2, float scale)
{
    pdl_wait();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sQ = smem, *sDO = smem + TILE, *sK = smem + 2 * TILE, *sV = smem + 4 * TILE, *sDS = smem + 6 * TILE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 7 * TILE);
    uint64_t *qd_full = bars, *kv_full = bars + 1, *kv_empty = bars + 3, *s_full = bars + 5, *s_empty = bars + 6;
    uint64_t *ds_full = bars + 7, *ds_empty = bars + 8, *dq_full = bars + 9;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nq = S / TQ;
    const int bh = gridDim.x / nq;
    const int i = nq - 1 - (int)blockIdx.x / bh;
    const int rem = (int)blockIdx.x % bh;
    const int h = rem % H, row0 = tok0 + (rem / H) * S;
    const int n = i + 1;                                 // key tiles 0 .. i

    if (warp == 1 && lane == 0) {
        mbar_init(qd_full, 1);
        for (int q = 0; q < 2; ++q) { mbar_init(&kv_full[q], 1); mbar_init(&kv_empty[q], 1); }
        mbar_init(s_full, 1); mbar_init(s_empty, 8); mbar_init(ds_full, 8); mbar_init(ds_empty, 1);
        mbar_init(dq_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const int qc = h * HD, kc = d + h * HD, vc = 2 * d + h * HD;
            const int qrow = row0 + i * TQ;
            mbar_expect_tx(qd_full, 2 * TILE);
            tma_load_2d(&tmQKV, qd_full, sQ, qc, qrow);
            tma_load_2d(&tmQKV, qd_full, sQ + BOX, qc + 64, qrow);
            tma_load_2d(&tmDO, qd_full, sDO, h * HD, qrow);
            tma_load_2d(&tmDO, qd_full, sDO + BOX, h * HD + 64, qrow);
            for (int jj = 0; jj < n; ++jj) {
                const int sl = jj & 1;
                mbar_wait(&kv_empty[sl], ((jj >> 1) & 1) ^ 1);
                mbar_expect_tx(&kv_full[sl], 2 * TILE);
                uint8_t* kd = sK + sl * TILE;
                uint8_t* vd = sV + sl * TILE;
                tma_load_2d(&tmQKV, &kv_full[sl], kd, kc, row0 + jj * TK);
                tma_load_2d(&tmQKV, &kv_full[sl], kd + BOX, kc + 64, row0 + jj * TK);
                tma_load_2d(&tmQKV, &kv_full[sl], vd, vc, row0 + jj * TK);
                tma_load_2d(&tmQKV, &kv_full[sl], vd + BOX, vc + 64, row0 + jj * TK);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t q_a = smem_u32(sQ), do_a = smem_u32(sDO), ds_a = smem_u32(sDS);
            mbar_wait(qd_full, 0);
            for (int jj = 0; jj < n; ++jj) {
                const int sl = jj & 1;
                const uint32_t k_a = smem_u32(sK + sl * TILE), v_a = smem_u32(sV + sl * TILE);
                mbar_wait(&kv_full[sl], (jj >> 1) & 1);
                mbar_wait(s_empty, (jj & 1) ^ 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)          // S = Q K^T
                    tc_mma<1>(tmem, kmaj(q_a, kk), kmaj(k_a, kk), idesc(false), kk > 0);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)          // dP = dO V^T
                    tc_mma<1>(tmem + 128, kmaj(do_a, kk), kmaj(v_a, kk), idesc(false), kk > 0);
                tc_commit<1>(s_full);
                mbar_wait(ds_full, jj & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)          // dQ += dS K   (K as MN-major B)
                    tc_mma<1>(tmem + 256, kmaj(ds_a, kk), mnmaj(k_a, kk), idesc(true), (jj > 0 || kk > 0));
                tc_commit<1>(&kv_empty[sl]);
                tc_commit<1>(ds_empty);
            }
            tc_commit<1>(dq_full);
        }
    } else if (warp >= 4) {
        const int quad = warp & 3, half = (warp - 4) >> 2;
        const int r = quad * 32 + lane;                 // query row
        const int qpos = i * TQ + r;
        const long tok = (long)row0 + qpos;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const float l2 = lse[(size_t)h * T_all + tok], dd = Dv[(size_t)h * T_all + tok];
        float s[64], dp[64];
        for (int jj = 0; jj < n; ++jj) {
            mbar_wait(s_full, jj & 1);
            tc_fence_after();
            ld64(tmem + lane_off + 64 * half, s);
            ld64(tmem + lane_off + 128 + 64 * half, dp);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_empty);
            if (jj == i) {                              // diagonal tile: key after query -> P = 0
#pragma unroll
                for (int c = 0; c < 64; ++c)
                    if (jj * TK + 64 * half + c > qpos) s[c] = -INFINITY;
            }
#pragma unroll
            for (int c = 0; c < 64; ++c) dp[c] = ex2(fmaf(s[c], scale_log2, -l2)) * (dp[c] - dd);
            mbar_wait(ds_empty, (jj & 1) ^ 1);
            st_row64(sDS + half * BOX + r * 128, r, dp);
            fence_proxy_async();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full);
        }
        mbar_wait(dq_full, 0);
        tc_fence_after();
        ld64(tmem + lane_off + 256 + 64 * half, s);
        store64_bf16(dqkv + tok * 3 * d + h * HD + 64 * half, s, scale);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

}  // namespace attnb

int launch_attention_bwd(const void* qkv, const void* att, const void* datt, const float* lse, float* Dbuf,
                         void* dqkv, int tok0, int n_seq, int S, int H, int d, int T_all, cudaStream_t s)
{
    using namespace attnb;
    if (d != H * HD || S % TQ || n_seq <= 0) return -1;
    CUtensorMap tqkv, tdo;
    if (!tc::make_map(&tqkv, qkv, 3ull * d, (uint64_t)T_all, 3ull * d, 64, 128)) return -1;
    if (!tc::make_map(&tdo, datt, (uint64_t)d, (uint64_t)T_all, (uint64_t)d, 64, 128)) return -1;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_bwd_kv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemKV);
        cudaFuncSetAttribute(attn_bwd_q_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemQ);
        attr = true;
    }
    const int rows = n_seq * S;
    launch_k(attn_bwd_d_kernel, ceil_div(rows * H * 32, 256), 256, 0, s, (const bf16*)datt, (const bf16*)att, Dbuf,
             tok0, rows, H, d, T_all);
    const float scale = 1.f / sqrtf((float)HD), scale_log2 = 1.4426950408889634f * scale;
    const int grid = n_seq * H * (S / TQ);
    if (launch_k(attn_bwd_kv_kernel, grid, kThreads, kSmemKV, s, tqkv, tdo, lse, (const float*)Dbuf, (bf16*)dqkv, tok0,
                 S, H, d, T_all, scale_log2, scale) != cudaSuccess)
        return -1;
    if (launch_k(attn_bwd_q_kernel, grid, kThreads, kSmemQ, s, tqkv, tdo, lse, (const float*)Dbuf, (bf16*)dqkv, tok0,
                 S, H, d, T_all, scale_log2, scale) != cudaSuccess)
        return -1;
    return 3;
}

// ---------------------------------------------------------------- LayerNorm backward --------
// Row kernel: one warp per row (d % 8 == 0), two passes over the row's columns (the second
// re-reads dy and x from L1 / L2 instead of holding them in registers):
//   xhat = (x - mean) rstd;  dxhat = dy g;  out = resid + rstd (dxhat - mean(dxhat) - xhat mean(dxhat xhat))
// Column kernel: dg = sum_t dy xhat, db = sum_t dy as [row chunks][2][d] partials, then a
// fixed-order reduction (deterministic).
__global__ void __launch_bounds__(256)
ln_bwd_rows_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x, const float* __restrict__ mean,
                   const float* __restrict__ rstd, const float* __restrict__ g, const bf16* __restrict__ resid,
                   bf16* __restrict__ out, int rows, int d)
{
    pdl_wait();
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (row >= rows) return;
    const long base = (long)row * d;
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll 4
    for (int col = lane * 8; col < d; col += 256) {
        float xv[8], dv[8], gg[8];
        unpack16<bf16>(ld_v4(x + base + col), xv);
        unpack16<bf16>(ld_v4(dy + base + col), dv);
        *reinterpret_cast<float4*>(gg) = *reinterpret_cast<const float4*>(g + col);
        *reinterpret_cast<float4*>(gg + 4) = *reinterpret_cast<const float4*>(g + col + 4);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float dx = dv[i] * gg[i];
            s1 += dx;
            s2 += dx * (xv[i] - mu) * rs;
        }
    }
    const float m1 = warp_sum(s1) / (float)d, m2 = warp_sum(s2) / (float)d;
#pragma unroll 4
    for (int col = lane * 8; col < d; col += 256) {
        float xv[8], dv[8], gg[8], rv[8], o[8];
        unpack16<bf16>(ld_v4(x + base + col), xv);
        unpack16<bf16>(ld_v4(dy + base + col), dv);
        unpack16<bf16>(ld_nc_v4(resid + base + col), rv);
        *reinterpret_cast<float4*>(gg) = *reinterpret_cast<const float4*>(g + col);
        *reinterpret_cast<float4*>(gg + 4) = *reinterpret_cast<const float4*>(g + col + 4);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = rv[i] + rs * (dv[i] * gg[i] - m1 - (xv[i] - mu) * rs * m2);
        st_v4(out + base + col, pack16<bf16>(o));
    }
}

constexpr int kLnColChunk = 32;    // rows per column-partial block
// thread = 8 consecutive columns (16-byte loads), block = 2048 columns x 32 rows
__global__ void __launch_bounds__(256)
ln_bwd_cols_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x, const float* __restrict__ mean,
                   const float* __restrict__ rstd, float* __restrict__ partial, int rows, int d)
{
    pdl_wait();
    const int col = (blockIdx.x * 256 + threadIdx.x) * 8;
    if (col >= d) return;
    const int r0 = blockIdx.y * kLnColChunk, r1 = min(rows, r0 + kLnColChunk);
    float a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = b[i] = 0.f;
#pragma unroll 4
    for (int r = r0; r < r1; ++r) {
        float dv[8], xv[8];
        unpack16<bf16>(ld_nc_v4(dy + (long)r * d + col), dv);
        unpack16<bf16>(ld_nc_v4(x + (long)r * d + col), xv);
        const float mu = __ldg(mean + r), rs = __ldg(rstd + r);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            a[i] = fmaf(dv[i], (xv[i] - mu) * rs, a[i]);
            b[i] += dv[i];
        }
    }
    float* pa = partial + ((size_t)blockIdx.y * 2 + 0) * d + col;
    float* pb = partial + ((size_t)blockIdx.y * 2 + 1) * d + col;
    *reinterpret_cast<float4*>(pa) = make_float4(a[0], a[1], a[2], a[3]);
    *reinterpret_cast<float4*>(pa + 4) = make_float4(a[4], a[5], a[6], a[7]);
    *reinterpret_cast<float4*>(pb) = make_float4(b[0], b[1], b[2], b[3]);
    *reinterpret_cast<float4*>(pb + 4) = make_float4(b[4], b[5], b[6], b[7]);
}

// dg[c] = sum_q partial[q][0][c], db[c] = sum_q partial[q][1][c]: block = 32 columns x 8 chunk
// groups (group g sums chunks g, g + 8, ...), the 8 group sums added in order (deterministic)
__global__ void __launch_bounds__(256)
ln_bwd_reduce_kernel(const float* __restrict__ partial, int nb, int d, float* __restrict__ dg,
                     float* __restrict__ db)
{
    pdl_wait();
    __shared__ float sa[8][32], sb[8][32];
    const int cl = threadIdx.x & 31, grp = threadIdx.x >> 5;
    const int c = blockIdx.x * 32 + cl;
    float a = 0.f, b = 0.f;
    if (c < d)
        for (int q = grp; q < nb; q += 8) {
            a += partial[((size_t)q * 2 + 0) * d + c];
            b += partial[((size_t)q * 2 + 1) * d + c];
        }
    sa[grp][cl] = a;
    sb[grp][cl] = b;
    __syncthreads();
    if (grp == 0 && c < d) {
        float ta = 0.f, tb = 0.f;
#pragma unroll
        for (int g = 0; g < 8; ++g) { ta += sa[g][cl]; tb += sb[g][cl]; }
        dg[c] = ta;
        db[c] = tb;
    }
}

size_t ln_bwd_partial_floats(int rows, int d) { return (size_t)ceil_div(rows, kLnColChunk) * 2 * d; }

int launch_layer_norm_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const float* g,
                          const void* resid, void* out, float* partial, float* dg, float* db, int rows, int d,
                          cudaStream_t s)
{
    if (d % 8 || rows <= 0) return -1;
    launch_k(ln_bwd_rows_kernel, ceil_div(rows * 32, 256), 256, 0, s, (const bf16*)dy, (const bf16*)x, mean, rstd, g,
             (const bf16*)resid, (bf16*)out, rows, d);
    const int nb = ceil_div(rows, kLnColChunk);
    launch_k(ln_bwd_cols_kernel, dim3(ceil_div(d, 2048), nb), 256, 0, s, (const bf16*)dy, (const bf16*)x, mean, rstd,
             partial, rows, d);
    launch_k(ln_bwd_reduce_kernel, ceil_div(d, 32), 256, 0, s, (const float*)partial, nb, d, dg, db);
    return 3;
}

}  // namespace lancet
