// attention.cu -- causal multi-head self-attention of the GPT-MoE block on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA), and the block's LayerNorm kernels.
//
// The block (R19): h = x + Attn(LN1(x)); out = h + MoE(LN2(h)) --
// GPT-2's pre-LN block whose self-attention is the non-MoE computation before
// the MoE layer that Lancet partitions into the all-to-all pipeline (L171-L173, fig:part_all).
//
// Attention kernel: one CTA per (128-query tile, head, sequence), head_dim 128, causal.  The
// softmax is evaluated EXACTLY in two passes over the key tiles instead of with a running
// rescale of the output: pass 1 computes S_j = Q K_j^T into TMEM and the row max m and the row
// sum l = sum exp2(s - m) online; pass 2 recomputes S_j, writes P_j = exp2(s - m) / l (bf16)
// into shared memory in the UMMA K-major layout and accumulates O += P_j V_j in TMEM with no
// correction step.  The extra Q K^T costs 1/3 more MMA work, which the tensor core has to spare
// here.  (ncu, configs[3] chunk launches: XU (exp2) pipe 39 % busy, FMA 10 %, issue 29 % -- the
// kernel is latency-bound on the S -> softmax -> P hand-offs, not SFU-bound.)
//
// Roles (384 threads): warp 0 TMA producer | warp 1 MMA issuer (one thread) | warp 2 TMEM
// allocator | warp 3 idle | warps 4-11 softmax + epilogue: thread = query row (TMEM lane
// quadrant warp % 4), column half (warp - 4) / 4 -- two warps per row share the exponentials;
// their pass-1 row statistics meet once, in shared memory, after the last key tile.
// Shared memory: Q 32 KiB | K ring 2 x 32 KiB | V ring 2 x 32 KiB | P 2 x 32 KiB.
// TMEM: S double buffer (2 x 128 columns) + O (128 columns) of a 512-column allocation.
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace lancet {
namespace attn {

using namespace lancet::tc;

constexpr int HD = 128;                 // head dim
constexpr int TQ = 128;                 // query rows per CTA
constexpr int TK = 128;                 // keys per tile
constexpr int kThreads = 384;
constexpr uint32_t TILE_BYTES = 128 * 128 * 2;     // one 128 x 128 bf16 operand = 32 KiB
constexpr uint32_t BOX_BYTES = 128 * 64 * 2;       // a [128 rows][64] K-major box = 16 KiB
constexpr size_t kSmem = 1024 + 7 * (size_t)TILE_BYTES + 256;
constexpr uint32_t TMEM_COLS = 512;

__device__ __forceinline__ constexpr uint32_t idesc(bool b_mn) {
    // F32 accumulate, BF16 A / B, A K-major, B K-major (S = Q K^T) or MN-major (O += P V),
    // N = 128, M = 128
    return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(128 >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// qkv [T][3d] bf16 (q | k | v, head h at columns h*128 of each); att [T][d] bf16 out;
// lse [H][T] fp32 out: log2 of the row normaliser in the scaled (log2) domain, m + log2(l).
// Tokens [tok0, tok0 + n_seq * S) are processed.  Persistent: CTA b takes work items b,
// b + gridDim.x, ... (item -> (query tile, head, sequence), the longest (last) query tiles
// first); every barrier phase runs on counters that continue across items, so the next item's
// K / V loads and Q K^T start while the current item's softmax and P V finish (Q is reloaded
// once the current item's last Q K^T has completed; O is drained before the next item's first
// P V).
__global__ void __launch_bounds__(kThreads, 1)
attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmV,
                bf16* __restrict__ att, float* __restrict__ lse, int tok0, int S, int H, int d, int T_all,
                float scale_log2, int n_items)
{
    pdl_wait();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + TILE_BYTES;              // [2] stages
    uint8_t* sV = sK + 2 * TILE_BYTES;          // [2]
    uint8_t* sP = sV + 2 * TILE_BYTES;          // [2]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * TILE_BYTES);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = bars + 3;
    uint64_t* v_full = bars + 5;
    uint64_t* v_empty = bars + 7;
    uint64_t* s_full = bars + 9;
    uint64_t* s_empty = bars + 11;
    uint64_t* p_full = bars + 13;
    uint64_t* p_empty = bars + 15;
    uint64_t* o_full = bars + 17;
    uint64_t* q_empty = bars + 18;
    uint64_t* o_empty = bars + 19;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);
    // [2 halves][m | l][128] row statistics of pass 1, in P buffer 1 (no P V reads it then)
    float* red = reinterpret_cast<float*>(sP + TILE_BYTES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nq = S / TQ;
    const int bh = n_items / nq;                   // (sequence, head) pairs
    auto decode = [&](int item, int& qi, int& h, int& row0) {
        qi = nq - 1 - item / bh;                   // longest tiles first
        const int rem = item % bh;
        h = rem % H;
        row0 = tok0 + (rem / H) * S;               // first token of the sequence
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmQK);
        tma_prefetch(&tmV);
    }
    if (warp == 1 && lane == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 8);
            mbar_init(&p_full[i], 8); mbar_init(&p_empty[i], 1);
        }
        mbar_init(o_full, 1);
        mbar_init(o_empty, 8);
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
        // ===================== TMA producer =====================
        if (lane == 0) {
            uint32_t kc = 0, vc = 0, ni = 0;            // K tiles, V tiles, items so far
            for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++ni) {
                int qi, h, row0;
                decode(item, qi, h, row0);
                const int n = qi + 1;
                const int qcol = h * HD, kcol = d + h * HD, vcol = 2 * d + h * HD;
                mbar_wait(q_empty, (ni & 1) ^ 1);       // the last item's Q K^T are done
                mbar_expect_tx(q_full, TILE_BYTES);
                tma_load_2d(&tmQK, q_full, sQ, qcol, row0 + qi * TQ);
                tma_load_2d(&tmQK, q_full, sQ + BOX_BYTES, qcol + 64, row0 + qi * TQ);
                for (int it = 0; it < 2 * n; ++it, ++kc) {
                    const int j = it < n ? it : it - n;
                    const int ks = kc & 1;
                    mbar_wait(&k_empty[ks], ((kc >> 1) & 1) ^ 1);
                    mbar_expect_tx(&k_full[ks], TILE_BYTES);
                    uint8_t* kd = sK + ks * TILE_BYTES;
                    tma_load_2d(&tmQK, &k_full[ks], kd, kcol, row0 + j * TK);
                    tma_load_2d(&tmQK, &k_full[ks], kd + BOX_BYTES, kcol + 64, row0 + j * TK);
                    if (it >= n) {
                        const int vs = vc & 1;
                        mbar_wait(&v_empty[vs], ((vc >> 1) & 1) ^ 1);
                        mbar_expect_tx(&v_full[vs], TILE_BYTES);
                        uint8_t* vd = sV + vs * TILE_BYTES;
                        // MN-major B operand: boxes of [64 keys][64 head dims], (key half, dim half)
                        for (int kb = 0; kb < 2; ++kb)
                            for (int nb = 0; nb < 2; ++nb)
                                tma_load_2d(&tmV, &v_full[vs], vd + (kb * 2 + nb) * 8192, vcol + 64 * nb,
                                            row0 + j * TK + 64 * kb);
                        ++vc;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            const uint32_t sq_addr = smem_u32(sQ);
            uint32_t kc = 0, pc = 0, ni = 0;        // S tiles (= K tiles), P V tiles, items
            auto pv = [&](int jp) {
                const int pb = pc & 1;
                if (jp == 0) {
                    mbar_wait(o_empty, (ni & 1) ^ 1);   // the last item's O has been read
                    tc_fence_after();
                }
                mbar_wait(&p_full[pb], (pc >> 1) & 1);
                mbar_wait(&v_full[pb], (pc >> 1) & 1);
                tc_fence_after();
                const uint32_t pa = smem_u32(sP + pb * TILE_BYTES), va = smem_u32(sV + pb * TILE_BYTES);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t ad = make_desc(pa + (kk >> 2) * BOX_BYTES + (kk & 3) * 32, 16, 1024);
                    const uint64_t bd = make_desc(va + (kk >> 2) * 16384 + (kk & 3) * 2048, 8192, 1024);
                    tc_mma<1>(tmem + 256, ad, bd, idesc(true), (jp > 0 || kk > 0) ? 1u : 0u);
                }
                tc_commit<1>(&v_empty[pb]);
                tc_commit<1>(&p_empty[pb]);
                ++pc;
            };
            for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++ni) {
                int qi, h, row0;
                decode(item, qi, h, row0);
                const int n = qi + 1;
                mbar_wait(q_full, ni & 1);
                for (int it = 0; it < 2 * n; ++it, ++kc) {
                    const int b = kc & 1;
                    mbar_wait(&s_empty[b], ((kc >> 1) & 1) ^ 1);
                    mbar_wait(&k_full[b], (kc >> 1) & 1);
                    tc_fence_after();
                    const uint32_t ka = smem_u32(sK + b * TILE_BYTES);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint64_t ad = make_desc(sq_addr + (kk >> 2) * BOX_BYTES + (kk & 3) * 32, 16, 1024);
                        const uint64_t bd = make_desc(ka + (kk >> 2) * BOX_BYTES + (kk & 3) * 32, 16, 1024);
                        tc_mma<1>(tmem + 128 * b, ad, bd, idesc(false), kk > 0 ? 1u : 0u);
                    }
                    tc_commit<1>(&k_empty[b]);
                    tc_commit<1>(&s_full[b]);
                    if (it == 2 * n - 1) tc_commit<1>(q_empty);   // Q is free for the next item
                    if (it > n) pv(it - 1 - n);  // P_(j-1) V_(j-1) behind S_j: the softmax of j-1 overlaps S_j
                }
                pv(n - 1);
                tc_commit<1>(o_full);
            }
        }
    } else if (warp >= 4) {
        // ===================== softmax + epilogue (thread = query row, column half) =====
        const int quad = warp & 3, half = (warp - 4) >> 2;
        const int r = quad * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        uint32_t sc = 0, pc = 0, ni = 0;              // S tiles, P tiles, items
        uint32_t v[32];
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++ni) {
            int qi, h, row0;
            decode(item, qi, h, row0);
            const int n = qi + 1;
            const int q_pos = qi * TQ + r;             // query position in the sequence
            float m = -INFINITY, l = 0.f;
            // pass 1: this half's row max and normaliser (both 32-column chunks loaded at once;
            // 4 independent max / sum chains: the serial reductions were the latency limit)
            for (int it = 0; it < n; ++it, ++sc) {
                const int b = sc & 1;
                mbar_wait(&s_full[b], (sc >> 1) & 1);
                tc_fence_after();
                const bool diag = it == qi;
                uint32_t w2[32];
                tmem_ld32_issue(tmem + lane_off + 128 * b + 32 * (2 * half), v);
                tmem_ld32_issue(tmem + lane_off + 128 * b + 32 * (2 * half + 1), w2);
                tmem_wait_ld(v);
                tmem_wait_ld(w2);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[b]);    // S buffer b is in registers
                if (diag) {                                   // keys after the query: -inf (raw s)
#pragma unroll
                    for (int i = 0; i < 64; ++i)
                        if (it * TK + 64 * half + i > q_pos) {
                            if (i < 32) v[i] = __float_as_uint(-INFINITY);
                            else w2[i - 32] = __float_as_uint(-INFINITY);
                        }
                }
                // max on the raw scores (scale_log2 > 0), then exp2(s * scale - m) as one FFMA
                float cm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int i = 0; i < 64; ++i)
                    cm[i & 3] = fmaxf(cm[i & 3], __uint_as_float(i < 32 ? v[i] : w2[i - 32]));
                const float mn = fmaxf(m, fmaxf(fmaxf(cm[0], cm[1]), fmaxf(cm[2], cm[3])) * scale_log2);
                if (mn != -INFINITY) {
                    float su[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int i = 0; i < 64; ++i)
                        su[i & 3] += ex2(fmaf(__uint_as_float(i < 32 ? v[i] : w2[i - 32]), scale_log2, -mn));
                    l = l * ex2(m - mn) + ((su[0] + su[1]) + (su[2] + su[3]));
                    m = mn;
                }
            }
            // the two halves' statistics of each row meet (named barrier of the 8 softmax warps)
            red[(half * 2 + 0) * 128 + r] = m;
            red[(half * 2 + 1) * 128 + r] = l;
            asm volatile("bar.sync 1, 256;" ::: "memory");
            {
                const float mo = red[((half ^ 1) * 2 + 0) * 128 + r], lo = red[((half ^ 1) * 2 + 1) * 128 + r];
                const float mm = fmaxf(m, mo);
                l = (m == -INFINITY ? 0.f : l * ex2(m - mm)) + (mo == -INFINITY ? 0.f : lo * ex2(mo - mm));
                m = mm;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");     // every read done before P buffer 1 is written
            const float mlog = m + __log2f(l);           // P = exp2(s * scale - m) / l in one FFMA + EX2
            // pass 2: P = exp2(s - m) / l into shared memory (K-major SW128: box `half` of P)
            for (int j = 0; j < n; ++j, ++sc, ++pc) {
                const int b = sc & 1, pb = pc & 1;
                mbar_wait(&s_full[b], (sc >> 1) & 1);
                mbar_wait(&p_empty[pb], ((pc >> 1) & 1) ^ 1);
                tc_fence_after();
                const bool diag = j == qi;
                uint8_t* box = sP + pb * TILE_BYTES + half * BOX_BYTES + r * 128;
                uint32_t w2[32];
                tmem_ld32_issue(tmem + lane_off + 128 * b + 32 * (2 * half), v);
                tmem_ld32_issue(tmem + lane_off + 128 * b + 32 * (2 * half + 1), w2);
                tmem_wait_ld(v);
                tmem_wait_ld(w2);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[b]);    // S buffer b is in registers
                if (diag) {
#pragma unroll
                    for (int i = 0; i < 64; ++i)
                        if (j * TK + 64 * half + i > q_pos) {
                            if (i < 32) v[i] = __float_as_uint(-INFINITY);
                            else w2[i - 32] = __float_as_uint(-INFINITY);
                        }
                }
#pragma unroll
                for (int c2 = 0; c2 < 2; ++c2) {
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const uint32_t r0 = c2 ? w2[2 * i] : v[2 * i], r1 = c2 ? w2[2 * i + 1] : v[2 * i + 1];
                        const float p0 = ex2(fmaf(__uint_as_float(r0), scale_log2, -mlog));
                        const float p1 = ex2(fmaf(__uint_as_float(r1), scale_log2, -mlog));
                        __nv_bfloat162 hv = __floats2bfloat162_rn(p0, p1);
                        pk[i] = *reinterpret_cast<uint32_t*>(&hv);
                    }
#pragma unroll
                    for (int c4 = 0; c4 < 4; ++c4) {
                        const int c16 = c2 * 4 + c4;
                        st_v4(box + ((c16 ^ (r & 7)) << 4), make_uint4(pk[4 * c4], pk[4 * c4 + 1], pk[4 * c4 + 2], pk[4 * c4 + 3]));
                    }
                }
                fence_proxy_async();            // generic-proxy stores -> visible to the tensor core
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[pb]);
            }
            // epilogue: this half's 64 columns of O (TMEM columns 256..383) -> bf16 rows of att
            mbar_wait(o_full, ni & 1);
            tc_fence_after();
            uint32_t o2[2][32];
            tmem_ld32(tmem + lane_off + 256 + 32 * (2 * half), o2[0]);
            tmem_ld32(tmem + lane_off + 256 + 32 * (2 * half + 1), o2[1]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_empty);        // the next item's first P V may overwrite O
            const long tok = (long)row0 + qi * TQ + r;
            bf16* orow = att + tok * d + h * HD;
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) {
                const int cc = 2 * half + c2;
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    __nv_bfloat162 hv = __floats2bfloat162_rn(__uint_as_float(o2[c2][2 * i]), __uint_as_float(o2[c2][2 * i + 1]));
                    pk[i] = *reinterpret_cast<uint32_t*>(&hv);
                }
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4)
                    st_v4(orow + 32 * cc + 8 * c4, make_uint4(pk[4 * c4], pk[4 * c4 + 1], pk[4 * c4 + 2], pk[4 * c4 + 3]));
            }
            if (half == 0) lse[(long)h * T_all + tok] = mlog;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

}  // namespace attn

int launch_attention_fwd(const void* qkv, void* att, float* lse, int tok0, int n_seq, int S, int H, int d,
                         int T_all, cudaStream_t s)
{
    using namespace attn;
    if (d != H * HD || S % TQ || n_seq <= 0) return -1;
    CUtensorMap tqk, tv;
    const uint64_t rows = (uint64_t)T_all;
    if (!tc::make_map(&tqk, qkv, 3ull * d, rows, 3ull * d, 64, 128)) return -1;
    if (!tc::make_map(&tv, qkv, 3ull * d, rows, 3ull * d, 64, 64)) return -1;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
        attr = true;
    }
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int items = n_seq * H * (S / TQ);
    const int grid = std::min(items, num_sms);      // persistent: one CTA per SM
    const float scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
    if (launch_k(attn_fwd_kernel, grid, kThreads, kSmem, s, tqk, tv, (bf16*)att, lse, tok0, S, H, d, T_all,
                 scale_log2, items) != cudaSuccess)
        return -1;
    return 1;
}

// ---------------------------------------------------------------- LayerNorm ---------------
// One warp per row (d % 8 == 0, d <= 4096): the row in registers (NV = ceil(d / 256) 16-byte
// vectors per lane), mean and variance in two passes over the registers (biased variance,
// GPT-2's LN), y = (x - mean) * rstd * g + b stored in bf16; mean and rstd kept (fp32) for the
// backward.  RESID: the input row is h = bf16(a + b) (the residual add before LN2), stored too.
template <int NV, bool RESID>
__global__ void __launch_bounds__(256)
ln_kernel(const bf16* __restrict__ a, const bf16* __restrict__ b2, bf16* __restrict__ hout,
          const float* __restrict__ g, const float* __restrict__ be, bf16* __restrict__ y,
          float* __restrict__ mean, float* __restrict__ rstd, int rows, int d, float eps)
{
    pdl_wait();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const long base = (long)warp * d;
    float x[NV][8];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const int col = (v * 32 + lane) * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) x[v][i] = 0.f;
        if (col < d) {
            unpack16<bf16>(ld_nc_v4(a + base + col), x[v]);
            if (RESID) {
                float o[8];
                unpack16<bf16>(ld_nc_v4(b2 + base + col), o);
#pragma unroll
                for (int i = 0; i < 8; ++i) x[v][i] = __bfloat162float(__float2bfloat16_rn(x[v][i] + o[i]));
                st_v4(hout + base + col, pack16<bf16>(x[v]));
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int i = 0; i < 8; ++i) s += x[v][i];
    const float mu = warp_sum(s) / (float)d;
    float q = 0.f;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        if ((v * 32 + lane) * 8 >= d) continue;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float c = x[v][i] - mu;
            q += c * c;
        }
    }
    const float rs = rsqrtf(warp_sum(q) / (float)d + eps);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const int col = (v * 32 + lane) * 8;
        if (col >= d) continue;
        float gg[8], bb[8], o[8];
        *reinterpret_cast<float4*>(gg) = *reinterpret_cast<const float4*>(g + col);
        *reinterpret_cast<float4*>(gg + 4) = *reinterpret_cast<const float4*>(g + col + 4);
        *reinterpret_cast<float4*>(bb) = *reinterpret_cast<const float4*>(be + col);
        *reinterpret_cast<float4*>(bb + 4) = *reinterpret_cast<const float4*>(be + col + 4);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = (x[v][i] - mu) * rs * gg[i] + bb[i];
        st_v4(y + base + col, pack16<bf16>(o));
    }
    if (lane == 0) {
        mean[warp] = mu;
        rstd[warp] = rs;
    }
}

int launch_layer_norm(const void* a, const void* resid, void* hout, const float* g, const float* b, void* y,
                      float* mean, float* rstd, int rows, int d, cudaStream_t s)
{
    if (d % 8 || d > 4096 || rows <= 0) return -1;
    const int blocks = ceil_div(rows, 8);
    const float eps = 1e-5f;
#define LN(NV)                                                                                                 \
    if (resid) launch_k(ln_kernel<NV, true>, blocks, 256, 0, s, (const bf16*)a, (const bf16*)resid, (bf16*)hout, g, \
                        b, (bf16*)y, mean, rstd, rows, d, eps);                                                  \
    else launch_k(ln_kernel<NV, false>, blocks, 256, 0, s, (const bf16*)a, (const bf16*)nullptr, (bf16*)nullptr, g, \
                  b, (bf16*)y, mean, rstd, rows, d, eps);
    switch (ceil_div(d, 256)) {
    case 1: LN(1) break;
    case 2: LN(2) break;
    case 3: LN(3) break;
    case 4: LN(4) break;
    case 5: case 6: LN(6) break;
    case 7: case 8: LN(8) break;
    case 9: case 10: case 11: case 12: LN(12) break;
    default: LN(16) break;
    }
#undef LN
    return 1;
}

}  // namespace lancet
