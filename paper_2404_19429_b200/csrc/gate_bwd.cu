// gate_bwd.cu -- K6 (dispatch backward + gate term of dx) and K7 (dWg) of the MoE layer.
//
//   dx_t     = sum_{admitted j} dX[row_tj] + sum_e dlogit_te Wg[:, e]
//   dlogit_t = p_t (g~_t - sum_j g_tj w_tj)                 (softmax Jacobian, R3)
//            = w_tj (g_tj - sum_j' g_tj' w_tj') at idx_tj   (renormalised weights)
//   dWg      = x^T dlogit     (local; the data-parallel all-reduce of the replicated gate,
//                              P:L110, is the caller's)
// Top-k and capacity decisions are piecewise constant and carry no gradient.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace lancet {

namespace {

template <int KK>
__device__ __forceinline__ void choices(const int* __restrict__ idx, const int* __restrict__ slot,
                                        const float* __restrict__ wts, const float* __restrict__ g,
                                        const int* __restrict__ send_off, int t, int k, int lane,
                                        int (&rows)[KK], float (&wj)[KK], int (&ids)[KK], float (&gj)[KK])
{
    int myrow = -1, myidx = -1;
    float myw = 0.f, myg = 0.f;
    if (lane < k) {
        const int s = slot[(size_t)t * k + lane];
        myidx = idx[(size_t)t * k + lane];
        myrow = s >= 0 ? send_off[myidx] + s : -1;
        myw = wts[(size_t)t * k + lane];
        myg = g[(size_t)t * k + lane];
    }
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        rows[j] = j < k ? __shfl_sync(0xffffffffu, myrow, j) : -1;
        wj[j] = __shfl_sync(0xffffffffu, myw, j);
        ids[j] = __shfl_sync(0xffffffffu, myidx, j);
        gj[j] = __shfl_sync(0xffffffffu, myg, j);
    }
}

// dlogit of token t into sdl[0..E) (and global dlogit), computed by one warp.
template <int KK>
__device__ __forceinline__ void token_dlogit(const float* __restrict__ logits, int t, int E, int k, int renorm,
                                             const int (&ids)[KK], const float (&wj)[KK], const float (&gj)[KK],
                                             int lane, float* sdl, float* __restrict__ dlogit)
{
    float sg = 0.f;                                    // sum_j g_j w_j
#pragma unroll
    for (int j = 0; j < KK; ++j)
        if (j < k) sg = fmaf(gj[j], wj[j], sg);
    const float* lr = logits + (size_t)t * E;
    float m = -INFINITY;
    for (int e = lane; e < E; e += 32) m = fmaxf(m, lr[e]);
    m = warp_max(m);
    float s = 0.f;
    for (int e = lane; e < E; e += 32) s += expf(lr[e] - m);
    s = warp_sum(s);
    for (int e = lane; e < E; e += 32) {
        float gt = 0.f, wsel = 0.f;
        bool sel = false;
#pragma unroll
        for (int j = 0; j < KK; ++j)
            if (j < k && ids[j] == e) { gt = gj[j]; wsel = wj[j]; sel = true; }
        const float dl = renorm ? (sel ? wsel * (gt - sg) : 0.f) : (expf(lr[e] - m) / s) * (gt - sg);
        sdl[e] = dl;
        dlogit[(size_t)t * E + e] = dl;
    }
}

constexpr int kWarps = 8;
constexpr int kTPW = 2;          // tokens per warp iteration (share every Wg^T vector load)

// K6.  Persistent blocks; Wg^T ([E][d] fp32) is staged once per block in shared memory when
// it fits (kSmemWg), else read through L1 from the transposed copy in global memory.
template <typename Elt, int KK, bool SMEM_WG>
__global__ void __launch_bounds__(kWarps * 32)
unpermute_gate_bwd_kernel(const Elt* __restrict__ dxe, const int* __restrict__ idx,
                          const int* __restrict__ slot, const float* __restrict__ wts,
                          const float* __restrict__ g, const float* __restrict__ logits,
                          const float* __restrict__ wg, const float* __restrict__ wgT,
                          const int* __restrict__ send_off, int renorm, int t0, int t1, int k, int d,
                          int E, Elt* __restrict__ dx, float* __restrict__ dlogit)
{
    extern __shared__ __align__(16) float ksm[];
    constexpr int V = Vec16<Elt>::N;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* sdl = ksm + (size_t)w * kTPW * E;          // [kTPW][E] per warp
    const float* W = wgT;
    if constexpr (SMEM_WG) {
        float* swt = ksm + (size_t)kWarps * kTPW * E;   // 16-byte aligned (kTPW*E*kWarps*4 % 16 == 0)
        for (int q = threadIdx.x; q < d * E / 4; q += blockDim.x)
            reinterpret_cast<float4*>(swt)[q] = __ldg(reinterpret_cast<const float4*>(wgT) + q);
        __syncthreads();
        W = swt;
    }
    const int nvec = d / V;
    const int step = gridDim.x * kWarps * kTPW;
    for (int tb = t0 + (blockIdx.x * kWarps + w) * kTPW; tb < t1; tb += step) {
        int rows[kTPW][KK];
#pragma unroll
        for (int q = 0; q < kTPW; ++q) {
            const int t = tb + q;
            if (t < t1) {
                int ids[KK];
                float wj[KK], gj[KK];
                choices<KK>(idx, slot, wts, g, send_off, t, k, lane, rows[q], wj, ids, gj);
                token_dlogit<KK>(logits, t, E, k, renorm, ids, wj, gj, lane, sdl + q * E, dlogit);
            } else {
#pragma unroll
                for (int j = 0; j < KK; ++j) rows[q][j] = -1;
                for (int e = lane; e < E; e += 32) sdl[q * E + e] = 0.f;
            }
        }
        __syncwarp();
        constexpr int U = 2;
        for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
            uint4 raw[kTPW][U][KK];
#pragma unroll
            for (int q = 0; q < kTPW; ++q)
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int j = 0; j < KK; ++j)
                        if (rows[q][j] >= 0 && v0 + 32 * u < nvec)
                            raw[q][u][j] = ld_nc_v4(reinterpret_cast<const uint4*>(dxe + (size_t)rows[q][j] * d) + v0 + 32 * u);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + 32 * u;
                if (v >= nvec) break;
                float acc[kTPW][V];
#pragma unroll
                for (int q = 0; q < kTPW; ++q) {
#pragma unroll
                    for (int i = 0; i < V; ++i) acc[q][i] = 0.f;
#pragma unroll
                    for (int j = 0; j < KK; ++j) {
                        if (rows[q][j] >= 0) {
                            float f[V];
                            unpack16<Elt>(raw[q][u][j], f);
#pragma unroll
                            for (int i = 0; i < V; ++i) acc[q][i] += f[i];
                        }
                    }
                }
                for (int e = 0; e < E; ++e) {
                    const float4* wt = reinterpret_cast<const float4*>(W + (size_t)e * d + (size_t)v * V);
                    float wv[V];
#pragma unroll
                    for (int h = 0; h < V / 4; ++h) {
                        const float4 w4 = SMEM_WG ? wt[h] : __ldg(wt + h);
                        wv[4 * h] = w4.x; wv[4 * h + 1] = w4.y; wv[4 * h + 2] = w4.z; wv[4 * h + 3] = w4.w;
                    }
#pragma unroll
                    for (int q = 0; q < kTPW; ++q) {
                        const float sv = sdl[q * E + e];
#pragma unroll
                        for (int i = 0; i < V; ++i) acc[q][i] = fmaf(sv, wv[i], acc[q][i]);
                    }
                }
#pragma unroll
                for (int q = 0; q < kTPW; ++q)
                    if (tb + q < t1) st_v4(reinterpret_cast<uint4*>(dx + (size_t)(tb + q) * d) + v, pack16<Elt>(acc[q]));
            }
        }
        __syncwarp();
    }
}

constexpr int kDwgTok = 64;      // tokens per partial block
constexpr int kDwgThreads = 256; // each thread owns 4 consecutive dims -> 1024 dims per block
constexpr int kDwgE = 8;         // experts per pass (32 accumulators per thread)
constexpr int kDwgU = 16;        // tokens whose loads are in flight together

template <typename Elt> struct Quad;                 // 4 consecutive elements
template <> struct Quad<bf16> {
    using T = uint2;
    static __device__ __forceinline__ void unpack(T v, float* f) {
        f[0] = __uint_as_float(v.x << 16); f[1] = __uint_as_float(v.x & 0xffff0000u);
        f[2] = __uint_as_float(v.y << 16); f[3] = __uint_as_float(v.y & 0xffff0000u);
    }
};
template <> struct Quad<float> {
    using T = uint4;
    static __device__ __forceinline__ void unpack(T v, float* f) {
        f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
        f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
    }
};

// K7 partials: block (token tile tb, dim slice, expert tile) -> partial[tb][d][E]
template <typename Elt>
__global__ void __launch_bounds__(kDwgThreads)
dwg_partial_kernel(const Elt* __restrict__ x, const float* __restrict__ dlogit, int T, int d,
                   int E, float* __restrict__ partial)
{
    using Q = Quad<Elt>;
    __shared__ __align__(16) float sdl[kDwgTok][kDwgE];
    const int i0 = (blockIdx.y * kDwgThreads + threadIdx.x) * 4;
    const int tb = blockIdx.x;
    const int e0 = blockIdx.z * kDwgE;
    const int ne = min(kDwgE, E - e0);
    const int tbeg = tb * kDwgTok, tend = min(T, tbeg + kDwgTok);
    for (int q = threadIdx.x; q < kDwgTok * kDwgE; q += kDwgThreads) {
        const int r = q / kDwgE, c = q % kDwgE, t = tbeg + r;
        sdl[r][c] = (t < tend && c < ne) ? dlogit[(size_t)t * E + e0 + c] : 0.f;
    }
    __syncthreads();
    if (i0 >= d) return;
    float acc[4][kDwgE];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < kDwgE; ++c) acc[a][c] = 0.f;
    for (int tt = tbeg; tt < tend; tt += kDwgU) {
        typename Q::T raw[kDwgU];
#pragma unroll
        for (int u = 0; u < kDwgU; ++u)
            if (tt + u < tend) raw[u] = __ldg(reinterpret_cast<const typename Q::T*>(x + (size_t)(tt + u) * d + i0));
#pragma unroll
        for (int u = 0; u < kDwgU; ++u) {
            if (tt + u >= tend) break;
            float xv[4];
            Q::unpack(raw[u], xv);
            const float4 l0 = *reinterpret_cast<const float4*>(&sdl[tt + u - tbeg][0]);
            const float4 l1 = *reinterpret_cast<const float4*>(&sdl[tt + u - tbeg][4]);
            const float lv[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < kDwgE; ++c) acc[a][c] = fmaf(xv[a], lv[c], acc[a][c]);
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        if (i0 + a >= d) break;
        float* out = partial + ((size_t)tb * d + i0 + a) * E + e0;
        for (int c = 0; c < ne; ++c) out[c] = acc[a][c];
    }
}

// Two-level deterministic reduction: block = 32 outputs x 8 warps; warp w sums partials
// b = w, w+8, ...; the 8 warp sums are added in warp order.
__global__ void __launch_bounds__(256)
dwg_reduce_kernel(const float* __restrict__ partial, int nb, int n_out, float* __restrict__ dwg)
{
    __shared__ float red[8][32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = blockIdx.x * 32 + lane;
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    if (q < n_out) {
        int b = w;
        for (; b + 24 < nb; b += 32) {
#pragma unroll
            for (int u = 0; u < 4; ++u) s[u] += partial[(size_t)(b + 8 * u) * n_out + q];
        }
        for (; b < nb; b += 8) s[0] += partial[(size_t)b * n_out + q];
    }
    red[w][lane] = (s[0] + s[1]) + (s[2] + s[3]);
    __syncthreads();
    if (w == 0 && q < n_out) {
        float r = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) r += red[i][lane];
        dwg[q] = r;
    }
}

__global__ void transpose_f32_kernel(const float* __restrict__ in, int rows, int cols,
                                     float* __restrict__ out)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= rows * cols) return;
    const int r = q / cols, c = q % cols;
    out[(size_t)c * rows + r] = in[q];
}

constexpr size_t kSmemWgMax = 96 * 1024;

}  // namespace

#define LANCET_DISPATCH_K(k, ...)                                             \
    do {                                                                      \
        if ((k) <= 1) { constexpr int KK = 1; __VA_ARGS__; }                  \
        else if ((k) <= 2) { constexpr int KK = 2; __VA_ARGS__; }             \
        else if ((k) <= 4) { constexpr int KK = 4; __VA_ARGS__; }             \
        else { constexpr int KK = 8; __VA_ARGS__; }                           \
    } while (0)

int launch_wg_transpose(const float* wg, int d, int E, float* wgT, cudaStream_t s)
{
    transpose_f32_kernel<<<ceil_div(d * E, 256), 256, 0, s>>>(wg, d, E, wgT);
    return 1;
}

bool gate_bwd_needs_wgT(int d, int E) { return (size_t)d * E * 4 > kSmemWgMax; }

template <typename Elt, int KK, bool SM>
static void launch_k6(const DispatchArgs& a, const void* dxe, const float* g, const float* logits,
                      const float* wg, const float* wgT, int renorm, void* dx, float* dlogit, int t0,
                      int t1, int num_sms, cudaStream_t s)
{
    const size_t smem = sizeof(float) * (kWarps * kTPW * a.E + (SM ? (size_t)a.d * a.E : 0));
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(unpermute_gate_bwd_kernel<Elt, KK, SM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kSmemWgMax + 16 * 1024));
        attr = true;
    }
    const int need = ceil_div(t1 - t0, kWarps * kTPW);
    const int grid = std::max(1, std::min(need, 2 * num_sms));
    unpermute_gate_bwd_kernel<Elt, KK, SM><<<grid, kWarps * 32, smem, s>>>(
        (const Elt*)dxe, a.idx, a.slot, a.w, g, logits, wg, wgT, a.send_off, renorm, t0, t1, a.k, a.d, a.E,
        (Elt*)dx, dlogit);
}

int launch_unpermute_gate_bwd(const DispatchArgs& a, const void* dxe, const float* g,
                              const float* logits, const float* wg, const float* wgT, int renorm,
                              void* dx, float* dlogit, int t0, int t1, int num_sms, bool is_bf16,
                              cudaStream_t s)
{
    if (t1 <= t0) return 0;
    const bool sm = !gate_bwd_needs_wgT(a.d, a.E);
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16) {
            if (sm) launch_k6<bf16, KK, true>(a, dxe, g, logits, wg, wgT, renorm, dx, dlogit, t0, t1, num_sms, s);
            else launch_k6<bf16, KK, false>(a, dxe, g, logits, wg, wgT, renorm, dx, dlogit, t0, t1, num_sms, s);
        } else {
            if (sm) launch_k6<float, KK, true>(a, dxe, g, logits, wg, wgT, renorm, dx, dlogit, t0, t1, num_sms, s);
            else launch_k6<float, KK, false>(a, dxe, g, logits, wg, wgT, renorm, dx, dlogit, t0, t1, num_sms, s);
        }
    });
    return 1;
}

size_t dwg_partial_floats(int T, int d, int E) { return (size_t)ceil_div(T, kDwgTok) * d * E; }

int launch_dwg(const void* x, const float* dlogit, int T, int d, int E, float* partial,
               float* dwg, bool is_bf16, cudaStream_t s)
{
    const int nb = ceil_div(T, kDwgTok);
    dim3 grid(nb, ceil_div(d, kDwgThreads * 4), ceil_div(E, kDwgE));
    if (is_bf16)
        dwg_partial_kernel<bf16><<<grid, kDwgThreads, 0, s>>>((const bf16*)x, dlogit, T, d, E, partial);
    else
        dwg_partial_kernel<float><<<grid, kDwgThreads, 0, s>>>((const float*)x, dlogit, T, d, E, partial);
    dwg_reduce_kernel<<<ceil_div(d * E, 32), 256, 0, s>>>(partial, nb, d * E, dwg);
    return 2;
}

}  // namespace lancet
