// gate_bwd.cu -- K6 (dispatch backward + gate term of dx) and K7 (dWg) of the MoE layer.
//
//   dx_t     = sum_{admitted j} dX[row_tj] + sum_e dlogit_te Wg[:, e]
//   dWg      = x^T dlogit     (local; the data-parallel all-reduce of the replicated gate,
//                              P:L110, is the caller's)
// dlogit (softmax Jacobian, R3) and the packed source rows row_tj are produced by
// K5 (combine_bwd_kernel, dispatch.cu), which already holds g_tj for the token.
// Top-k and capacity decisions are piecewise constant and carry no gradient.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace lancet {

namespace {

constexpr int kWarps = 8;
constexpr size_t kSmemWgMax = 64 * 1024;

// K6: each warp handles two tokens per pass, lanes over 16-byte vectors of dims; all row loads
// of the pass are issued before use (like the combine).  The gate term reads Wg^T ([E][d] fp32)
// from shared memory, staged once per persistent block in an interleaved layout
// [e][h][v][4] (h = which half of the lane's 8 dims) so a warp's 16-byte reads are contiguous
// (bank-conflict free), and each Wg^T vector serves both tokens.  dlogit_te is held by lane e
// and broadcast with shuffles.  Falls back to L1 reads of the plain [E][d] layout when the
// gate does not fit in shared memory.
constexpr int kK6T = 2;

template <typename Elt, int KK, bool SMEM_WG>
__global__ void __launch_bounds__(kWarps * 32)
k6_gather_kernel(const Elt* __restrict__ dxe, const int* __restrict__ prow,
                 const float* __restrict__ dlogit, const float* __restrict__ wgT, int t0, int t1,
                 int k, int d, int E, Elt* __restrict__ dx)
{
    extern __shared__ __align__(16) float swt[];
    constexpr int V = Vec16<Elt>::N;                   // dims per 16-byte vector (8 bf16 / 4 fp32)
    constexpr int H = V / 4;                           // float4 pieces of Wg per vector
    constexpr int U = 2;                               // vectors per lane per pass
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nvec = d / V;
    if constexpr (SMEM_WG) {
        // swt[((e * H + h) * nvec + v) * 4 + c] = Wg^T[e][v * V + 4 h + c]
        for (int q = threadIdx.x; q < E * nvec * H; q += blockDim.x) {
            const int e = q / (nvec * H), r = q % (nvec * H), v = r / H, h = r % H;
            reinterpret_cast<float4*>(swt)[(e * H + h) * nvec + v] =
                __ldg(reinterpret_cast<const float4*>(wgT + (size_t)e * d + (size_t)v * V) + h);
        }
        __syncthreads();
    }
    const int step = gridDim.x * kWarps * kK6T;
    for (int tb = t0 + (blockIdx.x * kWarps + w) * kK6T; tb < t1; tb += step) {
        int rows[kK6T][KK];
        float dl_lane[kK6T];
#pragma unroll
        for (int q = 0; q < kK6T; ++q) {
            const int t = tb + q;
            const bool ok = t < t1;
            const int myrow = (ok && lane < k) ? prow[(size_t)t * k + lane] : -1;
#pragma unroll
            for (int j = 0; j < KK; ++j) rows[q][j] = __shfl_sync(0xffffffffu, myrow, j);
            dl_lane[q] = (ok && lane < E) ? __ldg(dlogit + (size_t)t * E + lane) : 0.f;
        }
        for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
            uint4 raw[kK6T][U][KK];
#pragma unroll
            for (int q = 0; q < kK6T; ++q)
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int j = 0; j < KK; ++j)
                        if (rows[q][j] >= 0 && v0 + 32 * u < nvec)
                            raw[q][u][j] = ld_nc_v4(reinterpret_cast<const uint4*>(dxe + (size_t)rows[q][j] * d) + v0 + 32 * u);
            float acc[kK6T][U][V];
#pragma unroll
            for (int q = 0; q < kK6T; ++q)
#pragma unroll
                for (int u = 0; u < U; ++u) {
#pragma unroll
                    for (int i = 0; i < V; ++i) acc[q][u][i] = 0.f;
#pragma unroll
                    for (int j = 0; j < KK; ++j) {
                        if (rows[q][j] >= 0 && v0 + 32 * u < nvec) {
                            float f[V];
                            unpack16<Elt>(raw[q][u][j], f);
#pragma unroll
                            for (int i = 0; i < V; ++i) acc[q][u][i] += f[i];
                        }
                    }
                }
            for (int e = 0; e < E; ++e) {
                float sv[kK6T];                        // dlogit_te: lane e holds it when E <= 32
#pragma unroll
                for (int q = 0; q < kK6T; ++q)
                    sv[q] = E <= 32 ? __shfl_sync(0xffffffffu, dl_lane[q], e)
                                    : (tb + q < t1 ? __ldg(dlogit + (size_t)(tb + q) * E + e) : 0.f);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int v = v0 + 32 * u;
                    if (v >= nvec) break;
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        const float4 w4 = SMEM_WG
                            ? reinterpret_cast<const float4*>(swt)[(e * H + h) * nvec + v]
                            : __ldg(reinterpret_cast<const float4*>(wgT + (size_t)e * d + (size_t)v * V) + h);
#pragma unroll
                        for (int q = 0; q < kK6T; ++q) {
                            acc[q][u][4 * h + 0] = fmaf(sv[q], w4.x, acc[q][u][4 * h + 0]);
                            acc[q][u][4 * h + 1] = fmaf(sv[q], w4.y, acc[q][u][4 * h + 1]);
                            acc[q][u][4 * h + 2] = fmaf(sv[q], w4.z, acc[q][u][4 * h + 2]);
                            acc[q][u][4 * h + 3] = fmaf(sv[q], w4.w, acc[q][u][4 * h + 3]);
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kK6T; ++q)
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (tb + q < t1 && v0 + 32 * u < nvec)
                        st_v4(reinterpret_cast<uint4*>(dx + (size_t)(tb + q) * d) + v0 + 32 * u, pack16<Elt>(acc[q][u]));
        }
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
#pragma unroll
        for (int c = 0; c < kDwgE; ++c)
            if (c < ne) out[c] = acc[a][c];
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

bool gate_bwd_needs_wgT(int, int) { return true; }

template <typename Elt, int KK, bool SM>
static void launch_k6(const DispatchArgs& a, const void* dxe, const int* prow, const float* dlogit,
                      const float* wgT, void* dx, int t0, int t1, int num_sms, cudaStream_t s)
{
    const size_t smem = SM ? sizeof(float) * (size_t)a.d * a.E : 0;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k6_gather_kernel<Elt, KK, SM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kSmemWgMax);
        attr = true;
    }
    const int need = ceil_div(t1 - t0, kWarps * kK6T);
    const int grid = std::max(1, std::min(need, 4 * num_sms));
    k6_gather_kernel<Elt, KK, SM><<<grid, kWarps * 32, smem, s>>>((const Elt*)dxe, prow, dlogit, wgT, t0, t1,
                                                                  a.k, a.d, a.E, (Elt*)dx);
}

int launch_unpermute_gate_bwd(const DispatchArgs& a, const void* dxe, const int* prow,
                              const float* dlogit, const float* wgT, void* dx, int t0, int t1,
                              int num_sms, bool is_bf16, cudaStream_t s)
{
    if (t1 <= t0) return 0;
    const bool sm = (size_t)a.d * a.E * 4 <= kSmemWgMax;
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16) {
            if (sm) launch_k6<bf16, KK, true>(a, dxe, prow, dlogit, wgT, dx, t0, t1, num_sms, s);
            else launch_k6<bf16, KK, false>(a, dxe, prow, dlogit, wgT, dx, t0, t1, num_sms, s);
        } else {
            if (sm) launch_k6<float, KK, true>(a, dxe, prow, dlogit, wgT, dx, t0, t1, num_sms, s);
            else launch_k6<float, KK, false>(a, dxe, prow, dlogit, wgT, dx, t0, t1, num_sms, s);
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
