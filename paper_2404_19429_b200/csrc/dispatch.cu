// dispatch.cu -- data movement of the MoE layer and the gate backward.
//
// K3 permute:   "The tokens are re-arranged according to their target experts":
//               row x[t] -> xs[off_e + slot] for every admitted (t, j); one warp per token,
//               all 16-byte loads of the row issued before the k stores.  Expert e's rows of
//               chunk c are the contiguous range [off_e + S[e][c], off_e + S[e][c+1]) -- the
//               chunk's send message needs no repacking.
// K4 combine:   "Reverting tokens to their original order yields the MoE layer's output"
//               (gather): y_t = sum_{admitted j} w_tj o_tj as an fp32 fma chain
//               over j in order, dropped choices contribute 0 (R6).
// K5 combine backward:  g_tj = <dy_t, o_tj>, dcomb[off_e + slot] = w_tj dy_t.
// K6 dispatch backward + gate:  dx_t = sum_{admitted j} dX_e[off_e + slot]
//               + sum_e dlogit_te Wg[:, e], with dlogit from the softmax Jacobian (R3).
// K7 dWg = x^T dlogit (two-pass deterministic reduction over tokens).
//
// All token kernels are templated on KK >= k (compile-time top-k width) so a lane keeps the
// k source/destination rows of its vectors in registers and issues every load of an
// iteration before the first use (memory-level parallelism is what bounds them).
#include "common.cuh"
#include "kernels.h"

namespace lancet {

constexpr int kWarpsPerBlock = 8;

// rows[j] = packed row of choice j (-1 dropped or j >= k); wj[j] = combine weight; ids[j] = expert
template <int KK>
__device__ __forceinline__ void load_choices(const int* __restrict__ idx, const int* __restrict__ slot,
                                             const float* __restrict__ wts, const int* __restrict__ send_off,
                                             int t, int k, int lane, int (&rows)[KK], float (&wj)[KK],
                                             int (&ids)[KK])
{
    int myrow = -1, myidx = -1;
    float myw = 0.f;
    if (lane < k) {
        const int s = slot[(size_t)t * k + lane];
        myidx = idx[(size_t)t * k + lane];
        myrow = s >= 0 ? send_off[myidx] + s : -1;
        if (wts) myw = wts[(size_t)t * k + lane];
    }
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        rows[j] = __shfl_sync(0xffffffffu, myrow, j);
        wj[j] = __shfl_sync(0xffffffffu, myw, j);
        ids[j] = __shfl_sync(0xffffffffu, myidx, j);
        if (j >= k) rows[j] = -1;
    }
}

template <typename Elt, int KK>
__global__ void __launch_bounds__(256)
permute_kernel(const Elt* __restrict__ x, const int* __restrict__ idx, const int* __restrict__ slot,
               int T, int k, int d, const int* __restrict__ send_off,
               const int* __restrict__ send_rows, Elt* __restrict__ xs, int tok_blocks)
{
    constexpr int V = Vec16<Elt>::N;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nvec = d / V;
    if ((int)blockIdx.x < tok_blocks) {
        const int t = blockIdx.x * kWarpsPerBlock + w;
        if (t >= T) return;
        int rows[KK], ids[KK];
        float wj[KK];
        load_choices<KK>(idx, slot, nullptr, send_off, t, k, lane, rows, wj, ids);
        const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)t * d);
        constexpr int U = 4;
        for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
            uint4 val[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (v0 + 32 * u < nvec) val[u] = ld_nc_v4(src + v0 + 32 * u);
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                if (rows[j] >= 0) {
                    uint4* dst = reinterpret_cast<uint4*>(xs + (size_t)rows[j] * d);
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (v0 + 32 * u < nvec) st_v4(dst + v0 + 32 * u, val[u]);
                }
            }
        }
    } else {
        // zero the pad rows [off_e + rows_e, off_e + round_up(rows_e, 128)) of expert e
        const int e = blockIdx.x - tok_blocks;
        const int r0 = send_off[e] + send_rows[e];
        const int r1 = send_off[e] + round_up(send_rows[e], kRowAlign);
        for (int r = r0 + w; r < r1; r += kWarpsPerBlock) {
            uint4* dst = reinterpret_cast<uint4*>(xs + (size_t)r * d);
            for (int v = lane; v < nvec; v += 32) st_v4(dst + v, make_uint4(0, 0, 0, 0));
        }
    }
}

template <typename Elt, int KK>
__global__ void __launch_bounds__(256)
combine_kernel(const Elt* __restrict__ comb, const int* __restrict__ idx,
               const int* __restrict__ slot, const float* __restrict__ wts,
               const int* __restrict__ send_off, int t0, int t1, int k, int d,
               Elt* __restrict__ y)
{
    constexpr int V = Vec16<Elt>::N;
    constexpr int U = 2;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = t0 + blockIdx.x * kWarpsPerBlock + w;
    if (t >= t1) return;
    int rows[KK], ids[KK];
    float wj[KK];
    load_choices<KK>(idx, slot, wts, send_off, t, k, lane, rows, wj, ids);
    const int nvec = d / V;
    uint4* dst = reinterpret_cast<uint4*>(y + (size_t)t * d);
    for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
        uint4 raw[U][KK];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < KK; ++j)
                if (rows[j] >= 0 && v0 + 32 * u < nvec)
                    raw[u][j] = ld_nc_v4(reinterpret_cast<const uint4*>(comb + (size_t)rows[j] * d) + v0 + 32 * u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (v0 + 32 * u >= nvec) break;
            float acc[V];
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] = 0.f;
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                if (rows[j] >= 0) {
                    float f[V];
                    unpack16<Elt>(raw[u][j], f);
#pragma unroll
                    for (int q = 0; q < V; ++q) acc[q] = __fmaf_rn(wj[j], f[q], acc[q]);
                }
            }
            st_v4(dst + v0 + 32 * u, pack16<Elt>(acc));
        }
    }
}

template <typename Elt, int KK>
__global__ void __launch_bounds__(256)
combine_bwd_kernel(const Elt* __restrict__ dy, const Elt* __restrict__ comb,
                   const int* __restrict__ idx, const int* __restrict__ slot,
                   const float* __restrict__ wts, const int* __restrict__ send_off,
                   const int* __restrict__ send_rows, int t0, int t1, int k, int d,
                   float* __restrict__ g, Elt* __restrict__ dcomb, int tok_blocks)
{
    constexpr int V = Vec16<Elt>::N;
    constexpr int U = 2;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nvec = d / V;
    if ((int)blockIdx.x >= tok_blocks) {
        const int e = blockIdx.x - tok_blocks;
        const int r0 = send_off[e] + send_rows[e];
        const int r1 = send_off[e] + round_up(send_rows[e], kRowAlign);
        for (int r = r0 + w; r < r1; r += kWarpsPerBlock) {
            uint4* dst = reinterpret_cast<uint4*>(dcomb + (size_t)r * d);
            for (int v = lane; v < nvec; v += 32) st_v4(dst + v, make_uint4(0, 0, 0, 0));
        }
        return;
    }
    const int t = t0 + blockIdx.x * kWarpsPerBlock + w;
    if (t >= t1) return;
    int rows[KK], ids[KK];
    float wj[KK], part[KK];
    load_choices<KK>(idx, slot, wts, send_off, t, k, lane, rows, wj, ids);
#pragma unroll
    for (int j = 0; j < KK; ++j) part[j] = 0.f;
    const uint4* dyr = reinterpret_cast<const uint4*>(dy + (size_t)t * d);
    for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
        uint4 rdy[U], ro[U][KK];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (v0 + 32 * u < nvec) {
                rdy[u] = ld_nc_v4(dyr + v0 + 32 * u);
#pragma unroll
                for (int j = 0; j < KK; ++j)
                    if (rows[j] >= 0)
                        ro[u][j] = ld_nc_v4(reinterpret_cast<const uint4*>(comb + (size_t)rows[j] * d) + v0 + 32 * u);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (v0 + 32 * u >= nvec) break;
            float fdy[V];
            unpack16<Elt>(rdy[u], fdy);
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                if (rows[j] >= 0) {
                    float fo[V], sc[V];
                    unpack16<Elt>(ro[u][j], fo);
#pragma unroll
                    for (int q = 0; q < V; ++q) {
                        part[j] = fmaf(fdy[q], fo[q], part[j]);
                        sc[q] = wj[j] * fdy[q];
                    }
                    st_v4(reinterpret_cast<uint4*>(dcomb + (size_t)rows[j] * d) + v0 + 32 * u, pack16<Elt>(sc));
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        if (j < k) {
            const float s = warp_sum(part[j]);
            if (lane == 0) g[(size_t)t * k + j] = rows[j] >= 0 ? s : 0.f;
        }
    }
}

// K6: kTPW tokens per warp so each transposed-Wg vector is reused kTPW times.
constexpr int kTPW = 4;

template <typename Elt, int KK>
__global__ void __launch_bounds__(256)
unpermute_gate_bwd_kernel(const Elt* __restrict__ dxe, const int* __restrict__ idx,
                          const int* __restrict__ slot, const float* __restrict__ wts,
                          const float* __restrict__ g, const float* __restrict__ logits,
                          const float* __restrict__ wgT, const int* __restrict__ send_off,
                          int renorm, int t0, int t1, int k, int d, int E,
                          Elt* __restrict__ dx, float* __restrict__ dlogit)
{
    extern __shared__ float sdl_all[];                 // [warps][kTPW][E]
    constexpr int V = Vec16<Elt>::N;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tb = t0 + (blockIdx.x * kWarpsPerBlock + w) * kTPW;
    if (tb >= t1) return;
    float* sdl = sdl_all + (size_t)w * kTPW * E;
    int rows[kTPW][KK];
    bool valid[kTPW];
#pragma unroll
    for (int q = 0; q < kTPW; ++q) {
        const int t = tb + q;
        valid[q] = t < t1;
        int ids[KK];
        float wj[KK];
        if (valid[q]) {
            load_choices<KK>(idx, slot, wts, send_off, t, k, lane, rows[q], wj, ids);
            const float myg = lane < k ? g[(size_t)t * k + lane] : 0.f;
            float gj[KK];
            float sg = 0.f;                               // sum_j g_j w_j
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                gj[j] = __shfl_sync(0xffffffffu, myg, j);
                if (j < k) sg = fmaf(gj[j], wj[j], sg);
            }
            // softmax Jacobian (R3): dlogit_e = p_e (g~_e - sg), or renormalised at the selected e
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
                sdl[q * E + e] = dl;
                dlogit[(size_t)t * E + e] = dl;
            }
        } else {
#pragma unroll
            for (int j = 0; j < KK; ++j) rows[q][j] = -1;
            for (int e = lane; e < E; e += 32) sdl[q * E + e] = 0.f;
        }
    }
    __syncwarp();
    const int nvec = d / V;
    for (int v = lane; v < nvec; v += 32) {
        float acc[kTPW][V];
        uint4 raw[kTPW][KK];
#pragma unroll
        for (int q = 0; q < kTPW; ++q)
#pragma unroll
            for (int j = 0; j < KK; ++j)
                if (rows[q][j] >= 0)
                    raw[q][j] = ld_nc_v4(reinterpret_cast<const uint4*>(dxe + (size_t)rows[q][j] * d) + v);
#pragma unroll
        for (int q = 0; q < kTPW; ++q) {
#pragma unroll
            for (int i = 0; i < V; ++i) acc[q][i] = 0.f;
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                if (rows[q][j] >= 0) {
                    float f[V];
                    unpack16<Elt>(raw[q][j], f);
#pragma unroll
                    for (int i = 0; i < V; ++i) acc[q][i] += f[i];
                }
            }
        }
        // gate term: sum_e dlogit_e Wg[i][e]; Wg read transposed ([E][d]) so lanes coalesce
        for (int e = 0; e < E; ++e) {
            const float4* wt = reinterpret_cast<const float4*>(wgT + (size_t)e * d + (size_t)v * V);
            float wv[V];
#pragma unroll
            for (int h = 0; h < V / 4; ++h) {
                const float4 w4 = __ldg(wt + h);
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
            if (valid[q]) st_v4(reinterpret_cast<uint4*>(dx + (size_t)(tb + q) * d) + v, pack16<Elt>(acc[q]));
    }
}

// ---- K6 + K7 fused (E <= 8) --------------------------------------------------------------
// Block = 64 tokens x 1024 dims.  Prologue: one warp per token computes dlogit (softmax
// Jacobian, R3) into shared memory.  Main loop: thread owns 4 consecutive dims, keeps
// Wg[i0..i0+3][0..E) and its dWg partial in registers, and streams the block's tokens:
//   dx_t[i]  = sum_j dX[row_tj][i] + sum_e dlogit_te Wg[i][e]
//   dWg[i][e] += x_t[i] dlogit_te        (partial per block; reduced by dwg_reduce_kernel)
constexpr int kFTok = 64;
constexpr int kFThreads = 256;
constexpr int kFU = 4;           // tokens whose loads are in flight together

template <typename Elt> struct Quad;                 // 4 consecutive elements
template <> struct Quad<bf16> {
    using T = uint2;
    static __device__ __forceinline__ void unpack(T v, float* f) {
        f[0] = __uint_as_float(v.x << 16); f[1] = __uint_as_float(v.x & 0xffff0000u);
        f[2] = __uint_as_float(v.y << 16); f[3] = __uint_as_float(v.y & 0xffff0000u);
    }
    static __device__ __forceinline__ T pack(const float* f) {
        __nv_bfloat162 a = __floats2bfloat162_rn(f[0], f[1]), b = __floats2bfloat162_rn(f[2], f[3]);
        return make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
    }
};
template <> struct Quad<float> {
    using T = uint4;
    static __device__ __forceinline__ void unpack(T v, float* f) {
        f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
        f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
    }
    static __device__ __forceinline__ T pack(const float* f) {
        return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
    }
};

template <typename Elt, int KK>
__global__ void __launch_bounds__(kFThreads)
gate_bwd_fused_kernel(const Elt* __restrict__ dxe, const Elt* __restrict__ x,
                      const int* __restrict__ idx, const int* __restrict__ slot,
                      const float* __restrict__ wts, const float* __restrict__ g,
                      const float* __restrict__ logits, const float* __restrict__ wg,
                      const int* __restrict__ send_off, int renorm, int t0, int t1, int k, int d,
                      int E, Elt* __restrict__ dx, float* __restrict__ partial, int pbase)
{
    using Q = Quad<Elt>;
    __shared__ float sdl[kFTok][8];
    __shared__ int srow[kFTok][KK];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tb = t0 + blockIdx.x * kFTok;
    const int tn = min(kFTok, t1 - tb);
    for (int q = w; q < kFTok; q += kFThreads / 32) {
        const int t = tb + q;
        if (q >= tn) {
            if (lane < 8) sdl[q][lane] = 0.f;
            if (lane < KK) srow[q][lane] = -1;
            continue;
        }
        int rows[KK], ids[KK];
        float wj[KK];
        load_choices<KK>(idx, slot, wts, send_off, t, k, lane, rows, wj, ids);
        const float myg = lane < k ? g[(size_t)t * k + lane] : 0.f;
        float gj[KK];
        float sg = 0.f;
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            gj[j] = __shfl_sync(0xffffffffu, myg, j);
            if (j < k) sg = fmaf(gj[j], wj[j], sg);
        }
        const float* lr = logits + (size_t)t * E;
        const float l = lane < E ? lr[lane] : -INFINITY;
        const float m = warp_max(l);
        const float ex = lane < E ? expf(l - m) : 0.f;
        const float s = warp_sum(ex);
        float gt = 0.f, wsel = 0.f;
        bool sel = false;
#pragma unroll
        for (int j = 0; j < KK; ++j)
            if (j < k && ids[j] == lane) { gt = gj[j]; wsel = wj[j]; sel = true; }
        const float dl = renorm ? (sel ? wsel * (gt - sg) : 0.f) : (ex / s) * (gt - sg);
        if (lane < 8) sdl[q][lane] = lane < E ? dl : 0.f;
        if (lane < KK) srow[q][lane] = rows[lane];
    }
    __syncthreads();
    const int i0 = (blockIdx.y * kFThreads + threadIdx.x) * 4;
    if (i0 >= d) return;
    float wgr[4][8], acc[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            wgr[a][e] = e < E ? wg[(size_t)(i0 + a) * E + e] : 0.f;
            acc[a][e] = 0.f;
        }
    for (int q0 = 0; q0 < tn; q0 += kFU) {
        typename Q::T rx[kFU], rd[kFU][KK];
#pragma unroll
        for (int u = 0; u < kFU; ++u) {
            const int q = q0 + u;
            if (q < tn) {
                rx[u] = __ldg(reinterpret_cast<const typename Q::T*>(x + (size_t)(tb + q) * d + i0));
#pragma unroll
                for (int j = 0; j < KK; ++j) {
                    const int row = srow[q][j];
                    if (row >= 0) rd[u][j] = __ldg(reinterpret_cast<const typename Q::T*>(dxe + (size_t)row * d + i0));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kFU; ++u) {
            const int q = q0 + u;
            if (q >= tn) break;
            float dl[8];
            const float4 l0 = *reinterpret_cast<const float4*>(&sdl[q][0]);
            const float4 l1 = *reinterpret_cast<const float4*>(&sdl[q][4]);
            dl[0] = l0.x; dl[1] = l0.y; dl[2] = l0.z; dl[3] = l0.w;
            dl[4] = l1.x; dl[5] = l1.y; dl[6] = l1.z; dl[7] = l1.w;
            float o[4] = {0.f, 0.f, 0.f, 0.f}, xf[4];
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                if (srow[q][j] >= 0) {
                    float f[4];
                    Q::unpack(rd[u][j], f);
#pragma unroll
                    for (int a = 0; a < 4; ++a) o[a] += f[a];
                }
            }
            Q::unpack(rx[u], xf);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    o[a] = fmaf(dl[e], wgr[a][e], o[a]);
                    acc[a][e] = fmaf(xf[a], dl[e], acc[a][e]);
                }
            *reinterpret_cast<typename Q::T*>(dx + (size_t)(tb + q) * d + i0) = Q::pack(o);
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        float* out = partial + ((size_t)(pbase + blockIdx.x) * d + i0 + a) * E;
        for (int e = 0; e < E; ++e) out[e] = acc[a][e];
    }
}

constexpr int kDwgTok = 64;      // tokens per partial block
constexpr int kDwgThreads = 256; // each thread owns 4 consecutive dims -> 1024 dims per block
constexpr int kDwgE = 8;         // experts per pass (32 accumulators per thread)
constexpr int kDwgU = 8;         // tokens whose loads are in flight together

template <typename Elt>
__global__ void __launch_bounds__(kDwgThreads)
dwg_partial_kernel(const Elt* __restrict__ x, const float* __restrict__ dlogit, int T, int d,
                   int E, float* __restrict__ partial)
{
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
        float xv[kDwgU][4];
#pragma unroll
        for (int u = 0; u < kDwgU; ++u) {
            const int t = tt + u;
            if (t < tend) {
                if constexpr (sizeof(Elt) == 2) {
                    const uint2 raw = __ldg(reinterpret_cast<const uint2*>(x + (size_t)t * d + i0));
                    xv[u][0] = __uint_as_float(raw.x << 16); xv[u][1] = __uint_as_float(raw.x & 0xffff0000u);
                    xv[u][2] = __uint_as_float(raw.y << 16); xv[u][3] = __uint_as_float(raw.y & 0xffff0000u);
                } else {
                    const float4 f4 = __ldg(reinterpret_cast<const float4*>(x + (size_t)t * d + i0));
                    xv[u][0] = f4.x; xv[u][1] = f4.y; xv[u][2] = f4.z; xv[u][3] = f4.w;
                }
            } else {
                xv[u][0] = xv[u][1] = xv[u][2] = xv[u][3] = 0.f;
            }
        }
#pragma unroll
        for (int u = 0; u < kDwgU; ++u) {
            if (tt + u >= tend) break;
            const float4 l0 = *reinterpret_cast<const float4*>(&sdl[tt + u - tbeg][0]);
            const float4 l1 = *reinterpret_cast<const float4*>(&sdl[tt + u - tbeg][4]);
            const float lv[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < kDwgE; ++c) acc[a][c] = fmaf(xv[u][a], lv[c], acc[a][c]);
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        if (i0 + a >= d) break;
        float* out = partial + ((size_t)tb * d + i0 + a) * E + e0;
        for (int c = 0; c < ne; ++c) out[c] = acc[a][c];
    }
}

__global__ void dwg_reduce_kernel(const float* __restrict__ partial, int nb, int d, int E,
                                  float* __restrict__ dwg)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= d * E) return;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int b = 0;
    for (; b + 4 <= nb; b += 4) {
        s0 += partial[(size_t)b * d * E + q];
        s1 += partial[(size_t)(b + 1) * d * E + q];
        s2 += partial[(size_t)(b + 2) * d * E + q];
        s3 += partial[(size_t)(b + 3) * d * E + q];
    }
    for (; b < nb; ++b) s0 += partial[(size_t)b * d * E + q];
    dwg[q] = (s0 + s1) + (s2 + s3);
}

__global__ void transpose_f32_kernel(const float* __restrict__ in, int rows, int cols,
                                     float* __restrict__ out)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= rows * cols) return;
    const int r = q / cols, c = q % cols;
    out[(size_t)c * rows + r] = in[q];
}

__global__ void zero_pads_kernel(char* __restrict__ buf, int row_bytes,
                                 const int* __restrict__ grp_off, const int* __restrict__ grp_rows)
{
    const int g = blockIdx.x;
    const int r0 = grp_off[g] + grp_rows[g];
    const int r1 = grp_off[g] + round_up(grp_rows[g], kRowAlign);
    const int nv = row_bytes / 16;
    for (int q = threadIdx.x; q < (r1 - r0) * nv; q += blockDim.x) {
        const int r = r0 + q / nv, v = q % nv;
        st_v4(buf + (size_t)r * row_bytes + (size_t)v * 16, make_uint4(0, 0, 0, 0));
    }
}

// ---- launchers ---------------------------------------------------------------------------
// dispatch on KK = the smallest of {1, 2, 4, 8} >= k
#define LANCET_DISPATCH_K(k, ...)                                             \
    do {                                                                      \
        if ((k) <= 1) { constexpr int KK = 1; __VA_ARGS__; }                  \
        else if ((k) <= 2) { constexpr int KK = 2; __VA_ARGS__; }             \
        else if ((k) <= 4) { constexpr int KK = 4; __VA_ARGS__; }             \
        else { constexpr int KK = 8; __VA_ARGS__; }                           \
    } while (0)

int launch_permute(const DispatchArgs& a, const void* x, void* xs, bool is_bf16, cudaStream_t s)
{
    const int tok_blocks = ceil_div(a.T, kWarpsPerBlock);
    const int grid = tok_blocks + a.E;
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16)
            permute_kernel<bf16, KK><<<grid, 256, 0, s>>>((const bf16*)x, a.idx, a.slot, a.T, a.k, a.d,
                                                         a.send_off, a.send_rows, (bf16*)xs, tok_blocks);
        else
            permute_kernel<float, KK><<<grid, 256, 0, s>>>((const float*)x, a.idx, a.slot, a.T, a.k, a.d,
                                                          a.send_off, a.send_rows, (float*)xs, tok_blocks);
    });
    return 1;
}

int launch_combine(const DispatchArgs& a, const void* comb, void* y, int t0, int t1, bool is_bf16,
                   cudaStream_t s)
{
    if (t1 <= t0) return 0;
    const int grid = ceil_div(t1 - t0, kWarpsPerBlock);
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16)
            combine_kernel<bf16, KK><<<grid, 256, 0, s>>>((const bf16*)comb, a.idx, a.slot, a.w, a.send_off,
                                                         t0, t1, a.k, a.d, (bf16*)y);
        else
            combine_kernel<float, KK><<<grid, 256, 0, s>>>((const float*)comb, a.idx, a.slot, a.w,
                                                          a.send_off, t0, t1, a.k, a.d, (float*)y);
    });
    return 1;
}

int launch_combine_bwd(const DispatchArgs& a, const void* dy, const void* comb, float* g,
                       void* dcomb, int t0, int t1, bool zero_pads, bool is_bf16, cudaStream_t s)
{
    const int tok_blocks = ceil_div(t1 - t0, kWarpsPerBlock);
    const int grid = tok_blocks + (zero_pads ? a.E : 0);
    if (grid == 0) return 0;
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16)
            combine_bwd_kernel<bf16, KK><<<grid, 256, 0, s>>>((const bf16*)dy, (const bf16*)comb, a.idx,
                                                             a.slot, a.w, a.send_off, a.send_rows, t0, t1,
                                                             a.k, a.d, g, (bf16*)dcomb, tok_blocks);
        else
            combine_bwd_kernel<float, KK><<<grid, 256, 0, s>>>((const float*)dy, (const float*)comb, a.idx,
                                                              a.slot, a.w, a.send_off, a.send_rows, t0, t1,
                                                              a.k, a.d, g, (float*)dcomb, tok_blocks);
    });
    return 1;
}

int launch_wg_transpose(const float* wg, int d, int E, float* wgT, cudaStream_t s)
{
    transpose_f32_kernel<<<ceil_div(d * E, 256), 256, 0, s>>>(wg, d, E, wgT);
    return 1;
}

int launch_unpermute_gate_bwd(const DispatchArgs& a, const void* dxe, const float* g,
                              const float* logits, const float* wgT, int renorm, void* dx,
                              float* dlogit, int t0, int t1, bool is_bf16, cudaStream_t s)
{
    if (t1 <= t0) return 0;
    const int grid = ceil_div(t1 - t0, kWarpsPerBlock * kTPW);
    const size_t smem = sizeof(float) * kWarpsPerBlock * kTPW * a.E;
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16)
            unpermute_gate_bwd_kernel<bf16, KK><<<grid, 256, smem, s>>>(
                (const bf16*)dxe, a.idx, a.slot, a.w, g, logits, wgT, a.send_off, renorm, t0, t1, a.k,
                a.d, a.E, (bf16*)dx, dlogit);
        else
            unpermute_gate_bwd_kernel<float, KK><<<grid, 256, smem, s>>>(
                (const float*)dxe, a.idx, a.slot, a.w, g, logits, wgT, a.send_off, renorm, t0, t1, a.k,
                a.d, a.E, (float*)dx, dlogit);
    });
    return 1;
}

size_t dwg_partial_floats(int T, int d, int E)
{
    return (size_t)(ceil_div(T, kDwgTok > kFTok ? kFTok : kDwgTok) + kMaxChunks) * d * E;
}

int launch_gate_bwd_fused(const DispatchArgs& a, const void* dxe, const void* x, const float* g,
                          const float* logits, const float* wg, int renorm, void* dx, float* partial,
                          int pbase, int t0, int t1, bool is_bf16, cudaStream_t s)
{
    if (t1 <= t0) return 0;
    dim3 grid(ceil_div(t1 - t0, kFTok), ceil_div(a.d, kFThreads * 4));
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16)
            gate_bwd_fused_kernel<bf16, KK><<<grid, kFThreads, 0, s>>>(
                (const bf16*)dxe, (const bf16*)x, a.idx, a.slot, a.w, g, logits, wg, a.send_off, renorm,
                t0, t1, a.k, a.d, a.E, (bf16*)dx, partial, pbase);
        else
            gate_bwd_fused_kernel<float, KK><<<grid, kFThreads, 0, s>>>(
                (const float*)dxe, (const float*)x, a.idx, a.slot, a.w, g, logits, wg, a.send_off, renorm,
                t0, t1, a.k, a.d, a.E, (float*)dx, partial, pbase);
    });
    return 1;
}

int fused_partial_blocks(int t0, int t1) { return ceil_div(t1 - t0, kFTok); }

int launch_dwg_reduce(const float* partial, int nb, int d, int E, float* dwg, cudaStream_t s)
{
    dwg_reduce_kernel<<<ceil_div(d * E, 256), 256, 0, s>>>(partial, nb, d, E, dwg);
    return 1;
}

int launch_dwg(const void* x, const float* dlogit, int T, int d, int E, float* partial,
               float* dwg, bool is_bf16, cudaStream_t s)
{
    const int nb = ceil_div(T, kDwgTok);
    dim3 grid(nb, ceil_div(d, kDwgThreads * 4), ceil_div(E, kDwgE));
    if (is_bf16)
        dwg_partial_kernel<bf16><<<grid, kDwgThreads, 0, s>>>((const bf16*)x, dlogit, T, d, E, partial);
    else
        dwg_partial_kernel<float><<<grid, kDwgThreads, 0, s>>>((const float*)x, dlogit, T, d, E, partial);
    dwg_reduce_kernel<<<ceil_div(d * E, 256), 256, 0, s>>>(partial, nb, d, E, dwg);
    return 2;
}

int launch_zero_pads(void* buf, int row_elems, const int* grp_off, const int* grp_rows,
                     int n_groups, int elt_bytes, cudaStream_t s)
{
    if (n_groups <= 0) return 0;
    zero_pads_kernel<<<n_groups, 256, 0, s>>>((char*)buf, row_elems * elt_bytes, grp_off, grp_rows);
    return 1;
}

}  // namespace lancet
