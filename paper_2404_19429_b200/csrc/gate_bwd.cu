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

// dX row of a choice: local (dxe + row d), or -- push mode, the backward's second all-to-all
// fused into K6 -- row (row & mask) of the owner's dX buffer tab[row >> kPeerRowBits], read in
// place over peer memory
template <typename Elt>
__device__ __forceinline__ const Elt* dx_row(const Elt* dxe, const char* const* tab, int row, int d)
{
    if (tab)
        return reinterpret_cast<const Elt*>(tab[row >> kPeerRowBits]) + (size_t)(row & ((1 << kPeerRowBits) - 1)) * d;
    return dxe + (size_t)row * d;
}

template <typename Elt, int KK, bool SMEM_WG>
__global__ void __launch_bounds__(kWarps * 32)
k6_gather_kernel(const Elt* __restrict__ dxe, const int* __restrict__ prow,
                 const float* __restrict__ dlogit, const float* __restrict__ wgT, int t0, int t1,
                 int k, int d, int E, Elt* __restrict__ dx, const char* const* __restrict__ src_tab)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
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
        // every lane runs every pass (the dlogit broadcast below is a full-warp shuffle, so no
        // lane may leave early even when d / V < 32); loads and stores are guarded per vector
        for (int vb = 0; vb < nvec; vb += 32 * U) {
            const int v0 = vb + lane;
            uint4 raw[kK6T][U][KK];
#pragma unroll
            for (int q = 0; q < kK6T; ++q)
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int j = 0; j < KK; ++j)
                        if (rows[q][j] >= 0 && v0 + 32 * u < nvec)
                            raw[q][u][j] = ld_nc_v4(reinterpret_cast<const uint4*>(dx_row(dxe, src_tab, rows[q][j], d)) + v0 + 32 * u);
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
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
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
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
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
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= rows * cols) return;
    const int r = q / cols, c = q % cols;
    out[(size_t)c * rows + r] = in[q];
}


// ---------------------------------------------------------------------------------------
// Streaming variants for E <= 8, d % 256 == 0, d <= 2048 (the GPT-MoE shapes).  A block covers a
// contiguous token range; thread i owns dims [8i, 8i+8) of every token.  Row data reaches
// shared memory through a per-thread cp.async ring (each thread copies exactly the 16-byte
// pieces it later reads, so the ring needs no block barrier) -- the bytes in flight are
// bounded by shared memory rather than registers, which is what these HBM-latency-bound
// kernels need.  The packed rows / dlogit of the block's tokens are staged once up front.
constexpr int kStreamStages = 4;
constexpr int kDwgStreamMaxBlocks = 512;   // partial blocks of the streaming dWg paths
constexpr int kDwgStages = 6;    // K7: 2 blocks per SM, ~5 x 16 KB of x in flight each

template <typename Elt> struct Dims8 {                  // 8 elements = NV 16-byte vectors
    static constexpr int NV = 8 * (int)sizeof(Elt) / 16;
};

template <typename Elt>
__device__ __forceinline__ void unpack8(const uint4* v, float (&f)[8]) {
    if constexpr (sizeof(Elt) == 2) {
        unpack16<bf16>(v[0], f);
    } else {
        unpack16<float>(v[0], f);
        unpack16<float>(v[1], f + 4);
    }
}

__device__ __forceinline__ void cp_async16_s(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit_s() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_s() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Wg^T slice of a thread: wg2[e][q] = (Wg[i0+2q][e0+e], Wg[i0+2q+1][e0+e]) for e < EE.  With 8
// experts per lane and E % 4 == 0 the 8 rows are read as two 16-byte vectors each (the 64
// scalar loads of the general form were ~25 % of K6's stall samples: LSU throttle in the
// prologue of a one-wave grid)
template <int EE>
__device__ __forceinline__ void load_wgT(const float* __restrict__ wg, int E, int i0, int e0, float2 (&wg2)[EE][4])
{
    if (EE == 8 && E % 4 == 0 && e0 + 8 <= E) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4* ra = reinterpret_cast<const float4*>(wg + (size_t)(i0 + 2 * q) * E + e0);
            const float4* rb = reinterpret_cast<const float4*>(wg + (size_t)(i0 + 2 * q + 1) * E + e0);
            const float4 a0 = __ldg(ra), a1 = __ldg(ra + 1), b0 = __ldg(rb), b1 = __ldg(rb + 1);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int e = 0; e < EE; ++e) wg2[e][q] = make_float2(av[e & 7], bv[e & 7]);
        }
    } else {
#pragma unroll
        for (int e = 0; e < EE; ++e)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                wg2[e][q] = e0 + e < E ? make_float2(__ldg(wg + (size_t)(i0 + 2 * q) * E + e0 + e),
                                                     __ldg(wg + (size_t)(i0 + 2 * q + 1) * E + e0 + e))
                                       : make_float2(0.f, 0.f);
    }
}

template <typename Elt, int KK>
struct K6Geom {
    static constexpr int NV = Dims8<Elt>::NV;
    static constexpr int U = (8 / (KK * NV)) > 0 ? 8 / (KK * NV) : 1;   // tokens per ring slot
    static constexpr int SLOT = U * KK * NV;                              // 16-byte pieces per thread
};

// K6: dx_t = sum_j dX[prow_tj] + sum_e dlogit_te Wg[:, e]; Wg^T slice of the thread in registers
// EG > 1 (E = 8 EG, E <= 64): EG adjacent lanes share a dim group, each holding the Wg^T
// slice of 8 experts; their gate-term partials meet in an xor-shuffle tree; only the group's
// first lane copies row pieces into the ring (the others read them after __syncwarp).  A block
// covers 256 / EG dim groups (grid.y splits d).
template <typename Elt, int KK, int EE, int NTC, int EG = 1>
__global__ void __launch_bounds__(256)
k6_stream_kernel(const Elt* __restrict__ dxe, const int* __restrict__ prow,
                 const float* __restrict__ dlogit, const float* __restrict__ wg, int t0, int t1,
                 int k, int d, int E, int tpb, Elt* __restrict__ dx, const char* const* __restrict__ src_tab)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    using G = K6Geom<Elt, KK>;
    constexpr int NV = G::NV, U = G::U, S = kStreamStages;
    constexpr int ET = EG == 1 ? EE : 8 * EG;              // experts staged per token
    extern __shared__ __align__(16) uint4 ring[];          // [S][SLOT][NT / EG]
    const int NT = NTC > 0 ? NTC : (int)blockDim.x;
    const int NTD = NT / EG, dg = threadIdx.x / EG, eg = threadIdx.x % EG, tid = threadIdx.x;
    const bool copier = eg == 0;
    int* srow = reinterpret_cast<int*>(ring + (size_t)S * G::SLOT * NTD);  // [tpb][KK]
    // [tpb][ET], 16-byte aligned (float2 reads): tpb * KK ints rounded up to 4
    float* sdl = reinterpret_cast<float*>(srow + round_up(tpb * KK, 4));
    const int tb0 = t0 + blockIdx.x * tpb;
    const int tb1 = min(t1, tb0 + tpb);
    if (tb0 >= tb1) return;
    const int nt = tb1 - tb0;
    for (int q = tid; q < nt * KK; q += NT) {
        const int r = q / KK, j = q % KK;
        srow[q] = j < k ? prow[(size_t)(tb0 + r) * k + j] : -1;
    }
    for (int q = tid; q < nt * ET; q += NT) {
        const int r = q / ET, e = q % ET;
        sdl[q] = e < E ? dlogit[(size_t)(tb0 + r) * E + e] : 0.f;
    }
    const int i0 = (blockIdx.y * NTD + dg) * 8;
    const int e0 = eg * 8;                                  // this lane's experts (EG > 1)
    // this thread's Wg^T slice, read straight from Wg [d][E] (rows i0..i0+7)
    float2 wg2[EE][4];
    load_wgT<EE>(wg, E, i0, e0, wg2);
    __syncthreads();
    const int ng = ceil_div(nt, U);
    auto issue = [&](int g) {
        if (!copier) return;
        uint4* slot = ring + (size_t)(g % S) * G::SLOT * NTD;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = g * U + u;
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                const int row = r < nt ? srow[r * KK + j] : -1;
                if (row >= 0) {
                    const uint4* src = reinterpret_cast<const uint4*>(dx_row(dxe, src_tab, row, d) + i0);
#pragma unroll
                    for (int v = 0; v < NV; ++v) cp_async16_s(slot + ((u * KK + j) * NV + v) * NTD + dg, src + v);
                }
            }
        }
    };
#pragma unroll
    for (int g = 0; g < S - 1; ++g) {
        if (g < ng) issue(g);
        cp_async_commit_s();
    }
    for (int g = 0; g < ng; ++g) {
        if (g + S - 1 < ng) issue(g + S - 1);
        cp_async_commit_s();
        cp_async_wait_s<S - 1>();
        if constexpr (EG > 1) __syncwarp();                 // the group's copier has landed the slot
        const uint4* slot = ring + (size_t)(g % S) * G::SLOT * NTD;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = g * U + u;
            if (r >= nt) break;
            float acc[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = 0.f;
            int rw[KK];
#pragma unroll
            for (int j = 0; j < KK; ++j) rw[j] = srow[r * KK + j];
            float dlv[EE];
#pragma unroll
            for (int e = 0; e < EE; e += 2) {
                const float2 v = *reinterpret_cast<const float2*>(sdl + r * ET + e0 + e);
                dlv[e] = v.x; dlv[e + 1] = v.y;
            }
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                if (rw[j] >= 0) {
                    uint4 raw[NV];
#pragma unroll
                    for (int v = 0; v < NV; ++v) raw[v] = slot[((u * KK + j) * NV + v) * NTD + dg];
                    float f[8];
                    unpack8<Elt>(raw, f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] += f[i];
                }
            }
            float2 a2[4];
            if constexpr (EG == 1) {            // rows sum, then the gate term in e order
                a2[0] = make_float2(acc[0], acc[1]); a2[1] = make_float2(acc[2], acc[3]);
                a2[2] = make_float2(acc[4], acc[5]); a2[3] = make_float2(acc[6], acc[7]);
            } else {                            // this lane's 8-expert partial of the gate term
#pragma unroll
                for (int p = 0; p < 4; ++p) a2[p] = make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int e = 0; e < EE; ++e) {
                const float2 dl2 = make_float2(dlv[e], dlv[e]);
#pragma unroll
                for (int p = 0; p < 4; ++p) a2[p] = __ffma2_rn(dl2, wg2[e][p], a2[p]);
            }
            if constexpr (EG > 1) {             // partials of the EG lanes: fixed xor tree
#pragma unroll
                for (int m = 1; m < EG; m <<= 1)
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        a2[p].x += __shfl_xor_sync(0xffffffffu, a2[p].x, m);
                        a2[p].y += __shfl_xor_sync(0xffffffffu, a2[p].y, m);
                    }
#pragma unroll
                for (int p = 0; p < 4; ++p) a2[p] = make_float2(acc[2 * p] + a2[p].x, acc[2 * p + 1] + a2[p].y);
            }
            const float o[8] = {a2[0].x, a2[0].y, a2[1].x, a2[1].y, a2[2].x, a2[2].y, a2[3].x, a2[3].y};
            Elt* dst = dx + (size_t)(tb0 + r) * d + i0;
            if (!copier) continue;
            if constexpr (sizeof(Elt) == 2) {
                st_v4(dst, pack16<bf16>(o));
            } else {
                st_v4(dst, pack16<float>(o));
                st_v4(dst + 4, pack16<float>(o + 4));
            }
        }
        if constexpr (EG > 1) __syncwarp();                 // slot read by the group before refill
    }
    cp_async_wait_s<0>();
}

// K7 partials: block b sums x_t (x) dlogit_t over its contiguous token range -> partial[b][E][d]
// (EG > 1: E = 8 EG; EG adjacent lanes share a dim group, one group of 8 experts each; only
// the group's first lane copies the x pieces.  grid.y splits d.)
template <typename Elt, int EE, int NTC, int EG = 1>
__global__ void __launch_bounds__(256)
dwg_stream_kernel(const Elt* __restrict__ x, const float* __restrict__ dlogit, int T, int d, int E,
                  int tpb, float* __restrict__ partial)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    constexpr int NV = Dims8<Elt>::NV, U = 8 / NV, S = kDwgStages;
    constexpr int ET = EG == 1 ? EE : 8 * EG;              // experts staged per token
    extern __shared__ __align__(16) uint4 ring[];          // [S][U*NV][NT / EG]
    const int NT = NTC > 0 ? NTC : (int)blockDim.x, tid = threadIdx.x;
    const int NTD = NT / EG, dg = tid / EG, eg = tid % EG;
    const bool copier = eg == 0;
    float* sdl = reinterpret_cast<float*>(ring + (size_t)S * U * NV * NTD);  // [tpb][ET]
    const int tb0 = blockIdx.x * tpb;
    const int nt = max(0, min(T, tb0 + tpb) - tb0);
    const int i0 = (blockIdx.y * NTD + dg) * 8, e0 = eg * 8;
    const int ng = ceil_div(nt, U);
    auto issue = [&](int g) {
        if (!copier) return;
        uint4* slot = ring + (size_t)(g % S) * U * NV * NTD;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = g * U + u;
            if (r < nt) {
                const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)(tb0 + r) * d + i0);
#pragma unroll
                for (int v = 0; v < NV; ++v) cp_async16_s(slot + (u * NV + v) * NTD + dg, src + v);
            }
        }
    };
    // the x ring fills while dlogit is staged (one round trip of latency instead of two in a
    // one-wave grid)
#pragma unroll
    for (int g = 0; g < S - 1; ++g) {
        if (g < ng) issue(g);
        cp_async_commit_s();
    }
    for (int q = tid; q < nt * ET; q += NT) {
        const int r = q / ET, e = q % ET;
        sdl[q] = e < E ? dlogit[(size_t)(tb0 + r) * E + e] : 0.f;
    }
    float2 acc[8][EE / 2];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int p = 0; p < EE / 2; ++p) acc[a][p] = make_float2(0.f, 0.f);
    __syncthreads();
    for (int g = 0; g < ng; ++g) {
        if (g + S - 1 < ng) issue(g + S - 1);
        cp_async_commit_s();
        cp_async_wait_s<S - 1>();
        if constexpr (EG > 1) __syncwarp();                 // the group's copier has landed the slot
        const uint4* slot = ring + (size_t)(g % S) * U * NV * NTD;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = g * U + u;
            if (r >= nt) break;
            uint4 raw[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) raw[v] = slot[(u * NV + v) * NTD + dg];
            float xf[8];
            unpack8<Elt>(raw, xf);
            float2 dl[EE / 2];
#pragma unroll
            for (int p = 0; p < EE / 2; ++p) dl[p] = *reinterpret_cast<const float2*>(sdl + r * ET + e0 + 2 * p);
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int p = 0; p < EE / 2; ++p) acc[a][p] = __ffma2_rn(make_float2(xf[a], xf[a]), dl[p], acc[a][p]);
        }
        if constexpr (EG > 1) __syncwarp();                 // slot read by the group before refill
    }
    cp_async_wait_s<0>();
    // partial[b][e][i]: for each expert the block's threads store consecutive 32-byte runs
    float* out = partial + (size_t)blockIdx.x * E * d + (size_t)e0 * d + i0;
#pragma unroll
    for (int p = 0; p < EE / 2; ++p) {
        if (e0 + 2 * p < E) {
            float v[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) v[a] = acc[a][p].x;
            st_v4(out + (size_t)(2 * p) * d, pack16<float>(v));
            st_v4(out + (size_t)(2 * p) * d + 4, pack16<float>(v + 4));
        }
        if (e0 + 2 * p + 1 < E) {
            float v[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) v[a] = acc[a][p].y;
            st_v4(out + (size_t)(2 * p + 1) * d, pack16<float>(v));
            st_v4(out + (size_t)(2 * p + 1) * d + 4, pack16<float>(v + 4));
        }
    }
}


// K6 + K7 fused (world 1, one pass over all tokens): per token, dx_t from the k packed dX rows
// and the gate term (Wg^T slice in registers), and dWg partials x_t (x) dlogit_t (dWg slice in
// registers); dX rows and the x row stream through the per-thread cp.async ring together.
constexpr int kFusedStages = 6;

template <typename Elt, int KK>
struct FusedGeom {
    static constexpr int NV = Dims8<Elt>::NV;
    static constexpr int U = (8 / ((KK + 1) * NV)) > 0 ? 8 / ((KK + 1) * NV) : 1;   // tokens per slot
    static constexpr int SLOT = U * (KK + 1) * NV;                                    // 16-byte pieces
};

template <typename Elt, int KK, int EE, int NTC>
__global__ void __launch_bounds__(256)
gate_bwd_fused_kernel(const Elt* __restrict__ dxe, const int* __restrict__ prow,
                      const float* __restrict__ dlogit, const float* __restrict__ wg,
                      const Elt* __restrict__ x, int T, int k, int d, int E, int tpb,
                      Elt* __restrict__ dx, float* __restrict__ partial)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    using G = FusedGeom<Elt, KK>;
    constexpr int NV = G::NV, U = G::U, S = kFusedStages, P = (KK + 1) * NV;   // P: pieces per token
    extern __shared__ __align__(16) uint4 ring[];          // [S][SLOT][NT]
    const int NT = NTC > 0 ? NTC : (int)blockDim.x, tid = threadIdx.x;
    int* srow = reinterpret_cast<int*>(ring + (size_t)S * G::SLOT * NT);   // [tpb][KK]
    float* sdl = reinterpret_cast<float*>(srow + round_up(tpb * KK, 4));    // [tpb][EE], 16 B aligned
    const int tb0 = blockIdx.x * tpb;
    const int nt = max(0, min(T, tb0 + tpb) - tb0);
    for (int q = tid; q < nt * KK; q += NT) {
        const int r = q / KK, j = q % KK;
        srow[q] = j < k ? prow[(size_t)(tb0 + r) * k + j] : -1;
    }
    for (int q = tid; q < nt * EE; q += NT) {
        const int r = q / EE, e = q % EE;
        sdl[q] = e < E ? dlogit[(size_t)(tb0 + r) * E + e] : 0.f;
    }
    const int i0 = tid * 8;
    // this thread's Wg^T slice, read straight from Wg [d][E] (rows i0..i0+7)
    float2 wg2[EE][4];
    load_wgT<EE>(wg, E, i0, 0, wg2);
    float2 acc[8][EE / 2];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int p = 0; p < EE / 2; ++p) acc[a][p] = make_float2(0.f, 0.f);
    __syncthreads();
    const int ng = ceil_div(nt, U);
    auto issue = [&](int g) {
        uint4* slot = ring + (size_t)(g % S) * G::SLOT * NT;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = g * U + u;
            if (r < nt) {
#pragma unroll
                for (int j = 0; j < KK; ++j) {
                    const int row = srow[r * KK + j];
                    if (row >= 0) {
                        const uint4* src = reinterpret_cast<const uint4*>(dxe + (size_t)row * d + i0);
#pragma unroll
                        for (int v = 0; v < NV; ++v) cp_async16_s(slot + ((u * P) + j * NV + v) * NT + tid, src + v);
                    }
                }
                const uint4* xs = reinterpret_cast<const uint4*>(x + (size_t)(tb0 + r) * d + i0);
#pragma unroll
                for (int v = 0; v < NV; ++v) cp_async16_s(slot + ((u * P) + KK * NV + v) * NT + tid, xs + v);
            }
        }
    };
#pragma unroll
    for (int g = 0; g < S - 1; ++g) {
        if (g < ng) issue(g);
        cp_async_commit_s();
    }
    for (int g = 0; g < ng; ++g) {
        if (g + S - 1 < ng) issue(g + S - 1);
        cp_async_commit_s();
        cp_async_wait_s<S - 1>();
        const uint4* slot = ring + (size_t)(g % S) * G::SLOT * NT;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = g * U + u;
            if (r >= nt) break;
            float dlv[EE];
#pragma unroll
            for (int e = 0; e < EE; e += 2) {
                const float2 v = *reinterpret_cast<const float2*>(sdl + r * EE + e);
                dlv[e] = v.x; dlv[e + 1] = v.y;
            }
            // ---- K6: dx_t = sum_j dX[row_tj] (j order) + sum_e dlogit_te Wg[:, e] ----
            float s8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) s8[i] = 0.f;
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                if (srow[r * KK + j] >= 0) {
                    uint4 raw[NV];
#pragma unroll
                    for (int v = 0; v < NV; ++v) raw[v] = slot[((u * P) + j * NV + v) * NT + tid];
                    float f[8];
                    unpack8<Elt>(raw, f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) s8[i] += f[i];
                }
            }
            float2 a2[4] = {make_float2(s8[0], s8[1]), make_float2(s8[2], s8[3]),
                            make_float2(s8[4], s8[5]), make_float2(s8[6], s8[7])};
#pragma unroll
            for (int e = 0; e < EE; ++e) {
                const float2 dl2 = make_float2(dlv[e], dlv[e]);
#pragma unroll
                for (int q = 0; q < 4; ++q) a2[q] = __ffma2_rn(dl2, wg2[e][q], a2[q]);
            }
            const float o[8] = {a2[0].x, a2[0].y, a2[1].x, a2[1].y, a2[2].x, a2[2].y, a2[3].x, a2[3].y};
            Elt* dst = dx + (size_t)(tb0 + r) * d + i0;
            if constexpr (sizeof(Elt) == 2) {
                st_v4(dst, pack16<bf16>(o));
            } else {
                st_v4(dst, pack16<float>(o));
                st_v4(dst + 4, pack16<float>(o + 4));
            }
            // ---- K7: dWg[i][e] += x_ti dlogit_te ----
            uint4 xraw[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) xraw[v] = slot[((u * P) + KK * NV + v) * NT + tid];
            float xf[8];
            unpack8<Elt>(xraw, xf);
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int q = 0; q < EE / 2; ++q)
                    acc[a][q] = __ffma2_rn(make_float2(xf[a], xf[a]), make_float2(dlv[2 * q], dlv[2 * q + 1]), acc[a][q]);
        }
    }
    cp_async_wait_s<0>();
    float* out = partial + (size_t)blockIdx.x * E * d + i0;     // partial[b][e][i]
#pragma unroll
    for (int q = 0; q < EE / 2; ++q) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = 2 * q + h;
            if (e < E) {
                float v[8];
#pragma unroll
                for (int a = 0; a < 8; ++a) v[a] = h ? acc[a][q].y : acc[a][q].x;
                st_v4(out + (size_t)e * d, pack16<float>(v));
                st_v4(out + (size_t)e * d + 4, pack16<float>(v + 4));
            }
        }
    }
}

// Deterministic reduction of nb partials: block = 32 outputs (8 threads x float4) x 32 part
// streams; stream s sums partials s, s+32, ... in order, the 32 stream sums are added in order.
__global__ void __launch_bounds__(256)
dwg_reduce4_kernel(const float* __restrict__ partial, int nb, int n_out, int d_model, int E,
                   float* __restrict__ dwg)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    __shared__ float4 red[32][8];
    const int q4 = threadIdx.x & 7, st = threadIdx.x >> 3;
    const int o = blockIdx.x * 32 + q4 * 4;                 // n_out % 4 == 0
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    if (o < n_out) {
        // all of the stream's loads in flight at once (nb <= 32 * kRedMax), summed in b order
        constexpr int kRedMax = kDwgStreamMaxBlocks / 32;
        float4 v[kRedMax];
#pragma unroll
        for (int u = 0; u < kRedMax; ++u) {
            const int b = st + 32 * u;
            v[u] = b < nb ? __ldg(reinterpret_cast<const float4*>(partial + (size_t)b * n_out + o))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kRedMax; ++u) {
            s.x += v[u].x; s.y += v[u].y; s.z += v[u].z; s.w += v[u].w;
        }
    }
    red[st][q4] = s;
    __syncthreads();
    if (st == 0 && o < n_out) {
        float4 r = red[0][q4];
        for (int i = 1; i < 32; ++i) {
            const float4 v = red[i][q4];
            r.x += v.x; r.y += v.y; r.z += v.z; r.w += v.w;
        }
        // o indexes the [E][d] partial layout; dWg is [d][E]
        const int e = o / d_model, i = o % d_model;
        dwg[(size_t)i * E + e] = r.x;
        dwg[(size_t)(i + 1) * E + e] = r.y;
        dwg[(size_t)(i + 2) * E + e] = r.z;
        dwg[(size_t)(i + 3) * E + e] = r.w;
    }
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
    launch_k(transpose_f32_kernel, ceil_div(d * E, 256), 256, 0, s, wg, d, E, wgT);
    return 1;
}



template <typename Elt, int KK, bool SM>
static void launch_k6(const DispatchArgs& a, const void* dxe, const int* prow, const float* dlogit,
                      const float* wgT, void* dx, int t0, int t1, int num_sms, cudaStream_t s,
                      const char* const* src_tab)
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
    launch_k(k6_gather_kernel<Elt, KK, SM>, grid, kWarps * 32, smem, s, (const Elt*)dxe, prow, dlogit, wgT, t0, t1,
                                                                  a.k, a.d, a.E, (Elt*)dx, src_tab);
}

static bool stream_ok(int d, int E) { return E <= 8 && d % 256 == 0 && d <= 2048; }
// E = 8 EG, EG in {2, 4, 8}: the wide streaming K6 / K7
static bool wide_ok(int d, int E) { return (E == 16 || E == 32 || E == 64) && d % 256 == 0 && d <= 2048; }
bool gate_bwd_needs_wgT(int d, int E) { return !stream_ok(d, E) && !(wide_ok(d, E) && E >= 32); }
// Blocks for a per-block token range whose staged rows cost per_tok bytes of shared memory
// beside a fixed ring: at least `want` blocks, more if the range would not fit (large T).
static int blocks_for_smem(int ntok, int want, size_t ring, size_t per_tok)
{
    const size_t budget = 200 * 1024 - 16;     // - 16: the 16-byte alignment of the staged dlogit
    const int max_tpb = std::max(1, (int)((budget - std::min(ring, budget - per_tok)) / per_tok));
    return std::max(want, ceil_div(ntok, max_tpb));
}

// dim groups per block for EG lanes per group (<= 256 threads, dividing d / 8)
static int wide_ntd(int d, int EG)
{
    int ntd = 256 / EG;
    while ((d / 8) % ntd) ntd /= 2;
    return ntd;
}
static int ee_of(int E) { return E <= 2 ? 2 : E <= 4 ? 4 : 8; }

template <typename Elt, int KK, int EE>
static void launch_k6_stream(const DispatchArgs& a, const void* dxe, const int* prow, const float* dlogit,
                             const float* wg, void* dx, int t0, int t1, int num_sms, cudaStream_t s,
                             const char* const* src_tab)
{
    using G = K6Geom<Elt, KK>;
    const int NT = a.d / 8;
    // ~3 blocks per SM of 128 threads; a block's ring is kStreamStages slots of U tokens
    const int per_sm = std::max(1, 384 / NT);
    const int nb = blocks_for_smem(t1 - t0, std::max(1, std::min(ceil_div(t1 - t0, G::U), per_sm * num_sms)),
                                   (size_t)kStreamStages * G::SLOT * NT * 16, (size_t)(KK + EE) * 4);
    const int tpb = ceil_div(t1 - t0, nb);
    const size_t smem = (size_t)kStreamStages * G::SLOT * NT * 16 + ((size_t)round_up(tpb * KK, 4) + (size_t)tpb * EE) * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k6_stream_kernel<Elt, KK, EE, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k6_stream_kernel<Elt, KK, EE, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    if (NT == 128)      // d = 1024: compile-time ring strides
        launch_k(k6_stream_kernel<Elt, KK, EE, 128>, ceil_div(t1 - t0, tpb), NT, smem, s, 
            (const Elt*)dxe, prow, dlogit, wg, t0, t1, a.k, a.d, a.E, tpb, (Elt*)dx, src_tab);
    else
        launch_k(k6_stream_kernel<Elt, KK, EE, 0>, ceil_div(t1 - t0, tpb), NT, smem, s, 
            (const Elt*)dxe, prow, dlogit, wg, t0, t1, a.k, a.d, a.E, tpb, (Elt*)dx, src_tab);
}

template <typename Elt, int KK, int EG>
static void launch_k6_wide(const DispatchArgs& a, const void* dxe, const int* prow, const float* dlogit,
                           const float* wg, void* dx, int t0, int t1, int num_sms, cudaStream_t s,
                           const char* const* src_tab)
{
    using G = K6Geom<Elt, KK>;
    const int NTD = wide_ntd(a.d, EG), DS = a.d / 8 / NTD, NT = NTD * EG;
    const int nb = blocks_for_smem(t1 - t0, std::max(1, std::min(ceil_div(t1 - t0, G::U), std::max(1, 3 * num_sms / DS))),
                                   (size_t)kStreamStages * G::SLOT * NTD * 16, (size_t)(KK + 8 * EG) * 4);
    const int tpb = ceil_div(t1 - t0, nb);
    const size_t smem = (size_t)kStreamStages * G::SLOT * NTD * 16 + ((size_t)round_up(tpb * KK, 4) + (size_t)tpb * 8 * EG) * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k6_stream_kernel<Elt, KK, 8, 0, EG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    launch_k(k6_stream_kernel<Elt, KK, 8, 0, EG>, dim3(ceil_div(t1 - t0, tpb), DS), NT, smem, s,
             (const Elt*)dxe, prow, dlogit, wg, t0, t1, a.k, a.d, a.E, tpb, (Elt*)dx, src_tab);
}

int launch_unpermute_gate_bwd(const DispatchArgs& a, const void* dxe, const int* prow,
                              const float* dlogit, const float* wg, const float* wgT, void* dx, int t0, int t1,
                              int num_sms, bool is_bf16, cudaStream_t s, const char* const* src_tab)
{
    if (t1 <= t0) return 0;
    // wide K6 only from E = 32 (at E = 16 the shared-memory Wg^T kernel measured faster)
    if (wide_ok(a.d, a.E) && a.E >= 32 && a.k <= 4) {
#define K6W(Elt, KK)                                                                                              \
    do {                                                                                                          \
        if (a.E == 16) launch_k6_wide<Elt, KK, 2>(a, dxe, prow, dlogit, wg, dx, t0, t1, num_sms, s, src_tab);             \
        else if (a.E == 32) launch_k6_wide<Elt, KK, 4>(a, dxe, prow, dlogit, wg, dx, t0, t1, num_sms, s, src_tab);        \
        else launch_k6_wide<Elt, KK, 8>(a, dxe, prow, dlogit, wg, dx, t0, t1, num_sms, s, src_tab);                       \
    } while (0)
        if (is_bf16) {
            if (a.k == 1) K6W(bf16, 1); else if (a.k == 2) K6W(bf16, 2); else K6W(bf16, 4);
        } else {
            if (a.k == 1) K6W(float, 1); else if (a.k == 2) K6W(float, 2); else K6W(float, 4);
        }
#undef K6W
        return 1;
    }
    if (stream_ok(a.d, a.E) && a.k <= 4) {
        const int ee = ee_of(a.E);
#define K6S(Elt, KK)                                                                                              \
    do {                                                                                                          \
        if (ee == 2) launch_k6_stream<Elt, KK, 2>(a, dxe, prow, dlogit, wg, dx, t0, t1, num_sms, s, src_tab);            \
        else if (ee == 4) launch_k6_stream<Elt, KK, 4>(a, dxe, prow, dlogit, wg, dx, t0, t1, num_sms, s, src_tab);       \
        else launch_k6_stream<Elt, KK, 8>(a, dxe, prow, dlogit, wg, dx, t0, t1, num_sms, s, src_tab);                    \
    } while (0)
        if (is_bf16) {
            if (a.k == 1) K6S(bf16, 1); else if (a.k == 2) K6S(bf16, 2); else K6S(bf16, 4);
        } else {
            if (a.k == 1) K6S(float, 1); else if (a.k == 2) K6S(float, 2); else K6S(float, 4);
        }
#undef K6S
        return 1;
    }
    const bool sm = (size_t)a.d * a.E * 4 <= kSmemWgMax;
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16) {
            if (sm) launch_k6<bf16, KK, true>(a, dxe, prow, dlogit, wgT, dx, t0, t1, num_sms, s, src_tab);
            else launch_k6<bf16, KK, false>(a, dxe, prow, dlogit, wgT, dx, t0, t1, num_sms, s, src_tab);
        } else {
            if (sm) launch_k6<float, KK, true>(a, dxe, prow, dlogit, wgT, dx, t0, t1, num_sms, s, src_tab);
            else launch_k6<float, KK, false>(a, dxe, prow, dlogit, wgT, dx, t0, t1, num_sms, s, src_tab);
        }
    });
    return 1;
}

size_t dwg_partial_floats(int T, int d, int E)
{
    size_t n = (size_t)ceil_div(T, kDwgTok) * d * E;
    if (stream_ok(d, E) || wide_ok(d, E)) n = std::max(n, (size_t)kDwgStreamMaxBlocks * d * E);
    return n;
}

template <typename Elt, int EE>
static void launch_dwg_stream(const Elt* x, const float* dlogit, int T, int d, int E, float* partial,
                              float* dwg, int num_sms, cudaStream_t s)
{
    constexpr int NV = Dims8<Elt>::NV, U = 8 / NV;
    const int NT = d / 8;
    const int per_sm = std::max(1, 256 / NT);       // fewer, fatter blocks: fewer partials
    const int nb = std::min(kDwgStreamMaxBlocks,
                            blocks_for_smem(T, std::max(1, std::min({ceil_div(T, 2 * U), per_sm * num_sms,
                                                                     kDwgStreamMaxBlocks})),
                                            (size_t)kDwgStages * U * NV * NT * 16, (size_t)EE * 4));
    const int tpb = ceil_div(T, nb);
    const int grid = ceil_div(T, tpb);
    const size_t smem = (size_t)kDwgStages * U * NV * NT * 16 + (size_t)tpb * EE * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(dwg_stream_kernel<Elt, EE, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(dwg_stream_kernel<Elt, EE, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    if (NT == 128) launch_k(dwg_stream_kernel<Elt, EE, 128>, grid, NT, smem, s, x, dlogit, T, d, E, tpb, partial);
    else launch_k(dwg_stream_kernel<Elt, EE, 0>, grid, NT, smem, s, x, dlogit, T, d, E, tpb, partial);
    launch_k(dwg_reduce4_kernel, ceil_div(d * E, 32), 256, 0, s, partial, grid, d * E, d, E, dwg);
}

template <typename Elt, int EG>
static void launch_dwg_wide(const Elt* x, const float* dlogit, int T, int d, int E, float* partial,
                            float* dwg, int num_sms, cudaStream_t s)
{
    constexpr int NV = Dims8<Elt>::NV, U = 8 / NV;
    const int NTD = wide_ntd(d, EG), DS = d / 8 / NTD, NT = NTD * EG;
    // the per-block dlogit rows must fit beside the ring (T = 64k at E = 64: 94 blocks, not 74)
    const int nb = std::min(kDwgStreamMaxBlocks,
                            blocks_for_smem(T, std::max(1, std::min({ceil_div(T, 2 * U), std::max(1, 2 * num_sms / DS),
                                                                     kDwgStreamMaxBlocks})),
                                            (size_t)kDwgStages * U * NV * NTD * 16, (size_t)8 * EG * 4));
    const int tpb = ceil_div(T, nb);
    const int grid = ceil_div(T, tpb);
    const size_t smem = (size_t)kDwgStages * U * NV * NTD * 16 + (size_t)tpb * 8 * EG * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(dwg_stream_kernel<Elt, 8, 0, EG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    launch_k(dwg_stream_kernel<Elt, 8, 0, EG>, dim3(grid, DS), NT, smem, s, x, dlogit, T, d, E, tpb, partial);
    launch_k(dwg_reduce4_kernel, ceil_div(d * E, 32), 256, 0, s, partial, grid, d * E, d, E, dwg);
}

int launch_dwg(const void* x, const float* dlogit, int T, int d, int E, float* partial,
               float* dwg, bool is_bf16, int num_sms, cudaStream_t s)
{
    if (wide_ok(d, E)) {
#define DWW(Elt)                                                                                                  \
    do {                                                                                                          \
        if (E == 16) launch_dwg_wide<Elt, 2>((const Elt*)x, dlogit, T, d, E, partial, dwg, num_sms, s);          \
        else if (E == 32) launch_dwg_wide<Elt, 4>((const Elt*)x, dlogit, T, d, E, partial, dwg, num_sms, s);     \
        else launch_dwg_wide<Elt, 8>((const Elt*)x, dlogit, T, d, E, partial, dwg, num_sms, s);                  \
    } while (0)
        if (is_bf16) DWW(bf16); else DWW(float);
#undef DWW
        return 2;
    }
    if (stream_ok(d, E) && (d * E) % 4 == 0) {
        const int ee = ee_of(E);
#define DWS(Elt)                                                                                                  \
    do {                                                                                                          \
        if (ee == 2) launch_dwg_stream<Elt, 2>((const Elt*)x, dlogit, T, d, E, partial, dwg, num_sms, s);        \
        else if (ee == 4) launch_dwg_stream<Elt, 4>((const Elt*)x, dlogit, T, d, E, partial, dwg, num_sms, s);   \
        else launch_dwg_stream<Elt, 8>((const Elt*)x, dlogit, T, d, E, partial, dwg, num_sms, s);                \
    } while (0)
        if (is_bf16) DWS(bf16); else DWS(float);
#undef DWS
        return 2;
    }
    const int nb = ceil_div(T, kDwgTok);
    dim3 grid(nb, ceil_div(d, kDwgThreads * 4), ceil_div(E, kDwgE));
    if (is_bf16)
        launch_k(dwg_partial_kernel<bf16>, grid, kDwgThreads, 0, s, (const bf16*)x, dlogit, T, d, E, partial);
    else
        launch_k(dwg_partial_kernel<float>, grid, kDwgThreads, 0, s, (const float*)x, dlogit, T, d, E, partial);
    launch_k(dwg_reduce_kernel, ceil_div(d * E, 32), 256, 0, s, partial, nb, d * E, dwg);
    return 2;
}


template <typename Elt, int KK, int EE>
static void launch_fused(const DispatchArgs& a, const void* dxe, const int* prow, const float* dlogit,
                         const float* wg, const void* x, void* dx, float* partial, float* dwg,
                         int num_sms, cudaStream_t s)
{
    using G = FusedGeom<Elt, KK>;
    const int NT = a.d / 8;
    const int per_sm = std::max(1, 256 / NT);
    const int nb = std::min(kDwgStreamMaxBlocks,
                            blocks_for_smem(a.T, std::max(1, std::min({ceil_div(a.T, 4 * G::U), per_sm * num_sms,
                                                                       kDwgStreamMaxBlocks})),
                                            (size_t)kFusedStages * G::SLOT * NT * 16, (size_t)(KK + EE) * 4));
    const int tpb = ceil_div(a.T, nb);
    const int grid = ceil_div(a.T, tpb);
    const size_t smem = (size_t)kFusedStages * G::SLOT * NT * 16 + ((size_t)round_up(tpb * KK, 4) + (size_t)tpb * EE) * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gate_bwd_fused_kernel<Elt, KK, EE, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(gate_bwd_fused_kernel<Elt, KK, EE, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    if (NT == 128)
        launch_k(gate_bwd_fused_kernel<Elt, KK, EE, 128>, grid, NT, smem, s, 
            (const Elt*)dxe, prow, dlogit, wg, (const Elt*)x, a.T, a.k, a.d, a.E, tpb, (Elt*)dx, partial);
    else
        launch_k(gate_bwd_fused_kernel<Elt, KK, EE, 0>, grid, NT, smem, s, 
            (const Elt*)dxe, prow, dlogit, wg, (const Elt*)x, a.T, a.k, a.d, a.E, tpb, (Elt*)dx, partial);
    launch_k(dwg_reduce4_kernel, ceil_div(a.d * a.E, 32), 256, 0, s, partial, grid, a.d * a.E, a.d, a.E, dwg);
}

bool gate_bwd_fused_ok(int d, int E, int k) { return stream_ok(d, E) && k <= 4; }

int launch_gate_bwd_fused(const DispatchArgs& a, const void* dxe, const int* prow, const float* dlogit,
                          const float* wg, const void* x, void* dx, float* partial, float* dwg,
                          int num_sms, bool is_bf16, cudaStream_t s)
{
    if (!gate_bwd_fused_ok(a.d, a.E, a.k)) return -1;
    const int ee = ee_of(a.E);
#define FUS(Elt, KK)                                                                                                   \
    do {                                                                                                               \
        if (ee == 2) launch_fused<Elt, KK, 2>(a, dxe, prow, dlogit, wg, x, dx, partial, dwg, num_sms, s);            \
        else if (ee == 4) launch_fused<Elt, KK, 4>(a, dxe, prow, dlogit, wg, x, dx, partial, dwg, num_sms, s);       \
        else launch_fused<Elt, KK, 8>(a, dxe, prow, dlogit, wg, x, dx, partial, dwg, num_sms, s);                    \
    } while (0)
    if (is_bf16) {
        if (a.k == 1) FUS(bf16, 1); else if (a.k == 2) FUS(bf16, 2); else FUS(bf16, 4);
    } else {
        if (a.k == 1) FUS(float, 1); else if (a.k == 2) FUS(float, 2); else FUS(float, 4);
    }
#undef FUS
    return 2;
}

}  // namespace lancet
