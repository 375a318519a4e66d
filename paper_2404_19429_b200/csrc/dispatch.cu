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
// K5 combine backward:  g_tj = <dy_t, o_tj>, dcomb[off_e + slot] = w_tj dy_t; also dlogit
//               (softmax Jacobian, R3) and the packed source rows for K6/K7.
// (K6 dispatch backward + gate term and K7 dWg live in gate_bwd.cu.)
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
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
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

// K3 + C2 dispatch fused over peer memory (LANCET_FLAG_PEER_PUSH): each admitted row x[t] is
// written straight into the receive buffer of the rank that owns its expert (an IPC-mapped
// pointer; over NVLink on a multi-GPU node), at its final row base[e] + slot -- no send buffer,
// no copy-engine pass.  One launch per chunk (tokens [t0, t1), base = that chunk's table).
template <typename Elt, int KK>
__global__ void __launch_bounds__(256)
permute_push_kernel(const Elt* __restrict__ x, const int* __restrict__ idx, const int* __restrict__ slot,
                    int t0, int t1, int k, int d, int E_l, const int* __restrict__ base,
                    char* const* __restrict__ xe_ptrs)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    constexpr int V = Vec16<Elt>::N;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = t0 + blockIdx.x * kWarpsPerBlock + w;
    if (t >= t1) return;
    uint4* dst[KK];
    int myidx = -1, mys = -1;
    if (lane < k) {
        myidx = idx[(size_t)t * k + lane];
        mys = slot[(size_t)t * k + lane];
    }
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        const int e = __shfl_sync(0xffffffffu, myidx, j);
        const int sl = __shfl_sync(0xffffffffu, mys, j);
        dst[j] = nullptr;
        if (j < k && sl >= 0)
            dst[j] = reinterpret_cast<uint4*>(xe_ptrs[e / E_l] + (size_t)(base[e] + sl) * d * sizeof(Elt));
    }
    const int nvec = d / V;
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)t * d);
    constexpr int U = 4;
    for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
        uint4 val[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (v0 + 32 * u < nvec) val[u] = ld_nc_v4(src + v0 + 32 * u);
#pragma unroll
        for (int j = 0; j < KK; ++j)
            if (dst[j]) {
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (v0 + 32 * u < nvec) st_v4(dst[j] + v0 + 32 * u, val[u]);
            }
    }
}

template <typename Elt, int KK>
__global__ void __launch_bounds__(256)
combine_kernel(const Elt* __restrict__ comb, const int* __restrict__ idx,
               const int* __restrict__ slot, const float* __restrict__ wts,
               const int* __restrict__ send_off, int t0, int t1, int k, int d,
               Elt* __restrict__ y, const int* __restrict__ src_base, const char* const* __restrict__ src_tab,
               int E_l, const Elt* __restrict__ resid)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    constexpr int V = Vec16<Elt>::N;
    constexpr int U = 2;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = t0 + blockIdx.x * kWarpsPerBlock + w;
    if (t >= t1) return;
    int rows[KK], ids[KK];
    float wj[KK];
    load_choices<KK>(idx, slot, wts, send_off, t, k, lane, rows, wj, ids);
    // o row of choice j: the returned row in this rank's comb, or (fused combine exchange,
    // LANCET_FLAG_PEER_PUSH) the expert output row itself in the owner's buffer over peer memory
    const Elt* orow[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        orow[j] = nullptr;
        if (rows[j] >= 0)
            orow[j] = src_base ? reinterpret_cast<const Elt*>(src_tab[ids[j] / E_l] +
                                                               (size_t)(src_base[ids[j]] + rows[j] - send_off[ids[j]]) * d * sizeof(Elt))
                               : comb + (size_t)rows[j] * d;
    }
    const int nvec = d / V;
    uint4* dst = reinterpret_cast<uint4*>(y + (size_t)t * d);
    for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
        uint4 raw[U][KK];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < KK; ++j)
                if (rows[j] >= 0 && v0 + 32 * u < nvec)
                    raw[u][j] = ld_nc_v4(reinterpret_cast<const uint4*>(orow[j]) + v0 + 32 * u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (v0 + 32 * u >= nvec) break;
            float acc[V];
            if (resid) {   // the block's residual: y = h + sum_j w_j o_j (the chain starts at h)
                unpack16<Elt>(ld_nc_v4(reinterpret_cast<const uint4*>(resid + (size_t)t * d) + v0 + 32 * u), acc);
            } else {
#pragma unroll
                for (int q = 0; q < V; ++q) acc[q] = 0.f;
            }
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
                   float* __restrict__ g, Elt* __restrict__ dcomb, int tok_blocks,
                   const float* __restrict__ logits, int E, int renorm, float* __restrict__ dlogit,
                   int* __restrict__ prow, const int* __restrict__ push_base, char* const* __restrict__ push_dst,
                   int E_l, const char* const* __restrict__ src_tab)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
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
    // dO row of choice j: this rank's dcomb, or (push, LANCET_FLAG_PEER_PUSH) its final row in
    // the owning rank's receive buffer -- backward all-to-all #1 fused into this kernel
    Elt* drow[KK];
    const Elt* orow[KK];                               // o rows (fused combine: the owner's)
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        drow[j] = nullptr;
        orow[j] = nullptr;
        if (rows[j] >= 0)
            orow[j] = (push_base && src_tab)
                          ? reinterpret_cast<const Elt*>(src_tab[ids[j] / E_l] +
                                                         (size_t)(push_base[ids[j]] + rows[j] - send_off[ids[j]]) * d * sizeof(Elt))
                          : comb + (size_t)rows[j] * d;
        if (rows[j] >= 0) {
            if (push_base) {
                const int e = ids[j];
                drow[j] = reinterpret_cast<Elt*>(push_dst[e / E_l] +
                                                 (size_t)(push_base[e] + rows[j] - send_off[e]) * d * sizeof(Elt));
            } else {
                drow[j] = dcomb + (size_t)rows[j] * d;
            }
        }
    }
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
                        ro[u][j] = ld_nc_v4(reinterpret_cast<const uint4*>(orow[j]) + v0 + 32 * u);
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
                    st_v4(reinterpret_cast<uint4*>(drow[j]) + v0 + 32 * u, pack16<Elt>(sc));
                }
            }
        }
    }
    float gj[KK];
    float sg = 0.f;                                    // sum_j g_j w_j
    int myrow = -1;
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        gj[j] = 0.f;
        if (j < k) {
            const float s = warp_sum(part[j]);
            gj[j] = rows[j] >= 0 ? s : 0.f;
            if (lane == 0) g[(size_t)t * k + j] = gj[j];
            sg = fmaf(gj[j], wj[j], sg);
            // push mode: where K6 will read this choice's dX row -- (owner, row in its buffer)
            if (lane == j)
                myrow = (push_base && rows[j] >= 0)
                            ? (((ids[j] / E_l) << kPeerRowBits) | (push_base[ids[j]] + rows[j] - send_off[ids[j]]))
                            : rows[j];
        }
    }
    // inputs of the gate backward (K6/K7): packed source rows and dlogit from the softmax
    // Jacobian (R3): p_e (g~_e - sg), or renormalised at the selected experts
    if (lane < k) prow[(size_t)t * k + lane] = myrow;
    const float* lr = logits + (size_t)t * E;
    float m = -INFINITY;
    for (int e = lane; e < E; e += 32) m = fmaxf(m, lr[e]);
    m = warp_max(m);
    float se = 0.f;
    for (int e = lane; e < E; e += 32) se += expf(lr[e] - m);
    se = warp_sum(se);
    for (int e = lane; e < E; e += 32) {
        float gt = 0.f, wsel = 0.f;
        bool sel = false;
#pragma unroll
        for (int j = 0; j < KK; ++j)
            if (j < k && ids[j] == e) { gt = gj[j]; wsel = wj[j]; sel = true; }
        // renorm == 2: Random gate, no gate network (R18)
        dlogit[(size_t)t * E + e] = renorm == 2 ? 0.f
                                  : renorm ? (sel ? wsel * (gt - sg) : 0.f) : (expf(lr[e] - m) / se) * (gt - sg);
    }
}

__global__ void zero_pads_kernel(char* __restrict__ buf, int row_bytes,
                                 const int* __restrict__ grp_off, const int* __restrict__ grp_rows)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
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
            launch_k(permute_kernel<bf16, KK>, grid, 256, 0, s, (const bf16*)x, a.idx, a.slot, a.T, a.k, a.d,
                                                         a.send_off, a.send_rows, (bf16*)xs, tok_blocks);
        else
            launch_k(permute_kernel<float, KK>, grid, 256, 0, s, (const float*)x, a.idx, a.slot, a.T, a.k, a.d,
                                                          a.send_off, a.send_rows, (float*)xs, tok_blocks);
    });
    return 1;
}

int launch_permute_push(const DispatchArgs& a, const void* x, int t0, int t1, int E_l, const int* base,
                        char* const* xe_ptrs, bool is_bf16, cudaStream_t s)
{
    if (t1 <= t0) return 0;
    const int grid = ceil_div(t1 - t0, kWarpsPerBlock);
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16)
            launch_k(permute_push_kernel<bf16, KK>, grid, 256, 0, s, (const bf16*)x, a.idx, a.slot, t0, t1, a.k,
                     a.d, E_l, base, xe_ptrs);
        else
            launch_k(permute_push_kernel<float, KK>, grid, 256, 0, s, (const float*)x, a.idx, a.slot, t0, t1, a.k,
                     a.d, E_l, base, xe_ptrs);
    });
    return 1;
}

int launch_combine(const DispatchArgs& a, const void* comb, void* y, int t0, int t1, bool is_bf16,
                   cudaStream_t s, const int* src_base, const char* const* src_tab, int E_l, const void* resid)
{
    if (t1 <= t0) return 0;
    const int grid = ceil_div(t1 - t0, kWarpsPerBlock);
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16)
            launch_k(combine_kernel<bf16, KK>, grid, 256, 0, s, (const bf16*)comb, a.idx, a.slot, a.w, a.send_off,
                                                         t0, t1, a.k, a.d, (bf16*)y, src_base, src_tab, E_l,
                                                         (const bf16*)resid);
        else
            launch_k(combine_kernel<float, KK>, grid, 256, 0, s, (const float*)comb, a.idx, a.slot, a.w,
                                                          a.send_off, t0, t1, a.k, a.d, (float*)y, src_base, src_tab,
                                                          E_l, (const float*)resid);
    });
    return 1;
}

int launch_combine_bwd(const DispatchArgs& a, const void* dy, const void* comb, float* g,
                       void* dcomb, int t0, int t1, bool zero_pads, const float* logits, int renorm,
                       float* dlogit, int* prow, bool is_bf16, cudaStream_t s, const int* push_base,
                       char* const* push_dst, int E_l, const char* const* src_tab)
{
    const int tok_blocks = ceil_div(t1 - t0, kWarpsPerBlock);
    const int grid = tok_blocks + (zero_pads ? a.E : 0);
    if (grid == 0) return 0;
    LANCET_DISPATCH_K(a.k, {
        if (is_bf16)
            launch_k(combine_bwd_kernel<bf16, KK>, grid, 256, 0, s, (const bf16*)dy, (const bf16*)comb, a.idx,
                                                             a.slot, a.w, a.send_off, a.send_rows, t0, t1,
                                                             a.k, a.d, g, (bf16*)dcomb, tok_blocks, logits, a.E,
                                                             renorm, dlogit, prow, push_base, push_dst, E_l, src_tab);
        else
            launch_k(combine_bwd_kernel<float, KK>, grid, 256, 0, s, (const float*)dy, (const float*)comb, a.idx,
                                                              a.slot, a.w, a.send_off, a.send_rows, t0, t1,
                                                              a.k, a.d, g, (float*)dcomb, tok_blocks, logits, a.E,
                                                              renorm, dlogit, prow, push_base, push_dst, E_l, src_tab);
    });
    return 1;
}

int launch_zero_pads(void* buf, int row_elems, const int* grp_off, const int* grp_rows,
                     int n_groups, int elt_bytes, cudaStream_t s)
{
    if (n_groups <= 0) return 0;
    launch_k(zero_pads_kernel, n_groups, 256, 0, s, (char*)buf, row_elems * elt_bytes, grp_off, grp_rows);
    return 1;
}

}  // namespace lancet
