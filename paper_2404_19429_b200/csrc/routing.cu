// routing.cu -- K1 (gate + top-k + combine weights) and K2 (partition-invariant capacity
// slotting by a token-major prefix scan).
//
// K1: "assigning a gating score for each expert using a trainable linear layer, and choosing
//     k experts with highest scores".  logit[t][e] is the fp32 fma chain of
//     DESIGN.md R1 (increasing i, one rounding per step, no tensor cores) so routing is
//     bit-reproducible; top-k by (logit desc, e asc) (R2); w = softmax(logit)[idx] (R3).
// K2: capacity C per (rank, expert); a pair (t, j) routed to e takes
//     slot P_e(t) = #pairs routed to e by tokens before t (token-major, R7), admitted iff
//     P_e(t) < C.  Because P_e is a prefix over the WHOLE batch, chunk c's admissions are the
//     slots [S[e][c], S[e][c+1]) with S[e][c] = min(C, P_e(t_c)) -- exactly Lancet's
//     "gating operators that pass capacity information between partitions",
//     with the capacity state S computed for all chunks at once.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace lancet {

constexpr int kGateDT = 256;     // d-tile staged in shared memory (double-buffered cp.async)
constexpr int kGateMaxTB = 64;   // tokens per block
constexpr int kGateThreadCap = 128;

struct GateGeom {
    int ce;        // experts (R1 chains) per thread: 2 if E is even, else 1
    int tpt;       // threads per token = E / ce
    int TB;        // tokens per block
    int threads;   // TB * tpt
    int dt;        // dims per staged tile
    int row_bytes; // bytes per staged x row
    size_t buf_bytes, smem;
};

__host__ __device__ inline GateGeom gate_geom(int E, int elt_bytes)
{
    GateGeom g;
    g.ce = (E % 2 == 0) ? 2 : 1;   // 2 chains per thread: 4x the warps of 8, latency-bound kernel
    g.tpt = E / g.ce;
    g.TB = kGateThreadCap / g.tpt;
    if (g.TB > kGateMaxTB) g.TB = kGateMaxTB;
    if (g.TB < 1) g.TB = 1;
    g.threads = g.TB * g.tpt;
    // d-tile: 256 dims, fewer when the Wg tile (DT x E fp32) would exceed 16 KiB
    int dt = 4096 / E;
    dt = dt > kGateDT ? kGateDT : dt;
    dt = dt < 8 ? 8 : (dt & ~7);
    g.dt = dt;
    g.row_bytes = dt * elt_bytes + 16;                              // +16 B: fewer bank conflicts
    g.buf_bytes = (size_t)g.TB * g.row_bytes + (size_t)dt * E * 4;
    const size_t xs = 2 * g.buf_bytes;
    const size_t lg = sizeof(float) * (size_t)g.TB * E;
    g.smem = xs > lg ? xs : lg;
    return g;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename Elt>
__device__ __forceinline__ void gate_load_tile(const Elt* __restrict__ x, const float* __restrict__ wg,
                                               int T, int d, int E, int t0, const GateGeom& geo,
                                               int i0, uint8_t* buf)
{
    const int ilim = min(geo.dt, d - i0);
    const int cpr = ilim * (int)sizeof(Elt) / 16;                 // 16-byte chunks per x row
    for (int q = threadIdx.x; q < geo.TB * cpr; q += blockDim.x) {
        const int r = q / cpr, c = q % cpr, t = t0 + r;
        if (t < T)
            cp_async16(buf + (size_t)r * geo.row_bytes + c * 16,
                       reinterpret_cast<const uint8_t*>(x + (size_t)t * d + i0) + c * 16);
    }
    // Wg rows [i0, i0 + ilim) x E (contiguous in global memory)
    uint8_t* wb = buf + (size_t)geo.TB * geo.row_bytes;
    const int wchunks = ilim * E * 4 / 16;
    const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(wg + (size_t)i0 * E);
    for (int q = threadIdx.x; q < wchunks; q += blockDim.x) cp_async16(wb + q * 16, wsrc + q * 16);
}

// acc[c] = fma(xv, w[c], acc[c]) for the CE experts of this thread (one R1 step each)
template <int CE>
__device__ __forceinline__ void gate_fma_row(const float* w, float xv, float (&acc)[CE])
{
    if constexpr (CE % 4 == 0) {
#pragma unroll
        for (int h = 0; h < CE / 4; ++h) {
            const float4 w4 = *reinterpret_cast<const float4*>(w + 4 * h);
            acc[4 * h + 0] = __fmaf_rn(xv, w4.x, acc[4 * h + 0]);
            acc[4 * h + 1] = __fmaf_rn(xv, w4.y, acc[4 * h + 1]);
            acc[4 * h + 2] = __fmaf_rn(xv, w4.z, acc[4 * h + 2]);
            acc[4 * h + 3] = __fmaf_rn(xv, w4.w, acc[4 * h + 3]);
        }
    } else if constexpr (CE == 2) {
        const float2 w2 = *reinterpret_cast<const float2*>(w);
        acc[0] = __fmaf_rn(xv, w2.x, acc[0]);
        acc[1] = __fmaf_rn(xv, w2.y, acc[1]);
    } else {
        acc[0] = __fmaf_rn(xv, w[0], acc[0]);
    }
}

// K1.  Thread (token r, experts e0..e0+CE-1) runs CE independent R1 chains; tiles of x and of
// Wg stream through shared memory (cp.async, double-buffered).
template <typename Elt, int CE>
__global__ void __launch_bounds__(kGateThreadCap)
gate_topk_kernel(const Elt* __restrict__ x, const float* __restrict__ wg, int T, int d, int E,
                 int k, int renorm, float* __restrict__ logits, int* __restrict__ idx_out,
                 float* __restrict__ w_out, int* __restrict__ hist, int n_tiles)
{
    extern __shared__ __align__(16) uint8_t gsm[];
    __shared__ int sh_hist[2 * kMaxExperts];
    const GateGeom geo = gate_geom(E, sizeof(Elt));
    const int TB = geo.TB;
    uint8_t* buf0 = gsm;
    uint8_t* buf1 = gsm + geo.buf_bytes;
    const int tid = threadIdx.x;
    const int r = tid / geo.tpt;                      // token within block
    const int e0 = (tid % geo.tpt) * CE;
    const int t0 = blockIdx.x * TB;
    const bool active = tid < geo.threads;

    for (int q = tid; q < 2 * E; q += blockDim.x) sh_hist[q] = 0;

    float acc[CE];
#pragma unroll
    for (int c = 0; c < CE; ++c) acc[c] = 0.f;

    const int ntiles = ceil_div(d, geo.dt);
    gate_load_tile(x, wg, T, d, E, t0, geo, 0, buf0);
    cp_async_commit();
    for (int it = 0; it < ntiles; ++it) {
        uint8_t* cur = (it & 1) ? buf1 : buf0;
        uint8_t* nxt = (it & 1) ? buf0 : buf1;
        if (it + 1 < ntiles) gate_load_tile(x, wg, T, d, E, t0, geo, (it + 1) * geo.dt, nxt);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const int ilim = min(geo.dt, d - it * geo.dt);
        if (active && t0 + r < T) {
            const Elt* xr = reinterpret_cast<const Elt*>(cur + (size_t)r * geo.row_bytes);
            const float* ws = reinterpret_cast<const float*>(cur + (size_t)TB * geo.row_bytes) + e0;
            if constexpr (sizeof(Elt) == 2) {
                // two x values per 32-bit shared load
                const uint32_t* xp = reinterpret_cast<const uint32_t*>(xr);
#pragma unroll 4
                for (int i = 0; i < ilim; i += 2) {    // R1: increasing i, one fused step each
                    const uint32_t pr = xp[i >> 1];
                    gate_fma_row<CE>(ws + i * E, __uint_as_float(pr << 16), acc);
                    gate_fma_row<CE>(ws + (i + 1) * E, __uint_as_float(pr & 0xffff0000u), acc);
                }
            } else {
#pragma unroll 8
                for (int i = 0; i < ilim; ++i)         // R1: increasing i, one fused step each
                    gate_fma_row<CE>(ws + i * E, to_f(xr[i]), acc);
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();

    float* lg = reinterpret_cast<float*>(gsm);        // [TB][E]; x buffers are free now
    if (active) {
#pragma unroll
        for (int c = 0; c < CE; ++c) {
            lg[r * E + e0 + c] = acc[c];
            if (t0 + r < T) logits[(size_t)(t0 + r) * E + e0 + c] = acc[c];
        }
    }
    __syncthreads();

    const int tile0 = t0 / kScanTile;
    if (tid < TB && t0 + tid < T) {
        const int t = t0 + tid;
        const float* l = lg + tid * E;
        int sel[kMaxK];
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) {
            if (j >= k) break;
            int best = -1;
            float bv = 0.f;
            for (int e2 = 0; e2 < E; ++e2) {
                bool taken = false;
#pragma unroll
                for (int jj = 0; jj < kMaxK; ++jj)
                    if (jj < j && sel[jj] == e2) taken = true;
                if (taken) continue;
                const float v = l[e2];
                if (best < 0 || v > bv) { best = e2; bv = v; }   // strict >: ties -> lower e
            }
            sel[j] = best;
        }
        const float m = l[sel[0]];
        float s = 0.f;
        for (int e2 = 0; e2 < E; ++e2) s += expf(l[e2] - m);
        float ev[kMaxK], ssel = 0.f;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
            if (j < k) { ev[j] = expf(l[sel[j]] - m); ssel += ev[j]; }
        const float denom = renorm ? ssel : s;
        const int tile = t / kScanTile - tile0;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) {
            if (j < k) {
                idx_out[(size_t)t * k + j] = sel[j];
                w_out[(size_t)t * k + j] = ev[j] / denom;
                atomicAdd(&sh_hist[tile * E + sel[j]], 1);
            }
        }
    }
    __syncthreads();
    for (int q = tid; q < 2 * E; q += blockDim.x) {
        const int tile = tile0 + q / E;
        if (sh_hist[q] && tile < n_tiles) atomicAdd(&hist[tile * E + (q % E)], sh_hist[q]);
    }
}

// One block per kScanTile tokens.  smem: base[E] | wcnt[32][E] | wbal[32][E] | adm[E]
__global__ void __launch_bounds__(kScanTile)
slot_scan_kernel(const int* __restrict__ idx, int T, int k, int E, int C, int n,
                 const int* __restrict__ hist, int n_tiles, int* __restrict__ slot_out,
                 int* __restrict__ S, int* __restrict__ send_rows, int* __restrict__ send_off)
{
    extern __shared__ int ism[];
    int* base = ism;
    int* wcnt = base + E;
    unsigned* wbal = reinterpret_cast<unsigned*>(wcnt + 32 * E);
    int* adm = reinterpret_cast<int*>(wbal + 32 * E);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int b = blockIdx.x;

    if (tid < E) {
        int s = 0;
        for (int q = 0; q < b; ++q) s += hist[q * E + tid];
        base[tid] = s;
        if (b == 0) {
            int tot = 0;
            for (int q = 0; q < n_tiles; ++q) tot += hist[q * E + tid];
            const int a = min(C, tot);
            adm[tid] = a;
            S[tid * (n + 1)] = 0;
            S[tid * (n + 1) + n] = a;
            send_rows[tid] = a;
        }
    }

    const int t = b * kScanTile + tid;
    const bool valid = t < T;
    int mine[kMaxK], pre[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
        mine[j] = (valid && j < k) ? idx[(size_t)t * k + j] : -1;
        pre[j] = 0;
    }
    const int cs = valid ? chunk_starting_at(T, n, t) : -1;
    const bool warp_has_cs = __any_sync(0xffffffffu, cs >= 0);
    const unsigned lt = (1u << lane) - 1u;
    for (int e = 0; e < E; ++e) {
        bool has = false;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) has |= (mine[j] == e);
        const unsigned bal = __ballot_sync(0xffffffffu, has);
        if (lane == 0) {
            wcnt[w * E + e] = __popc(bal);
            if (warp_has_cs) wbal[w * E + e] = bal;
        }
        const int p = __popc(bal & lt);
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
            if (mine[j] == e) pre[j] = p;
    }
    __syncthreads();
    if (tid < E) {
        int run = 0;
        for (int ww = 0; ww < 32; ++ww) {
            const int c = wcnt[ww * E + tid];
            wcnt[ww * E + tid] = run;
            run += c;
        }
    }
    __syncthreads();
    if (valid) {
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) {
            if (j < k) {
                const int e = mine[j];
                const int P = base[e] + wcnt[w * E + e] + pre[j];
                slot_out[(size_t)t * k + j] = P < C ? P : -1;
            }
        }
    }
    if (cs >= 0) {
        for (int e = 0; e < E; ++e) {
            const int P = base[e] + wcnt[w * E + e] + __popc(wbal[w * E + e] & lt);
            S[e * (n + 1) + cs] = min(C, P);
        }
    }
    if (b == 0) {
        __syncthreads();
        if (tid == 0) {
            int off = 0;
            for (int e = 0; e < E; ++e) {
                send_off[e] = off;
                off += round_up(adm[e], kRowAlign);
            }
        }
    }
}

int launch_routing(const RouteArgs& a, bool is_bf16, cudaStream_t s)
{
    const int n_tiles = ceil_div(a.T, kScanTile);
    cudaMemsetAsync(a.hist, 0, sizeof(int) * n_tiles * a.E, s);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gate_topk_kernel<bf16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(gate_topk_kernel<bf16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(gate_topk_kernel<float, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(gate_topk_kernel<bf16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(gate_topk_kernel<float, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(gate_topk_kernel<float, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(slot_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    const GateGeom g = gate_geom(a.E, is_bf16 ? 2 : 4);
    const int blocks = ceil_div(a.T, g.TB);
    const int thr = round_up(g.threads, 32);
#define GATE_ARGS a.T, a.d, a.E, a.k, a.renorm, a.logits, a.idx, a.w, a.hist, n_tiles
    if (is_bf16) {
        if (g.ce == 2) gate_topk_kernel<bf16, 2><<<blocks, thr, g.smem, s>>>((const bf16*)a.x, a.wg, GATE_ARGS);
        else if (g.ce == 4) gate_topk_kernel<bf16, 4><<<blocks, thr, g.smem, s>>>((const bf16*)a.x, a.wg, GATE_ARGS);
        else gate_topk_kernel<bf16, 1><<<blocks, thr, g.smem, s>>>((const bf16*)a.x, a.wg, GATE_ARGS);
    } else {
        if (g.ce == 2) gate_topk_kernel<float, 2><<<blocks, thr, g.smem, s>>>((const float*)a.x, a.wg, GATE_ARGS);
        else if (g.ce == 4) gate_topk_kernel<float, 4><<<blocks, thr, g.smem, s>>>((const float*)a.x, a.wg, GATE_ARGS);
        else gate_topk_kernel<float, 1><<<blocks, thr, g.smem, s>>>((const float*)a.x, a.wg, GATE_ARGS);
    }
#undef GATE_ARGS
    const size_t smem2 = sizeof(int) * (a.E + 32 * a.E + 32 * a.E + a.E);
    slot_scan_kernel<<<n_tiles, kScanTile, smem2, s>>>(a.idx, a.T, a.k, a.E, a.C, a.n_chunks,
                                                       a.hist, n_tiles, a.slot, a.S, a.send_rows,
                                                       a.send_off);
    return 2;
}

}  // namespace lancet
