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

constexpr int kGateThreads = 256;
constexpr int kGateTPT = 4;    // (token, expert) chains per thread: 4 tokens x 1 expert
constexpr int kGateTI = 64;    // d-tile staged in shared memory
constexpr int kGateMaxGroups = 64;   // <= 256 tokens per block

template <typename Elt>
__global__ void __launch_bounds__(kGateThreads)
gate_topk_kernel(const Elt* __restrict__ x, const float* __restrict__ wg, int T, int d, int E,
                 int k, int renorm, float* __restrict__ logits, int* __restrict__ idx_out,
                 float* __restrict__ w_out, int* __restrict__ hist, int n_tiles)
{
    extern __shared__ float smem[];
    __shared__ int sh_hist[2 * kMaxExperts];
    const int ngroups = min(kGateThreads / E, kGateMaxGroups);
    const int TB = ngroups * kGateTPT;              // tokens of this block (<= 256)
    constexpr int LD = kGateTI + 1;
    float* xs = smem;                                // [TB][LD]
    float* ws = xs + TB * LD;                        // [TI][E]
    const int tid = threadIdx.x;
    const int e = tid % E, grp = tid / E;
    const bool active = grp < ngroups;
    const int t0 = blockIdx.x * TB;

    for (int q = tid; q < 2 * E; q += kGateThreads) sh_hist[q] = 0;

    float acc[kGateTPT];
#pragma unroll
    for (int c = 0; c < kGateTPT; ++c) acc[c] = 0.f;

    for (int i0 = 0; i0 < d; i0 += kGateTI) {
        const int ilim = min(kGateTI, d - i0);
        for (int q = tid; q < TB * kGateTI; q += kGateThreads) {
            const int r = q / kGateTI, c = q % kGateTI, t = t0 + r;
            xs[r * LD + c] = (t < T && c < ilim) ? to_f(x[(size_t)t * d + i0 + c]) : 0.f;
        }
        for (int q = tid; q < kGateTI * E; q += kGateThreads) {
            const int i = q / E;
            ws[q] = (i < ilim) ? wg[(size_t)(i0 + i) * E + (q % E)] : 0.f;
        }
        __syncthreads();
        if (active) {
            const float* xr = xs + grp * kGateTPT * LD;
            for (int i = 0; i < ilim; ++i) {            // R1: increasing i, fused steps
                const float wv = ws[i * E + e];
#pragma unroll
                for (int c = 0; c < kGateTPT; ++c) acc[c] = __fmaf_rn(xr[c * LD + i], wv, acc[c]);
            }
        }
        __syncthreads();
    }

    float* lg = smem;                                // [TB][E] (xs is free now)
    if (active) {
#pragma unroll
        for (int c = 0; c < kGateTPT; ++c) {
            const int r = grp * kGateTPT + c, t = t0 + r;
            lg[r * E + e] = acc[c];
            if (t < T) logits[(size_t)t * E + e] = acc[c];
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
    for (int q = tid; q < 2 * E; q += kGateThreads) {
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

size_t routing_smem_bytes(int E);

int launch_routing(const RouteArgs& a, bool is_bf16, cudaStream_t s)
{
    const int n_tiles = ceil_div(a.T, kScanTile);
    cudaMemsetAsync(a.hist, 0, sizeof(int) * n_tiles * a.E, s);
    const size_t smem = routing_smem_bytes(a.E);
    const int TB = std::min(kGateThreads / a.E, kGateMaxGroups) * kGateTPT;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gate_topk_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(gate_topk_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(slot_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    const int blocks = ceil_div(a.T, TB);
    if (is_bf16)
        gate_topk_kernel<bf16><<<blocks, kGateThreads, smem, s>>>(
            (const bf16*)a.x, a.wg, a.T, a.d, a.E, a.k, a.renorm, a.logits, a.idx, a.w, a.hist,
            n_tiles);
    else
        gate_topk_kernel<float><<<blocks, kGateThreads, smem, s>>>(
            (const float*)a.x, a.wg, a.T, a.d, a.E, a.k, a.renorm, a.logits, a.idx, a.w, a.hist,
            n_tiles);
    const size_t smem2 = sizeof(int) * (a.E + 32 * a.E + 32 * a.E + a.E);
    slot_scan_kernel<<<n_tiles, kScanTile, smem2, s>>>(a.idx, a.T, a.k, a.E, a.C, a.n_chunks,
                                                       a.hist, n_tiles, a.slot, a.S, a.send_rows,
                                                       a.send_off);
    return 2;
}

// Host-side shared-memory needs (checked against the device limit at context creation).
size_t routing_smem_bytes(int E)
{
    const int TB = std::min(kGateThreads / E, kGateMaxGroups) * kGateTPT;
    return sizeof(float) * (TB * (kGateTI + 1) + kGateTI * E);
}

}  // namespace lancet
