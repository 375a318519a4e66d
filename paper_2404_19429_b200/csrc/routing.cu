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

// d-tile staged in shared memory (cp.async ring): 128 dims, 64 when 8 experts per thread (the
// Wg tile, DT x E fp32, dominates the stage and bounds the blocks per SM)
__host__ __device__ constexpr int gate_dt(int ce) { return ce >= 8 ? 64 : 128; }
__host__ __device__ constexpr int gate_stages(int ce) { return ce >= 8 ? 3 : 4; }   // ring depth
constexpr int kGateThreads = 256;
constexpr int kGateMaxTB = 64;   // tokens per block (T=16k -> 256 blocks, all resident)

// Thread (tokens r..r+TT-1, experts e0..e0+CE-1) runs TT*CE independent R1 chains, two at a
// time with the packed fp32 FMA (fma.rn.f32x2: two IEEE fused multiply-adds, each rounded once
// -- bitwise the same as two fmaf).  CE = 8, 4, 2 or 1 (largest dividing E); TT = 2 tokens per
// thread when CE >= 4, so each staged Wg value feeds two tokens (the kernel is bound by
// shared-memory reads and FMA-chain latency, not by HBM).
struct GateGeom {
    int ce;        // experts (R1 chains) per thread
    int tt;        // tokens per thread
    int tpt;       // threads per token group = E / ce
    int TB;        // tokens per block
    int threads;   // TB / tt * tpt
    int row_bytes; // bytes per staged x row (kGateDT elements + 16 B against bank conflicts)
    size_t x_bytes, buf_bytes, smem;
};

__host__ __device__ inline int gate_ce(int E)
{
    return (E % 8 == 0 && E >= 16) ? 8 : (E % 4 == 0) ? 4 : (E % 2 == 0) ? 2 : 1;
}

// floats per expert group of the staged Wg tile (+4: groups start in different banks)
__host__ __device__ constexpr int gate_wg_stride(int ce) { return gate_dt(ce) * ce + 4; }

__host__ __device__ inline GateGeom gate_geom(int E, int elt_bytes)
{
    GateGeom g;
    g.ce = gate_ce(E);
    g.tt = g.ce >= 4 ? 2 : 1;
    g.tpt = E / g.ce;
    g.TB = kGateThreads * g.tt / g.tpt;
    if (g.TB > kGateMaxTB) g.TB = kGateMaxTB;
    if (g.TB < g.tt) g.TB = g.tt;
    g.threads = g.TB / g.tt * g.tpt;
    g.row_bytes = gate_dt(g.ce) * elt_bytes + 16;
    g.x_bytes = (size_t)g.TB * g.row_bytes;
    g.buf_bytes = g.x_bytes + (size_t)g.tpt * gate_wg_stride(g.ce) * 4;   // x tile | Wg tile [E/CE][DT][CE]
    const size_t xs = gate_stages(g.ce) * g.buf_bytes;
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

// acc = fma(x, w, acc) on both halves (one IEEE rounding each)
__device__ __forceinline__ void ffma2(float2& acc, float x, float2 w)
{
    asm("{\n\t.reg .b64 xx, ww, aa;\n\t"
        "mov.b64 xx, {%2, %2};\n\t"
        "mov.b64 ww, {%3, %4};\n\t"
        "mov.b64 aa, {%0, %1};\n\t"
        "fma.rn.f32x2 aa, xx, ww, aa;\n\t"
        "mov.b64 {%0, %1}, aa;\n\t}"
        : "+f"(acc.x), "+f"(acc.y)
        : "f"(x), "f"(w.x), "f"(w.y));
}

// Stage x rows [t0, t0+TB) x dims [i0, i0+ilim) and Wg rows [i0, i0+ilim), the latter
// regrouped as [E/CE][DT][CE] so a thread's CE weights of one dim are contiguous.
template <typename Elt, int CE>
__device__ __forceinline__ void gate_load_tile(const Elt* __restrict__ x, const float* __restrict__ wg,
                                               int T, int d, int E, int t0, const GateGeom& geo,
                                               int i0, uint8_t* buf)
{
    constexpr int DT = gate_dt(CE);
    const int ilim = min(DT, d - i0);
    constexpr int kFull = DT * (int)sizeof(Elt) / 16;            // 16-byte chunks per full row
    if (ilim == DT) {
        for (int q = threadIdx.x; q < geo.TB * kFull; q += blockDim.x) {
            const int r = q / kFull, c = q % kFull, t = t0 + r;     // kFull: power of two
            if (t < T)
                cp_async16(buf + (size_t)r * geo.row_bytes + c * 16,
                           reinterpret_cast<const uint8_t*>(x + (size_t)t * d + i0) + c * 16);
        }
    } else {
        const int cpr = ilim * (int)sizeof(Elt) / 16;
        for (int q = threadIdx.x; q < geo.TB * cpr; q += blockDim.x) {
            const int r = q / cpr, c = q % cpr, t = t0 + r;
            if (t < T)
                cp_async16(buf + (size_t)r * geo.row_bytes + c * 16,
                           reinterpret_cast<const uint8_t*>(x + (size_t)t * d + i0) + c * 16);
        }
    }
    float* wb = reinterpret_cast<float*>(buf + geo.x_bytes);
    const float* wsrc = wg + (size_t)i0 * E;
    if constexpr (CE >= 4) {
        const int q4 = E / 4;                                     // 16-byte chunks per Wg row
        for (int q = threadIdx.x; q < ilim * q4; q += blockDim.x) {
            const int i = q / q4, e = (q % q4) * 4;
            cp_async16(wb + (size_t)(e / CE) * gate_wg_stride(CE) + i * CE + (e % CE), wsrc + (size_t)i * E + e);
        }
    } else {
        for (int q = threadIdx.x; q < ilim * E; q += blockDim.x) {
            const int i = q / E, e = q % E;
            wb[(size_t)(e / CE) * gate_wg_stride(CE) + i * CE + (e % CE)] = __ldg(wsrc + q);
        }
    }
}

// Top-k selection (R2: logit desc, expert asc) and combine weights (R3) of token t from its
// E fp32 logits l; counts the choices into the block's per-scan-tile histogram row.
__device__ __forceinline__ void gate_select_token(const float* l, int t, int E, int k, int renorm,
                                                  int* __restrict__ idx_out, float* __restrict__ w_out,
                                                  int* sh_hist_row)
{
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
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
        if (j < k) {
            idx_out[(size_t)t * k + j] = sel[j];
            w_out[(size_t)t * k + j] = ev[j] / denom;
            atomicAdd(&sh_hist_row[sel[j]], 1);
        }
    }
}

// K1.  Tiles of x and of Wg stream through shared memory (cp.async ring).
template <typename Elt, int CE, int TT>
__global__ void __launch_bounds__(kGateThreads)
gate_topk_kernel(const Elt* __restrict__ x, const float* __restrict__ wg, int T, int d, int E,
                 int k, int renorm, float* __restrict__ logits, int* __restrict__ idx_out,
                 float* __restrict__ w_out, int* __restrict__ hist, int n_tiles)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    extern __shared__ __align__(16) uint8_t gsm[];
    __shared__ int sh_hist[2 * kMaxExperts];
    constexpr int V = Vec16<Elt>::N;                  // x values per 16-byte shared load
    constexpr int P = CE >= 2 ? CE / 2 : 1;           // packed chain pairs
    const GateGeom geo = gate_geom(E, sizeof(Elt));
    const int TB = geo.TB;
    const int tid = threadIdx.x;
    const int q = tid / geo.tpt;                      // token group: rows q*TT .. q*TT+TT-1
    const int grp = tid % geo.tpt;                    // expert group: e0 = grp * CE
    const int e0 = grp * CE;
    const int t0 = blockIdx.x * TB;
    const bool active = tid < geo.threads;

    for (int i = tid; i < 2 * E; i += blockDim.x) sh_hist[i] = 0;

    float2 acc2[TT][P];
    float acc1[TT];
#pragma unroll
    for (int u = 0; u < TT; ++u) {
        acc1[u] = 0.f;
#pragma unroll
        for (int c = 0; c < P; ++c) acc2[u][c] = make_float2(0.f, 0.f);
    }

    constexpr int DT = gate_dt(CE), NS = gate_stages(CE);
    const int ntiles = ceil_div(d, DT);
#pragma unroll
    for (int st = 0; st < NS - 1; ++st) {                      // prologue: tiles 0..S-2
        if (st < ntiles) gate_load_tile<Elt, CE>(x, wg, T, d, E, t0, geo, st * DT, gsm + st * geo.buf_bytes);
        cp_async_commit();
    }
    for (int it = 0; it < ntiles; ++it) {
        uint8_t* cur = gsm + (it % NS) * geo.buf_bytes;
        const int nx = it + NS - 1;                             // refill the slot freed last round
        if (nx < ntiles) gate_load_tile<Elt, CE>(x, wg, T, d, E, t0, geo, nx * DT, gsm + (nx % NS) * geo.buf_bytes);
        cp_async_commit();
        cp_async_wait<NS - 1>();
        __syncthreads();
        const int ilim = min(DT, d - it * DT);        // multiple of 8 (d % 8 == 0)
        if (active) {
            const uint8_t* xrow = cur + (size_t)(q * TT) * geo.row_bytes;
            const float* wp = reinterpret_cast<const float*>(cur + geo.x_bytes) + (size_t)grp * gate_wg_stride(CE);
#pragma unroll 2
            for (int iv = 0; iv < ilim / V; ++iv) {
                float xf[TT][V];
#pragma unroll
                for (int u = 0; u < TT; ++u)
                    unpack16<Elt>(reinterpret_cast<const uint4*>(xrow + (size_t)u * geo.row_bytes)[iv], xf[u]);
                const float* w = wp + iv * V * CE;
#pragma unroll
                for (int s = 0; s < V; ++s) {                   // R1: increasing i, one fused step each
                    if constexpr (CE >= 4) {
#pragma unroll
                        for (int h = 0; h < CE / 4; ++h) {
                            const float4 w4 = *reinterpret_cast<const float4*>(w + s * CE + 4 * h);
#pragma unroll
                            for (int u = 0; u < TT; ++u) {
                                ffma2(acc2[u][2 * h], xf[u][s], make_float2(w4.x, w4.y));
                                ffma2(acc2[u][2 * h + 1], xf[u][s], make_float2(w4.z, w4.w));
                            }
                        }
                    } else if constexpr (CE == 2) {
                        const float2 w2 = *reinterpret_cast<const float2*>(w + s * 2);
#pragma unroll
                        for (int u = 0; u < TT; ++u) ffma2(acc2[u][0], xf[u][s], w2);
                    } else {
#pragma unroll
                        for (int u = 0; u < TT; ++u) acc1[u] = __fmaf_rn(xf[u][s], w[s], acc1[u]);
                    }
                }
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();

    float* lg = reinterpret_cast<float*>(gsm);        // [TB][E]; x buffers are free now
    if (active) {
#pragma unroll
        for (int u = 0; u < TT; ++u) {
            const int r = q * TT + u;
            float acc[CE];
            if constexpr (CE >= 2) {
#pragma unroll
                for (int c = 0; c < P; ++c) { acc[2 * c] = acc2[u][c].x; acc[2 * c + 1] = acc2[u][c].y; }
            } else {
                acc[0] = acc1[u];
            }
#pragma unroll
            for (int c = 0; c < CE; ++c) lg[r * E + e0 + c] = acc[c];
            if (t0 + r < T) {
                float* dst = logits + (size_t)(t0 + r) * E + e0;
                if constexpr (CE % 4 == 0) {
#pragma unroll
                    for (int c = 0; c < CE; c += 4) *reinterpret_cast<float4*>(dst + c) = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
                } else {
#pragma unroll
                    for (int c = 0; c < CE; ++c) dst[c] = acc[c];
                }
            }
        }
    }
    __syncthreads();

    const int tile0 = t0 / kScanTile;
    for (int rr = tid; rr < TB; rr += blockDim.x) {
        const int t = t0 + rr;
        if (t >= T) break;
        gate_select_token(lg + rr * E, t, E, k, renorm, idx_out, w_out, sh_hist + (t / kScanTile - tile0) * E);
    }
    __syncthreads();
    for (int q = tid; q < 2 * E; q += blockDim.x) {
        const int tile = tile0 + q / E;
        if (sh_hist[q] && tile < n_tiles) atomicAdd(&hist[tile * E + (q % E)], sh_hist[q]);
    }
}


// ---------------------------------------------------------------------------------------
// K1, warp-streaming variant (E % 4 == 0, d % 64 == 0, Wg resident in shared memory): the
// whole Wg is staged once per block (regrouped [E/4][d][4]); each warp then streams its own
// tokens' x rows through a private cp.async ring of 64-dim slices and runs the R1 chains with
// no block barrier in the loop.  Thread (token lane/tpt, experts 4*(lane%tpt)..+3), two
// chains per fma.rn.f32x2.  4 warps per block; 2 blocks per SM at d = 1024, E = 8.
constexpr int kGsDT = 64;
constexpr int kGsCE = 4, kGsTT = 1;   // experts per thread, tokens per thread (CE=2 / CE=8 /
                                      // TT=2 measured slower)
constexpr int kGsTokensPerBlock = 64; // 4 warps at E = 8, 8 at E = 16
constexpr size_t kGsSmemMax = 110 * 1024;   // two blocks per SM

__host__ __device__ inline int gs_tpw(int E) { return 32 / (E / kGsCE) * kGsTT; } // tokens per warp
__host__ __device__ inline int gs_row_bytes(int elt) { return kGsDT * elt + 16; }
__host__ __device__ inline size_t gs_wg_bytes(int d, int E) { return (size_t)(E / kGsCE) * (d * kGsCE + 4) * 4; }
__host__ __device__ inline int gs_warps(int E) { return kGsTokensPerBlock / gs_tpw(E) > 0 ? kGsTokensPerBlock / gs_tpw(E) : 1; }
// ring depth: 8 slices if they fit beside the resident Wg, else 4
static int gs_stages(int d, int E, int elt)
{
    const size_t per_stage = (size_t)gs_warps(E) * gs_tpw(E) * gs_row_bytes(elt);
    return gs_wg_bytes(d, E) + 8 * per_stage <= kGsSmemMax ? 8 : 4;
}
static size_t gs_smem(int d, int E, int elt)
{
    // a warp's logits [tpw][E] fit in its ring
    return gs_wg_bytes(d, E) + (size_t)gs_stages(d, E, elt) * gs_warps(E) * gs_tpw(E) * gs_row_bytes(elt);
}
static bool gs_ok(int d, int E, int elt)
{
    return E % 4 == 0 && E / kGsCE <= 32 && 32 % (E / kGsCE) == 0 && d % kGsDT == 0 && gs_warps(E) <= 16 &&
           gs_smem(d, E, elt) <= kGsSmemMax;
}

template <typename Elt, int S>
__global__ void __launch_bounds__(512)
gate_stream_kernel(const Elt* __restrict__ x, const float* __restrict__ wg, int T, int d, int E,
                   int k, int renorm, float* __restrict__ logits, int* __restrict__ idx_out,
                   float* __restrict__ w_out, int* __restrict__ hist, int n_tiles)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    extern __shared__ __align__(16) uint8_t gsm[];
    __shared__ int sh_hist[2 * kMaxExperts];
    constexpr int V = Vec16<Elt>::N;                   // dims per 16-byte chunk
    constexpr int CPR = kGsDT / V;                     // chunks per row slice
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int CE = kGsCE, TT = kGsTT;
    const int tpt = E / CE, tpw = 32 / tpt * TT;
    const int RB = gs_row_bytes(sizeof(Elt));
    const int gstride = d * CE + 4;                    // floats per expert group (+4: bank offset)
    float* swg = reinterpret_cast<float*>(gsm);
    uint8_t* ring = gsm + gs_wg_bytes(d, E) + (size_t)warp * S * tpw * RB;
    const int t0 = blockIdx.x * (int)(blockDim.x >> 5) * tpw;
    const int tw = t0 + warp * tpw;                    // this warp's first token

    for (int i = tid; i < 2 * E; i += blockDim.x) sh_hist[i] = 0;
    // Wg [d][E] -> swg[(e/CE) * gstride + i * CE + e % CE]
    {
        const int q4 = E / 4;
        for (int q = tid; q < d * q4; q += blockDim.x) {
            const int i = q / q4, e = (q % q4) * 4;
            if constexpr (CE == 4) {
                cp_async16(swg + (size_t)(e / 4) * gstride + i * 4, wg + (size_t)i * E + e);
            } else {
                const float4 v = __ldg(reinterpret_cast<const float4*>(wg + (size_t)i * E + e));
                *reinterpret_cast<float2*>(swg + (size_t)(e / 2) * gstride + i * 2) = make_float2(v.x, v.y);
                *reinterpret_cast<float2*>(swg + (size_t)(e / 2 + 1) * gstride + i * 2) = make_float2(v.z, v.w);
            }
        }
        cp_async_commit();
    }
    const int nst = d / kGsDT;
    auto issue = [&](int st) {
        uint8_t* slot = ring + (size_t)(st % S) * tpw * RB;
        for (int q = lane; q < tpw * CPR; q += 32) {
            const int rr = q / CPR, c = q % CPR, t = tw + rr;
            if (t < T)
                cp_async16(slot + rr * RB + c * 16,
                           reinterpret_cast<const uint8_t*>(x + (size_t)t * d + st * kGsDT) + c * 16);
        }
    };
#pragma unroll
    for (int st = 0; st < S - 1; ++st) {
        if (st < nst) issue(st);
        cp_async_commit();
    }
    cp_async_wait<S - 1>();                            // Wg (the oldest group) has landed
    __syncthreads();

    const int r = lane / tpt, grp = lane % tpt;        // tokens r*TT .. r*TT+TT-1
    const float* wbase = swg + (size_t)grp * gstride;
    float2 acc0[TT], acc1[TT];
#pragma unroll
    for (int u = 0; u < TT; ++u) acc0[u] = acc1[u] = make_float2(0.f, 0.f);
    for (int st = 0; st < nst; ++st) {
        if (st + S - 1 < nst) issue(st + S - 1);
        cp_async_commit();
        cp_async_wait<S - 1>();
        __syncwarp();                                  // every lane's pieces of slice st landed
        const uint8_t* xrow = ring + (size_t)(st % S) * tpw * RB + (size_t)(r * TT) * RB;
        const float* wp = wbase + st * kGsDT * CE;
#pragma unroll
        for (int c = 0; c < CPR; ++c) {
            float xf[TT][V];
#pragma unroll
            for (int tt = 0; tt < TT; ++tt)
                unpack16<Elt>(reinterpret_cast<const uint4*>(xrow + tt * RB)[c], xf[tt]);
#pragma unroll
            for (int u = 0; u < V; ++u) {               // R1: increasing i, one fused step each
                if constexpr (CE == 4) {
                    const float4 w4 = *reinterpret_cast<const float4*>(wp + (c * V + u) * 4);
#pragma unroll
                    for (int tt = 0; tt < TT; ++tt) {
                        ffma2(acc0[tt], xf[tt][u], make_float2(w4.x, w4.y));
                        ffma2(acc1[tt], xf[tt][u], make_float2(w4.z, w4.w));
                    }
                } else {
                    const float2 w2 = *reinterpret_cast<const float2*>(wp + (c * V + u) * 2);
#pragma unroll
                    for (int tt = 0; tt < TT; ++tt) ffma2(acc0[tt], xf[tt][u], w2);
                }
            }
        }
        __syncwarp();                                  // slice read by all lanes before refill
    }
    cp_async_wait<0>();
    __syncwarp();
    // logits of the warp's tokens -> shared [tpw][E] in the warp's own (now idle) ring, then
    // top-k per token
    float* lg = reinterpret_cast<float*>(ring);
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) {
        const int rr = r * TT + tt, t = tw + rr;
        if constexpr (CE == 4) {
            const float4 v = make_float4(acc0[tt].x, acc0[tt].y, acc1[tt].x, acc1[tt].y);
            *reinterpret_cast<float4*>(lg + rr * E + grp * 4) = v;
            if (t < T) *reinterpret_cast<float4*>(logits + (size_t)t * E + grp * 4) = v;
        } else {
            *reinterpret_cast<float2*>(lg + rr * E + grp * 2) = acc0[tt];
            if (t < T) *reinterpret_cast<float2*>(logits + (size_t)t * E + grp * 2) = acc0[tt];
        }
    }
    __syncwarp();
    const int tile0 = t0 / kScanTile;
    for (int q = lane; q < tpw; q += 32)
        if (tw + q < T)
            gate_select_token(lg + q * E, tw + q, E, k, renorm, idx_out, w_out,
                              sh_hist + ((tw + q) / kScanTile - tile0) * E);
    __syncthreads();
    for (int q = tid; q < 2 * E; q += blockDim.x) {
        const int tile = tile0 + q / E;
        if (sh_hist[q] && tile < n_tiles) atomicAdd(&hist[tile * E + (q % E)], sh_hist[q]);
    }
}

// One block per kScanTile tokens.  smem: base[E] | wcnt[32][E] | wbal[32][E] | adm[E] | hist copy
constexpr int kScanHistMax = 16384;  // ints of the staged tile histograms (64 KiB)
__global__ void __launch_bounds__(kScanTile)
slot_scan_kernel(const int* __restrict__ idx, int T, int k, int E, int C, int n,
                 const int* __restrict__ hist, int n_tiles, int* __restrict__ slot_out,
                 int* __restrict__ S, int* __restrict__ send_rows, int* __restrict__ send_off)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    extern __shared__ int ism[];
    int* base = ism;
    int* wcnt = base + E;
    unsigned* wbal = reinterpret_cast<unsigned*>(wcnt + 32 * E);
    int* adm = reinterpret_cast<int*>(wbal + 32 * E);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int b = blockIdx.x;

    // the per-tile histograms, all loads in flight at once (a serial prefix of dependent global
    // loads would cost one L2 round trip per tile)
    int* sh_h = adm + E;                                   // [n_tiles][E] when it fits
    const bool staged = n_tiles * E <= kScanHistMax;
    if (staged) {
        for (int i = tid; i < n_tiles * E; i += blockDim.x) sh_h[i] = hist[i];
        __syncthreads();
    }
    const int* hs = staged ? sh_h : hist;
    if (tid < E) {
        int s = 0;
        for (int q = 0; q < b; ++q) s += hs[q * E + tid];
        base[tid] = s;
        if (b == 0) {
            int tot = 0;
            for (int q = 0; q < n_tiles; ++q) tot += hs[q * E + tid];
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
        for (int ww = 0; ww < kScanTile / 32; ++ww) {
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
#define SET(Elt, CE) cudaFuncSetAttribute(gate_topk_kernel<Elt, CE, (CE >= 4 ? 2 : 1)>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)
        SET(bf16, 8); SET(bf16, 4); SET(bf16, 2); SET(bf16, 1);
        SET(float, 8); SET(float, 4); SET(float, 2); SET(float, 1);
#undef SET
        cudaFuncSetAttribute(slot_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    const int elt = is_bf16 ? 2 : 4;
    if (gs_ok(a.d, a.E, elt)) {
        static bool gs_attr = false;
        if (!gs_attr) {
            cudaFuncSetAttribute(gate_stream_kernel<bf16, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            cudaFuncSetAttribute(gate_stream_kernel<float, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            cudaFuncSetAttribute(gate_stream_kernel<bf16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            cudaFuncSetAttribute(gate_stream_kernel<float, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            gs_attr = true;
        }
        const int W = gs_warps(a.E), per_block = W * gs_tpw(a.E), S = gs_stages(a.d, a.E, elt);
        const size_t smem = gs_smem(a.d, a.E, elt);
        const dim3 grid(ceil_div(a.T, per_block)), block(W * 32);
#define GS(Elt, SS) launch_k(gate_stream_kernel<Elt, SS>, grid, block, smem, s, (const Elt*)a.x, a.wg, a.T, a.d, \
                             a.E, a.k, a.renorm, a.logits, a.idx, a.w, a.hist, n_tiles)
        if (is_bf16) { if (S == 8) GS(bf16, 8); else GS(bf16, 4); }
        else { if (S == 8) GS(float, 8); else GS(float, 4); }
#undef GS
    } else {
    const GateGeom g = gate_geom(a.E, elt);
    const int blocks = ceil_div(a.T, g.TB);
    const int thr = round_up(g.threads, 32);
#define GATE_ARGS a.T, a.d, a.E, a.k, a.renorm, a.logits, a.idx, a.w, a.hist, n_tiles
#define GATE_LAUNCH(Elt)                                                                                    \
    switch (g.ce) {                                                                                         \
    case 8: launch_k(gate_topk_kernel<Elt, 8, 2>, blocks, thr, g.smem, s, (const Elt*)a.x, a.wg, GATE_ARGS); break;  \
    case 4: launch_k(gate_topk_kernel<Elt, 4, 2>, blocks, thr, g.smem, s, (const Elt*)a.x, a.wg, GATE_ARGS); break;  \
    case 2: launch_k(gate_topk_kernel<Elt, 2, 1>, blocks, thr, g.smem, s, (const Elt*)a.x, a.wg, GATE_ARGS); break;  \
    default: launch_k(gate_topk_kernel<Elt, 1, 1>, blocks, thr, g.smem, s, (const Elt*)a.x, a.wg, GATE_ARGS); break; \
    }
    if (is_bf16) { GATE_LAUNCH(bf16) } else { GATE_LAUNCH(float) }
#undef GATE_LAUNCH
#undef GATE_ARGS
    }
    const size_t smem2 = sizeof(int) * (a.E + 32 * a.E + 32 * a.E + a.E +
                                        (n_tiles * a.E <= kScanHistMax ? n_tiles * a.E : 0));
    launch_k(slot_scan_kernel, n_tiles, kScanTile, smem2, s, a.idx, a.T, a.k, a.E, a.C, a.n_chunks,
                                                       a.hist, n_tiles, a.slot, a.S, a.send_rows,
                                                       a.send_off);
    return 2;
}

}  // namespace lancet
