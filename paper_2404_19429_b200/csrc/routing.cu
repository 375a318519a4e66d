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
#include <cstdlib>

namespace lancet {

// d-tile staged in shared memory (cp.async ring): 128 dims, 64 when 8 experts per thread (the
// Wg tile, DT x E fp32, dominates the stage and bounds the blocks per SM)
__host__ __device__ constexpr int gate_dt(int ce) { return ce >= 8 ? 64 : 128; }
__host__ __device__ constexpr int gate_stages(int ce) { return ce >= 8 ? 3 : 4; }   // ring depth
constexpr int kGateThreads = 256;
constexpr int kGateMaxTB = 64;   // tokens per block (T=16k -> 256 blocks, all resident)
#ifndef LANCET_GATE_TT8
#define LANCET_GATE_TT8 4
#endif
// tokens per thread at 8 experts per thread (E >= 16 on the tiled path): each staged Wg value
// feeds 4 tokens.  ncu at d=1024 (round 1, session 3): E=64 T=16k 110 -> 92 us, T=64k 369 ->
// 299 us; E=32 66 -> 62 / 209 -> 182 us against 2; 8 tokens per thread is slower (fewer warps)
constexpr int kGateTT8 = LANCET_GATE_TT8;

// Thread (tokens r..r+TT-1, experts e0..e0+CE-1) runs TT*CE independent R1 chains, two at a
// time with the packed fp32 FMA (fma.rn.f32x2: two IEEE fused multiply-adds, each rounded once
// -- bitwise the same as two fmaf).  CE = 8, 4, 2 or 1 (largest dividing E); TT = 4 tokens per
// thread at CE = 8 and 2 at CE = 4, so each staged Wg value feeds several tokens (the kernel is
// bound by shared-memory reads and FMA-chain latency, not by HBM).
struct GateGeom {
    int ce;        // experts (R1 chains) per thread
    int tt;        // tokens per thread
    int tpt;       // threads per token group = E / ce
    int TB;        // tokens per block
    int threads;   // TB / tt * tpt
    int row_bytes; // bytes per staged x row (kGateDT elements + 16 B against bank conflicts)
    size_t x_bytes, buf_bytes, smem;
};

// experts (chains) per thread: 8 (x 4 tokens: each staged Wg value feeds 4 chains) where the
// batch still gives >= 4 warps per SM with them; else 4 (x 2 tokens), which quadruples the
// threads -- at T = 8192, E = 32 (configs[3]) 8 x 4 left 128 blocks of 2 warps for 148 SMs
constexpr int kGateMinThreads8 = 148 * 64;
__host__ __device__ inline int gate_ce(int E, int T)
{
    if (E % 8 == 0 && E >= 16 && (long)T * E / (8 * kGateTT8) >= kGateMinThreads8) return 8;
    return (E % 4 == 0) ? 4 : (E % 2 == 0) ? 2 : 1;
}

// floats per expert group of the staged Wg tile (+4: groups start in different banks)
__host__ __device__ constexpr int gate_wg_stride(int ce) { return gate_dt(ce) * ce + 4; }

__host__ __device__ inline GateGeom gate_geom(int E, int elt_bytes, int ce, int tb_max)
{
    GateGeom g;
    g.ce = ce;
    g.tt = g.ce >= 8 ? kGateTT8 : (g.ce >= 4 ? 2 : 1);
    g.tpt = E / g.ce;
    g.TB = kGateThreads * g.tt / g.tpt;
    if (g.TB > tb_max) g.TB = tb_max;
    g.TB = g.TB / g.tt * g.tt;                  // whole token groups (E = 192: 42 -> 40)
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
                 float* __restrict__ w_out, int* __restrict__ hist, int n_tiles, int tb_max)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    extern __shared__ __align__(16) uint8_t gsm[];
    __shared__ int sh_hist[2 * kMaxExperts];
    constexpr int V = Vec16<Elt>::N;                  // x values per 16-byte shared load
    constexpr int P = CE >= 2 ? CE / 2 : 1;           // packed chain pairs
    const GateGeom geo = gate_geom(E, sizeof(Elt), CE, tb_max);
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
// no block barrier in the loop.  Thread (tokens TT*(lane/tpt)..+TT-1, experts
// 4*(lane%tpt)..+3), two chains per fma.rn.f32x2 and token; 64 tokens per block.
constexpr int kGsDT = 64;
constexpr int kGsCE = 4;              // experts per thread (CE=2 / CE=8 measured slower)
constexpr int kGsTokensPerBlock = 64; // E = 8: 4 warps (1 token per thread) or 2 (2 tokens)
constexpr size_t kGsSmemMax = 110 * 1024;   // two blocks per SM

// tokens per thread: 2 where the batch still gives every SM a block (each staged Wg value
// then feeds two tokens: half the shared-memory bytes per FMA; E = 8 / 16 at T = 16k:
// -12 % / -31 %), else 1 (more warps)
static int gs_tt(int T, int E)
{
    static const int forced = [] { const char* e = getenv("LANCET_GATE_TT"); return e ? atoi(e) : 0; }();
    if (forced == 1 || forced == 2) return forced;   // A/B runs
    return (E <= 16 && T >= 148 * kGsTokensPerBlock) ? 2 : 1;
}
__host__ __device__ inline int gs_tpw(int E, int tt) { return 32 / (E / kGsCE) * tt; } // tokens per warp
__host__ __device__ inline int gs_row_bytes(int elt) { return kGsDT * elt + 16; }
__host__ __device__ inline size_t gs_wg_bytes(int d, int E) { return (size_t)(E / kGsCE) * (d * kGsCE + 4) * 4; }
__host__ __device__ inline int gs_warps(int E, int tt) { return kGsTokensPerBlock / gs_tpw(E, tt) > 0 ? kGsTokensPerBlock / gs_tpw(E, tt) : 1; }
// ring depth: 8 slices if they fit beside the resident Wg, else 4
static int gs_stages(int d, int E, int elt, int tt)
{
    const size_t per_stage = (size_t)gs_warps(E, tt) * gs_tpw(E, tt) * gs_row_bytes(elt);
    return gs_wg_bytes(d, E) + 8 * per_stage <= kGsSmemMax ? 8 : 4;
}
static size_t gs_smem(int d, int E, int elt, int tt)
{
    // a warp's logits [tpw][E] fit in its ring
    return gs_wg_bytes(d, E) + (size_t)gs_stages(d, E, elt, tt) * gs_warps(E, tt) * gs_tpw(E, tt) * gs_row_bytes(elt);
}
static bool gs_ok(int d, int E, int elt, int tt)
{
    return E % 4 == 0 && E / kGsCE <= 32 && 32 % (E / kGsCE) == 0 && d % kGsDT == 0 && gs_warps(E, tt) <= 16 &&
           gs_smem(d, E, elt, tt) <= kGsSmemMax;
}

template <typename Elt, int S, int TT>
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
    constexpr int CE = kGsCE;
    const int tpt = E / CE, tpw = 32 / tpt * TT;
    const int RB = gs_row_bytes(sizeof(Elt));
    const int gstride = d * CE + 4;                    // floats per expert group (+4: bank offset)
    float* swg = reinterpret_cast<float*>(gsm);
    uint8_t* ring = gsm + gs_wg_bytes(d, E) + (size_t)warp * S * tpw * RB;
    const int t0 = blockIdx.x * (int)(blockDim.x >> 5) * tpw;
    const int tw = t0 + warp * tpw;                    // this warp's first token

    for (int i = tid; i < 2 * E; i += blockDim.x) sh_hist[i] = 0;
    // Wg [d][E] -> swg[(e/4) * gstride + i * 4 + e % 4] (no integer division in the copy loop:
    // it showed up as ~15 % of the kernel's stall samples)
    for (int e4 = 0; e4 < E / 4; ++e4)
        for (int i = tid; i < d; i += blockDim.x)
            cp_async16(swg + (size_t)e4 * gstride + i * 4, wg + (size_t)i * E + e4 * 4);
    cp_async_commit();
    const int nst = d / kGsDT;
    // lane copies 16-byte column cl of rows rl, rl + RSTEP, ... of each slice (pointers stepped,
    // no per-copy 64-bit index arithmetic)
    constexpr int RSTEP = 32 / CPR;
    const int cl = lane % CPR, rl = lane / CPR;
    const uint8_t* xl = reinterpret_cast<const uint8_t*>(x) + (size_t)(tw + rl) * d * sizeof(Elt) + cl * 16;
    const size_t xstep = (size_t)RSTEP * d * sizeof(Elt);
    auto issue = [&](int st) {
        uint8_t* sl = ring + (size_t)(st % S) * tpw * RB + rl * RB + cl * 16;
        const uint8_t* g = xl + (size_t)st * kGsDT * sizeof(Elt);
        for (int rr = rl; rr < tpw; rr += RSTEP, sl += RSTEP * RB, g += xstep)
            if (tw + rr < T) cp_async16(sl, g);
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
                const float4 w4 = *reinterpret_cast<const float4*>(wp + (c * V + u) * CE);
#pragma unroll
                for (int tt = 0; tt < TT; ++tt) {
                    ffma2(acc0[tt], xf[tt][u], make_float2(w4.x, w4.y));
                    ffma2(acc1[tt], xf[tt][u], make_float2(w4.z, w4.w));
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

// K1 for the Random gate (R18): thread per token, block = one scan
// tile.  Draw j of token t: r = splitmix64(8t + j) mod (E - j), the r-th expert not drawn
// before (walking the earlier draws in increasing order); weights 1/k; logits reported as 0.
__device__ __forceinline__ unsigned long long splitmix64_at(unsigned long long key, unsigned long long seed)
{
    unsigned long long z = seed + (key + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void __launch_bounds__(kScanTile)
random_gate_kernel(int T, int E, int k, unsigned long long seed, float* __restrict__ logits,
                   int* __restrict__ idx_out, float* __restrict__ w_out, int* __restrict__ hist, int t_base)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    __shared__ int sh_hist[kMaxExperts];
    const int tid = threadIdx.x;
    for (int e = tid; e < E; e += blockDim.x) sh_hist[e] = 0;
    __syncthreads();
    const int t = blockIdx.x * kScanTile + tid;
    if (t < T) {
        int sorted[kMaxK];                              // earlier draws, ascending
        const float wk = 1.0f / (float)k;
        for (int j = 0; j < k; ++j) {
            int e = (int)(splitmix64_at(8ull * (unsigned long long)(t + t_base) + (unsigned long long)j, seed) %
                          (unsigned long long)(E - j));
            int pos = 0;
            for (int q = 0; q < j; ++q) {               // r-th free expert
                if (sorted[q] <= e) { ++e; pos = q + 1; }
            }
            for (int q = j; q > pos; --q) sorted[q] = sorted[q - 1];
            sorted[pos] = e;
            idx_out[(size_t)t * k + j] = e;
            w_out[(size_t)t * k + j] = wk;
            atomicAdd(&sh_hist[e], 1);
        }
        for (int e = 0; e < E; ++e) logits[(size_t)t * E + e] = 0.f;
    }
    __syncthreads();
    for (int e = tid; e < E; e += blockDim.x) hist[blockIdx.x * E + e] = sh_hist[e];
}

// The slot scan (K2) runs in one of three modes:
//   SCAN_SLOTS      token-major admission (R7): slot = P_e(t) if < C, capacity state S, offsets;
//   SCAN_BPR_LIST   Batch Prioritized Routing, pass 1 (R16): the unclamped P_e(t) of every pair
//                   places its pair id t*k+j at list[off_e + P_e(t)] (pairs grouped by expert, in
//                   token order), and the token's fp64 importance score is written;
//   SCAN_BPR_SLOTS  BPR pass 3: SCAN_SLOTS over the ADMITTED pairs only (bpr_adm), tile
//                   histograms from bpr_select_kernel -- slot = token-major rank among admitted.
enum ScanMode { SCAN_SLOTS = 0, SCAN_BPR_LIST = 1, SCAN_BPR_SLOTS = 2 };

// BPR importance score ("the sum of top-k largest gating scores", R16):
// s = (sum_j exp(l_idx_j - m)) / (sum_e exp(l_e - m)) in fp64, both sums sequential, m = the
// top-1 logit (= the row maximum by R2).
__device__ __forceinline__ double bpr_score(const float* __restrict__ lg, const int* mine, int E, int k)
{
    const double m = (double)lg[mine[0]];
    double Z = 0.0, num = 0.0;
    for (int e = 0; e < E; ++e) Z += exp((double)lg[e] - m);
    for (int j = 0; j < k; ++j) num += exp((double)lg[mine[j]] - m);
    return num / Z;
}

// One block per kScanTile tokens.  smem: base[E] | wcnt[32][E] | wbal[32][E] | adm[E] | offs[E] |
// hist copy
constexpr int kScanHistMax = 16384;  // ints of the staged tile histograms (64 KiB)
template <int MODE>
__global__ void __launch_bounds__(kScanTile)
slot_scan_kernel(const int* __restrict__ idx, int T, int k, int E, int C, int n,
                 const int* __restrict__ hist, int n_tiles, int* __restrict__ slot_out,
                 int* __restrict__ S, int* __restrict__ send_rows, int* __restrict__ send_off,
                 const float* __restrict__ logits, double* __restrict__ score, int* __restrict__ list,
                 int* __restrict__ bpr_meta, const unsigned char* __restrict__ bpr_adm,
                 const int* __restrict__ carry_in, int* __restrict__ carry_out, int carry_chunk,
                 int* __restrict__ carry_counts)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    extern __shared__ int ism[];
    int* base = ism;
    int* wcnt = base + E;
    unsigned* wbal = reinterpret_cast<unsigned*>(wcnt + 32 * E);
    int* adm = reinterpret_cast<int*>(wbal + 32 * E);
    int* offs = adm + E;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int b = blockIdx.x;

    // the per-tile histograms, all loads in flight at once (a serial prefix of dependent global
    // loads would cost one L2 round trip per tile)
    int* sh_h = offs + E;                                  // [n_tiles][E] when it fits
    const bool staged = n_tiles * E <= kScanHistMax;
    if (staged) {
        for (int i = tid; i < n_tiles * E; i += blockDim.x) sh_h[i] = hist[i];
        __syncthreads();
    }
    const int* hs = staged ? sh_h : hist;
    if (tid < E) {
        int s = carry_in ? carry_in[tid] : 0;    // capacity passing from earlier chunks (L255)
        for (int q = 0; q < b; ++q) s += hs[q * E + tid];
        base[tid] = s;
        if (MODE == SCAN_SLOTS && carry_in) {
            if (b == 0) {
                int tot = 0;
                for (int q = 0; q < n_tiles; ++q) tot += hs[q * E + tid];
                const int p0 = carry_in[tid], p1 = p0 + tot;
                const int s0 = min(C, p0), s1 = min(C, p1);
                carry_out[tid] = p1;
                S[tid * (n + 1) + carry_chunk] = s0;
                S[tid * (n + 1) + carry_chunk + 1] = s1;
                carry_counts[tid * n + carry_chunk] = s1 - s0;
            }
        } else if (MODE == SCAN_BPR_LIST) {
            int tot = 0;
            for (int q = 0; q < n_tiles; ++q) tot += hs[q * E + tid];
            adm[tid] = tot;                    // pairs routed to e (before any drop)
        } else if (b == 0) {
            int tot = 0;
            for (int q = 0; q < n_tiles; ++q) tot += hs[q * E + tid];
            const int a = min(C, tot);
            adm[tid] = a;
            S[tid * (n + 1)] = 0;
            S[tid * (n + 1) + n] = a;
            send_rows[tid] = a;
        }
    }
    if (MODE == SCAN_BPR_LIST) {
        __syncthreads();
        if (tid == 0) {
            int o = 0;
            for (int e = 0; e < E; ++e) { offs[e] = o; o += adm[e]; }
        }
        if (b == 0 && tid < E) bpr_meta[tid] = adm[tid];
    }

    const int t = b * kScanTile + tid;
    const bool valid = t < T;
    int mine[kMaxK], pre[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
        mine[j] = (valid && j < k) ? idx[(size_t)t * k + j] : -1;
        pre[j] = 0;
    }
    if (MODE == SCAN_BPR_LIST && valid) score[t] = bpr_score(logits + (size_t)t * E, mine, E, k);
    if (MODE == SCAN_BPR_SLOTS) {
        // dropped by priority: the pair takes no place in its expert's buffer
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
            if (j < k && valid && !bpr_adm[(size_t)t * k + j]) mine[j] = -2;
    }
    const int cs = (MODE != SCAN_BPR_LIST && valid && !carry_in) ? chunk_starting_at(T, n, t) : -1;
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
                if (MODE == SCAN_BPR_LIST) {
                    list[offs[e] + base[e] + wcnt[w * E + e] + pre[j]] = t * k + j;
                } else if (MODE == SCAN_BPR_SLOTS && e < 0) {
                    slot_out[(size_t)t * k + j] = -1;
                } else {
                    const int P = base[e] + wcnt[w * E + e] + pre[j];
                    slot_out[(size_t)t * k + j] = P < C ? P : -1;
                }
            }
        }
    }
    if (MODE == SCAN_BPR_LIST) return;
    if (cs >= 0) {
        for (int e = 0; e < E; ++e) {
            const int P = base[e] + wcnt[w * E + e] + __popc(wbal[w * E + e] & lt);
            S[e * (n + 1) + cs] = min(C, P);
        }
    }
    if (b == 0 && !carry_in) {
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

// BPR pass 2 (R16): one block per expert.  Expert e's pairs sit in list[off_e, off_e + n_e) in
// token order.  If n_e > C, an MSD radix select over the 64-bit patterns of the (positive)
// fp64 scores (monotone in the score) finds the byte-granular prefix K* of the C-th largest
// score and how many pairs sharing that prefix still fit; those go to the lower token indices
// (ordered block scan).  The select starts at the highest byte where the smallest and largest
// key differ (the scores share their exponent bytes) and stops as soon as the pairs sharing the
// prefix all fit.  Writes bpr_adm for every pair of e and the per-tile admitted counts
// hist2[tile][e] (every tile written: no memset needed).
constexpr int kSelThreads = 1024;
constexpr size_t kSelSmem = 200 * 1024;   // key cache + tile counts
__global__ void __launch_bounds__(kSelThreads)
bpr_select_kernel(const int* __restrict__ list, const int* __restrict__ bpr_meta,
                  const double* __restrict__ score, int E, int k, int C, int n_tiles, int cap,
                  unsigned char* __restrict__ bpr_adm, int* __restrict__ hist2)
{
    pdl_wait();
    extern __shared__ unsigned long long kcache[];  // [cap] keys of the first cap pairs of e
    int* tiles = reinterpret_cast<int*>(kcache + cap);   // [n_tiles] admitted pairs per token tile
    __shared__ int hist[256];
    __shared__ int wsum[kSelThreads / 32];
    __shared__ unsigned long long wmin[kSelThreads / 32], wmax[kSelThreads / 32];
    __shared__ unsigned long long s_prefix;
    __shared__ int s_need, s_run, s_shift, s_done;
    const int e = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    int off = 0;
    for (int q = 0; q < e; ++q) off += bpr_meta[q];
    const int ne = bpr_meta[e];
    const int* L = list + off;
    for (int q = tid; q < n_tiles; q += kSelThreads) tiles[q] = 0;
    const bool all = ne <= C;
    auto key_of = [&](int i) -> unsigned long long {
        return i < cap ? kcache[i] : (unsigned long long)__double_as_longlong(score[L[i] / k]);
    };
    if (!all) {
        // one gather pass stages the keys (the select passes and the admission re-read them;
        // pairs beyond the cache are re-gathered from global memory) and finds min / max
        unsigned long long mn = ~0ull, mx = 0ull;
        for (int i = tid; i < ne; i += kSelThreads) {
            const unsigned long long key = (unsigned long long)__double_as_longlong(score[L[i] / k]);
            if (i < cap) kcache[i] = key;
            mn = min(mn, key);
            mx = max(mx, key);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) { wmin[w] = mn; wmax[w] = mx; }
        __syncthreads();
        if (tid == 0) {
            for (int q = 1; q < kSelThreads / 32; ++q) { mn = min(mn, wmin[q]); mx = max(mx, wmax[q]); }
            mn = min(mn, wmin[0]); mx = max(mx, wmax[0]);
            s_need = C;
            s_run = 0;
            if (mn == mx) {                    // one score for every pair: all ties
                s_prefix = mn; s_shift = 0; s_done = 1;
            } else {
                const int hb = 63 - __clzll(mn ^ mx);          // highest differing bit
                const int sh = (hb / 8) * 8;                    // first byte to select on
                s_prefix = sh == 56 ? 0ull : (mn >> (sh + 8)) << (sh + 8);
                s_shift = sh + 8;                               // bytes above are common
                s_done = 0;
            }
        }
        __syncthreads();
        while (!s_done) {
            const int shift = s_shift - 8;
            for (int q = tid; q < 256; q += kSelThreads) hist[q] = 0;
            __syncthreads();
            const unsigned long long pre = s_prefix;
            for (int i = tid; i < ne; i += kSelThreads) {
                const unsigned long long key = key_of(i);
                if (shift == 56 || (key >> (shift + 8)) == (pre >> (shift + 8)))
                    atomicAdd(&hist[(key >> shift) & 255u], 1);
            }
            __syncthreads();
            if (w == 0) {
                // lane owns bins 255-8*lane .. 248-8*lane (descending); find the bin where the
                // count of larger-or-equal keys reaches s_need
                const int need = s_need;
                int c[8], sum = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) { c[q] = hist[255 - 8 * lane - q]; sum += c[q]; }
                int ex = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, ex, o);
                    if (lane >= o) ex += v;
                }
                ex -= sum;
                if (ex < need && need <= ex + sum) {
                    int r = ex;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (r < need && need <= r + c[q]) {
                            s_prefix = pre | ((unsigned long long)(255 - 8 * lane - q) << shift);
                            s_need = need - r;
                            s_shift = shift;
                            // every pair sharing the prefix fits, or no byte is left
                            s_done = (need - r == c[q]) || shift == 0;
                        }
                        r += c[q];
                    }
                }
            }
            __syncthreads();
        }
    } else if (tid == 0) {
        s_prefix = 0ull; s_shift = 0; s_need = 0; s_run = 0;
    }
    __syncthreads();
    // admission: key above the prefix K*, or sharing it among the first s_need such pairs in
    // token order
    const int fs = s_shift;
    const unsigned long long kstar = fs == 64 ? 0ull : s_prefix >> fs;
    const int need = s_need;
    for (int i0 = 0; i0 < ne; i0 += kSelThreads) {
        const int i = i0 + tid;
        unsigned long long kh = 0;
        if (i < ne && !all) kh = fs == 64 ? 0ull : key_of(i) >> fs;
        const bool tie = i < ne && !all && kh == kstar;
        const unsigned bal = __ballot_sync(0xffffffffu, tie);
        if (lane == 0) wsum[w] = __popc(bal);
        __syncthreads();
        int before = s_run;
        for (int q = 0; q < w; ++q) before += wsum[q];
        before += __popc(bal & ((1u << lane) - 1u));
        if (i < ne) {
            const bool a = all || kh > kstar || (tie && before < need);
            const int pid = L[i];
            bpr_adm[pid] = a ? 1 : 0;
            if (a) atomicAdd(&tiles[(pid / k) / kScanTile], 1);
        }
        __syncthreads();
        if (tid == 0) for (int q = 0; q < kSelThreads / 32; ++q) s_run += wsum[q];
        __syncthreads();
    }
    for (int q = tid; q < n_tiles; q += kSelThreads) hist2[q * E + e] = tiles[q];
}

int launch_routing(const RouteArgs& a, bool is_bf16, cudaStream_t s)
{
    const int n_tiles = ceil_div(a.T, kScanTile);
    cudaMemsetAsync(a.hist, 0, sizeof(int) * n_tiles * a.E, s);
    static bool attr_set = false;
    if (!attr_set) {
// 225 KiB: the 227 KiB opt-in minus the static histogram (E = 256 stages 207 KiB of x / Wg tiles)
#define SET(Elt, CE) cudaFuncSetAttribute(gate_topk_kernel<Elt, CE, (CE >= 8 ? kGateTT8 : CE >= 4 ? 2 : 1)>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024)
        SET(bf16, 8); SET(bf16, 4); SET(bf16, 2); SET(bf16, 1);
        SET(float, 8); SET(float, 4); SET(float, 2); SET(float, 1);
#undef SET
        cudaFuncSetAttribute(slot_scan_kernel<SCAN_SLOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(slot_scan_kernel<SCAN_BPR_LIST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(slot_scan_kernel<SCAN_BPR_SLOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    const int elt = is_bf16 ? 2 : 4;
    if (a.random) {
        launch_k(random_gate_kernel, n_tiles, kScanTile, 0, s, a.T, a.E, a.k, a.seed, a.logits, a.idx, a.w,
                 a.hist, a.t_base);
    } else if (gs_ok(a.d, a.E, elt, gs_tt(a.T, a.E))) {
        static bool gs_attr = false;
        if (!gs_attr) {
#define GSA(Elt, SS, TTT) cudaFuncSetAttribute(gate_stream_kernel<Elt, SS, TTT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)
            GSA(bf16, 8, 1); GSA(bf16, 4, 1); GSA(float, 8, 1); GSA(float, 4, 1);
            GSA(bf16, 8, 2); GSA(bf16, 4, 2); GSA(float, 8, 2); GSA(float, 4, 2);
#undef GSA
            gs_attr = true;
        }
        const int tt = gs_tt(a.T, a.E);
        const int W = gs_warps(a.E, tt), per_block = W * gs_tpw(a.E, tt), S = gs_stages(a.d, a.E, elt, tt);
        const size_t smem = gs_smem(a.d, a.E, elt, tt);
        const dim3 grid(ceil_div(a.T, per_block)), block(W * 32);
#define GS(Elt, SS, TTT) launch_k(gate_stream_kernel<Elt, SS, TTT>, grid, block, smem, s, (const Elt*)a.x, a.wg, a.T, a.d, \
                                  a.E, a.k, a.renorm, a.logits, a.idx, a.w, a.hist, n_tiles)
        if (tt == 2) {
            if (is_bf16) { if (S == 8) GS(bf16, 8, 2); else GS(bf16, 4, 2); }
            else { if (S == 8) GS(float, 8, 2); else GS(float, 4, 2); }
        } else {
            if (is_bf16) { if (S == 8) GS(bf16, 8, 1); else GS(bf16, 4, 1); }
            else { if (S == 8) GS(float, 8, 1); else GS(float, 4, 1); }
        }
#undef GS
    } else {
    // 64 tokens per block (32 measured slower even where it doubles the blocks: each block
    // stages the whole Wg, so fewer tokens per block means more Wg traffic per FMA)
    const int tb_max = kGateMaxTB;
    const GateGeom g = gate_geom(a.E, elt, gate_ce(a.E, a.T), tb_max);
    const int blocks = ceil_div(a.T, g.TB);
    const int thr = round_up(g.threads, 32);
#define GATE_ARGS a.T, a.d, a.E, a.k, a.renorm, a.logits, a.idx, a.w, a.hist, n_tiles, tb_max
#define GATE_LAUNCH(Elt)                                                                                    \
    switch (g.ce) {                                                                                         \
    case 8: launch_k(gate_topk_kernel<Elt, 8, kGateTT8>, blocks, thr, g.smem, s, (const Elt*)a.x, a.wg, GATE_ARGS); break;  \
    case 4: launch_k(gate_topk_kernel<Elt, 4, 2>, blocks, thr, g.smem, s, (const Elt*)a.x, a.wg, GATE_ARGS); break;  \
    case 2: launch_k(gate_topk_kernel<Elt, 2, 1>, blocks, thr, g.smem, s, (const Elt*)a.x, a.wg, GATE_ARGS); break;  \
    default: launch_k(gate_topk_kernel<Elt, 1, 1>, blocks, thr, g.smem, s, (const Elt*)a.x, a.wg, GATE_ARGS); break; \
    }
    if (is_bf16) { GATE_LAUNCH(bf16) } else { GATE_LAUNCH(float) }
#undef GATE_LAUNCH
#undef GATE_ARGS
    }
    const size_t smem2 = sizeof(int) * (a.E + 32 * a.E + 32 * a.E + 2 * a.E +
                                        (n_tiles * a.E <= kScanHistMax ? n_tiles * a.E : 0));
    if (!a.bpr) {
        launch_k(slot_scan_kernel<SCAN_SLOTS>, n_tiles, kScanTile, smem2, s, a.idx, a.T, a.k, a.E, a.C,
                 a.carry_in ? a.carry_n : a.n_chunks, (const int*)a.hist, n_tiles, a.slot, a.S, a.send_rows,
                 a.send_off, (const float*)nullptr, (double*)nullptr, (int*)nullptr, (int*)nullptr,
                 (const unsigned char*)nullptr, a.carry_in, a.carry_out, a.carry_chunk, a.carry_counts);
        return 2;
    }
    // Batch Prioritized Routing (R16): pairs grouped by expert + scores, per-expert priority
    // admission, then the token-major scan over the admitted pairs
    launch_k(slot_scan_kernel<SCAN_BPR_LIST>, n_tiles, kScanTile, smem2, s, a.idx, a.T, a.k, a.E, a.C,
             a.n_chunks, (const int*)a.hist, n_tiles, a.slot, a.S, a.send_rows, a.send_off,
             (const float*)a.logits, a.score, a.list, a.bpr_meta, (const unsigned char*)nullptr,
             (const int*)nullptr, (int*)nullptr, 0, (int*)nullptr);
    const int cap = std::min(a.T * a.k, (int)((kSelSmem - sizeof(int) * n_tiles) / 8));
    static bool sel_attr = false;
    if (!sel_attr) {
        cudaFuncSetAttribute(bpr_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelSmem);
        sel_attr = true;
    }
    launch_k(bpr_select_kernel, a.E, kSelThreads, 8 * (size_t)cap + sizeof(int) * n_tiles, s,
             (const int*)a.list, (const int*)a.bpr_meta, (const double*)a.score, a.E, a.k, a.C, n_tiles,
             cap, a.bpr_adm, a.hist2);
    launch_k(slot_scan_kernel<SCAN_BPR_SLOTS>, n_tiles, kScanTile, smem2, s, a.idx, a.T, a.k, a.E, a.C,
             a.n_chunks, (const int*)a.hist2, n_tiles, a.slot, a.S, a.send_rows, a.send_off,
             (const float*)nullptr, (double*)nullptr, (int*)nullptr, (int*)nullptr,
             (const unsigned char*)a.bpr_adm, (const int*)nullptr, (int*)nullptr, 0, (int*)nullptr);
    return 4;
}

}  // namespace lancet
