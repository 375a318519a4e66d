// common.cuh -- small device helpers shared by the lancet_moe kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "lancet_moe is written for sm_100a (B200) only"
#endif

namespace lancet {

// Programmatic dependent launch: kernels may be launched before their stream predecessor has
// finished (launch_k with PDL on); every kernel waits here before touching global memory the
// predecessor writes or reads.  A no-op for normally launched kernels.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }


using bf16 = __nv_bfloat16;

constexpr int kRowAlign = 128;   // expert / (expert, chunk) row blocks start on 128-row
                                 // boundaries: one tcgen05 M tile never straddles groups
constexpr int kMaxK = 8;         // top-k bound on the device side
constexpr int kMaxChunks = 64;
constexpr int kMaxExperts = 256;
constexpr int kPeerRowBits = 24; // push mode: K5 hands K6 (owner rank << 24) | row in the owner's
                                 // dX buffer (lancet_create_peer bounds rows and world)
constexpr int kScanTile = 256;   // tokens per block of the slot scan (K2); >= kMaxExperts

__host__ __device__ inline int round_up(int a, int b) { return (a + b - 1) / b * b; }
__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// 16-byte vector of elements
template <typename T> struct Vec16 { static constexpr int N = 16 / sizeof(T); };

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
    return *reinterpret_cast<const uint4*>(p);
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

// unpack / pack 16 bytes <-> float[N]
template <typename T> __device__ __forceinline__ void unpack16(uint4 v, float* f);
template <> __device__ __forceinline__ void unpack16<float>(uint4 v, float* f) {
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
}
template <> __device__ __forceinline__ void unpack16<bf16>(uint4 v, float* f) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}
template <typename T> __device__ __forceinline__ uint4 pack16(const float* f);
template <> __device__ __forceinline__ uint4 pack16<float>(const float* f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
}
template <> __device__ __forceinline__ uint4 pack16<bf16>(const float* f) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
        w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Chunk boundaries of DESIGN.md R9: n contiguous chunks, sizes differ by <= 1, larger first.
__host__ __device__ inline int chunk_start(int T, int n, int c) {
    const int base = T / n, extra = T % n;
    return c * base + (c < extra ? c : extra);
}
// Index c in [1, n) with chunk_start(c) == t, or -1.
__device__ inline int chunk_starting_at(int T, int n, int t) {
    if (t == 0 || n <= 1) return -1;
    const int base = T / n, extra = T % n;
    const int big = extra * (base + 1);
    int c;
    if (t < big) {
        if (t % (base + 1)) return -1;
        c = t / (base + 1);
    } else {
        if ((t - big) % base) return -1;
        c = extra + (t - big) / base;
    }
    return (c > 0 && c < n) ? c : -1;
}
__device__ inline int chunk_of(int T, int n, int t) {
    const int base = T / n, extra = T % n;
    const int big = extra * (base + 1);
    return t < big ? t / (base + 1) : extra + (t - big) / base;
}

// Activation of the expert FFN (R5) and its derivative, fp32.
enum ActKind { ACT_GELU_TANH = 0, ACT_RELU = 1, ACT_IDENTITY = 2 };

__device__ __forceinline__ void act_fwd_grad(int act, float a, float& h, float& g) {
    if (act == ACT_RELU) {
        h = a > 0.f ? a : 0.f;
        g = a > 0.f ? 1.f : 0.f;
    } else {
        const float c = 0.7978845608028654f;          // sqrt(2/pi)
        const float u = c * fmaf(0.044715f * a, a * a, a);
        const float th = tanhf(u);
        h = 0.5f * a * (1.f + th);
        g = 0.5f * (1.f + th) + 0.5f * a * (1.f - th * th) * c * fmaf(3.f * 0.044715f, a * a, 1.f);
    }
}

// bf16-output variant (tcgen05 epilogues): tanh via the SFU (tanh.approx.f32, ~2^-11 rel.
// error, far below the bf16 rounding of the stored result).
__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void act_fwd_grad_fast(int act, float a, float& h, float& g) {
    if (act == ACT_RELU) {
        h = a > 0.f ? a : 0.f;
        g = a > 0.f ? 1.f : 0.f;
    } else {
        const float c = 0.7978845608028654f;
        const float a2 = a * a;
        const float th = tanh_fast(c * fmaf(0.044715f * a, a2, a));
        const float hp = 0.5f * (1.f + th);
        h = a * hp;
        g = fmaf(0.5f * a * (1.f - th * th) * c, fmaf(3.f * 0.044715f, a2, 1.f), hp);
    }
}

// GELU-tanh and its derivative for two elements at a time on the packed fp32 pipe
// (FFMA2 / FMUL2), 9 paired ops + 2 SFU tanh:
//   u = a (c + c k1 a^2),  th = tanh(u),  hp = (1 + th) / 2,  h = a hp,
//   g = hp + a (1 - th^2) c (1 + 3 k1 a^2) / 2
// (the tcgen05 fc1 epilogue; same formula as act_fwd_grad_fast).
__device__ __forceinline__ void gelu_fwd_grad_fast2(float2 a, float2& h, float2& g) {
    constexpr float c = 0.7978845608028654f, k1 = 0.044715f;
    const float2 a2 = __fmul2_rn(a, a);
    const float2 t = __ffma2_rn(make_float2(c * k1, c * k1), a2, make_float2(c, c));
    const float2 u = __fmul2_rn(a, t);
    const float2 th = make_float2(tanh_fast(u.x), tanh_fast(u.y));
    const float2 hp = __ffma2_rn(make_float2(0.5f, 0.5f), th, make_float2(0.5f, 0.5f));
    h = __fmul2_rn(a, hp);
    const float2 om = __ffma2_rn(make_float2(-th.x, -th.y), th, make_float2(1.f, 1.f));
    const float2 sd = __ffma2_rn(make_float2(1.5f * c * k1, 1.5f * c * k1), a2, make_float2(0.5f * c, 0.5f * c));
    g = __ffma2_rn(__fmul2_rn(a, sd), om, hp);
}

}  // namespace lancet
