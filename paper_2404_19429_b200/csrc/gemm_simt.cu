// gemm_simt.cu -- G0: grouped SIMT GEMM for the fp32 mode (tcgen05 has no fp32-exact kind,
// DESIGN.md R14) and as a cross-check of the tcgen05 path (LANCET_FLAG_SIMT_GEMM).
//
// Expert computation: "Each expert processes the C received tokens" -- an FFN per
// expert, so the GEMMs are grouped by expert (or (expert, chunk)) with group sizes
// that live on the device (irregular partitioning).  M-grouped: rows of group g are
// [off_g, off_g + rows_g) (computed up to the 128-row pad; pad rows are zero so the outputs
// there are act(0)).  K-grouped (weight gradients): group g reduces over token rows
// [off_g, off_g + round_up(rows_g, 128)).  The K-grouped sum is accumulated in two levels
// (fresh 64-term partials added to the running sum) for the fp32 tolerance.
#include "common.cuh"
#include "kernels.h"

namespace lancet {

constexpr int SBM = 64, SBN = 64, SBK = 16;

template <typename Elt, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(256) simt_gemm_kernel(GemmArgs p)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    __shared__ float As[SBK][SBM + 4];
    __shared__ float Bs[SBK][SBN + 4];
    const int g = blockIdx.z;
    const int m0 = blockIdx.y * SBM, n0 = blockIdx.x * SBN;
    const int rows_g = p.grp_rows[g];
    const long row0 = p.grp_off[g];
    int Mg, Kg;
    if (p.mode == GEMM_M_GROUPED) {
        Mg = round_up(rows_g, kRowAlign);
        Kg = p.K;
    } else {
        Mg = p.M;
        Kg = round_up(rows_g, kRowAlign);
    }
    if (m0 >= Mg) return;
    const Elt* A = reinterpret_cast<const Elt*>(p.A);
    const Elt* B = reinterpret_cast<const Elt*>(p.B) + (long)((g / p.gpw) % p.n_weights) * p.b_group_stride;
    const long krow0 = p.mode == GEMM_K_GROUPED ? row0 : 0;
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;

    float acc[4][4], part[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = part[i][j] = 0.f;

    int kt = 0;
    for (int k0 = 0; k0 < Kg; k0 += SBK, ++kt) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int id = tid + q * 256;
            int mm, kk;
            if (A_MN) { kk = id / SBM; mm = id % SBM; } else { mm = id / SBK; kk = id % SBK; }
            const int m = m0 + mm, kx = k0 + kk;
            float v = 0.f;
            if (m < Mg && kx < Kg) {
                if (A_MN) v = to_f(A[(krow0 + kx) * p.lda + m]);
                else v = to_f(A[(row0 + m) * p.lda + kx]);
            }
            As[kk][mm] = v;
            int nn;
            if (B_MN) { kk = id / SBN; nn = id % SBN; } else { nn = id / SBK; kk = id % SBK; }
            const int n = n0 + nn, kb = k0 + kk;
            float u = 0.f;
            if (n < p.N && kb < Kg) {
                if (B_MN) u = to_f(B[(krow0 + kb) * p.ldb + n]);
                else u = to_f(B[(long)n * p.ldb + kb]);
            }
            Bs[kk][nn] = u;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < SBK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) part[i][j] = fmaf(a[i], b[j], part[i][j]);
        }
        __syncthreads();
        if ((kt & 3) == 3) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) { acc[i][j] += part[i][j]; part[i][j] = 0.f; }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += part[i][j];

#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= Mg) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= p.N) continue;
            const float v = acc[i][j];
            if (p.epi == EPI_F32) {
                float* C = reinterpret_cast<float*>(p.C) + (long)g * p.c_group_stride;
                const long o = (long)m * p.ldc + n;
                C[o] = p.accumulate ? C[o] + v : v;
            } else {
                const long o = (row0 + m) * p.ldc + n;
                Elt* C = reinterpret_cast<Elt*>(p.C);
                if (p.epi == EPI_STORE) {
                    C[o] = from_f<Elt>(v);
                } else if (p.epi == EPI_ACT) {
                    float h, gr;
                    act_fwd_grad(p.act, v, h, gr);
                    C[o] = from_f<Elt>(h);
                    reinterpret_cast<Elt*>(p.C2)[o] = from_f<Elt>(gr);
                } else {  // EPI_DACT
                    C[o] = from_f<Elt>(v * to_f(reinterpret_cast<const Elt*>(p.aux)[o]));
                }
            }
        }
    }
}

template <typename Elt>
static void launch_t(const GemmArgs& a, cudaStream_t s)
{
    const int mrows = a.mode == GEMM_M_GROUPED ? a.max_rows : a.M;
    dim3 grid(ceil_div(a.N, SBN), ceil_div(mrows, SBM), a.n_groups);
    if (!a.a_mn && !a.b_mn) launch_k(simt_gemm_kernel<Elt, false, false>, grid, 256, 0, s, a);
    else if (!a.a_mn && a.b_mn) launch_k(simt_gemm_kernel<Elt, false, true>, grid, 256, 0, s, a);
    else if (a.a_mn && a.b_mn) launch_k(simt_gemm_kernel<Elt, true, true>, grid, 256, 0, s, a);
    else launch_k(simt_gemm_kernel<Elt, true, false>, grid, 256, 0, s, a);
}

int launch_gemm_simt(const GemmArgs& a, bool is_bf16, cudaStream_t s)
{
    if (a.n_groups <= 0) return 0;
    if (is_bf16) launch_t<bf16>(a, s);
    else launch_t<float>(a, s);
    return 1;
}

}  // namespace lancet
