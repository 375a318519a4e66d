/*
 * oracle/gate_logits.c -- TEST INFRASTRUCTURE, not product code.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this file's shared object.  It shares no code with paper_2404_19429_b200/.
 *
 * The gate score of the paper: "assigning a gating score for each expert using a trainable
 * linear layer" (§2.1 "Routing algorithms").  The paper does not fix the
 * arithmetic; reading R1 fixes it so that routing is reproducible bit for bit:
 *
 *     logit[t][e] = fp32 chain   acc = 0;  for i = 0..d-1:  acc = fmaf(x[t][i], Wg[i][e], acc)
 *
 * i.e. one IEEE-754 fused multiply-add (single rounding) per step, in increasing i, with no
 * reassociation.  This file must be compiled with -ffp-contract=off and without -ffast-math;
 * fmaf() is the C99 correctly-rounded fused multiply-add.
 *
 * x  : [T][d] float32 (bf16-valued in bf16 mode), row-major
 * wg : [d][E] float32, row-major
 * out: [T][E] float32, row-major
 */
#include <math.h>
#include <stdint.h>

void oracle_gate_logits(const float *x, const float *wg, int64_t T, int32_t d, int32_t E,
                        float *logits)
{
    int64_t t;
#pragma omp parallel for schedule(static)
    for (t = 0; t < T; ++t) {
        for (int32_t e = 0; e < E; ++e) {
            float acc = 0.0f;
            for (int32_t i = 0; i < d; ++i)
                acc = fmaf(x[t * (int64_t)d + i], wg[(int64_t)i * E + e], acc);
            logits[t * (int64_t)E + e] = acc;
        }
    }
}
