/*
 * exflow_model_oracle.c -- CPU oracle for the MoE-layer arithmetic that the
 * reference leaves out (no gate: SPEC.md:108; no FFN: SPEC.md:8). The
 * semantics follow the paper: GShard softmax gating with top-1 routing and
 * experts that are plain FFNs.
 *
 * TEST INFRASTRUCTURE ONLY (see exflow_oracle.h).
 *
 * Arithmetic contract shared with the sm_100a gate kernel
 * (paper_2401_08383_b200/csrc/gate_dispatch.cu):
 *   logits[e] = dot(x, wg[e]) summed in fp32 in a FIXED order: 32 lane
 *   partials, lane l accumulating elements k = c*256 + l*8 + i for
 *   c = 0..d/256-1, i = 0..7 (c-major, i-minor) with fused multiply-add, then
 *   a butterfly over lanes (xor 16, 8, 4, 2, 1). bf16 x bf16 products are
 *   exact in fp32, so the only rounding is in the additions, which this code
 *   performs in the identical order => bit-identical logits and routing.
 *   top-1 = argmax with the lowest index on ties (the tie rule of
 *   most_affiliated, proj/src/trace.cpp:255-258); prob = 1/sum_e exp(l_e - l_max).
 * Expert FFN (tolerance contract, not bitwise):
 *   h = bf16(gelu_erf(x W1^T + b1)); y = h W2^T + b2; out = bf16(x + prob*y)
 *   computed here in fp64 accumulation.
 */
#include "exflow_oracle.h"

#include <math.h>
#include <string.h>

float orc_bf16_to_f32(uint16_t v) {
    uint32_t u = (uint32_t)v << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

uint16_t orc_f32_to_bf16(float f) { /* round-to-nearest-even, NaN preserved */
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

void orc_gate_logits(const uint16_t* x, const uint16_t* wg, int32_t d, int32_t E,
                     float* logits) {
    const int32_t chunks = d / 256;
    for (int32_t e = 0; e < E; ++e) {
        const uint16_t* w = wg + (int64_t)e * d;
        float lane[32];
        for (int32_t l = 0; l < 32; ++l) {
            float acc = 0.0f;
            for (int32_t c = 0; c < chunks; ++c)
                for (int32_t i = 0; i < 8; ++i) {
                    const int32_t k = c * 256 + l * 8 + i;
                    acc = fmaf(orc_bf16_to_f32(x[k]), orc_bf16_to_f32(w[k]), acc);
                }
            lane[l] = acc;
        }
        for (int32_t off = 16; off >= 1; off >>= 1) {
            float nxt[32];
            for (int32_t l = 0; l < 32; ++l) nxt[l] = lane[l] + lane[l ^ off];
            memcpy(lane, nxt, sizeof(lane));
        }
        logits[e] = lane[0];
    }
}

static double gelu_erf(double v) { return 0.5 * v * (1.0 + erf(v * 0.70710678118654752440)); }

void orc_gate_logits_f32(const float* x, const float* wg, int32_t d, int32_t E, float* logits) {
    /* same order as orc_gate_logits: lane l accumulates k = c*256 + l*8 + i
     * (c-major, i-minor) with fmaf, then the xor butterfly 16..1 */
    const int32_t chunks = d / 256;
    for (int32_t e = 0; e < E; ++e) {
        const float* w = wg + (int64_t)e * d;
        float lane[32];
        for (int32_t l = 0; l < 32; ++l) {
            float acc = 0.0f;
            for (int32_t c = 0; c < chunks; ++c)
                for (int32_t i = 0; i < 8; ++i) {
                    const int32_t k = c * 256 + l * 8 + i;
                    acc = fmaf(x[k], w[k], acc);
                }
            lane[l] = acc;
        }
        for (int32_t off = 16; off >= 1; off >>= 1) {
            float nxt[32];
            for (int32_t l = 0; l < 32; ++l) nxt[l] = lane[l] + lane[l ^ off];
            memcpy(lane, nxt, sizeof(lane));
        }
        logits[e] = lane[0];
    }
}

void orc_expert_ffn_f32(const float* x, const float* w1, const float* b1, const float* w2,
                        const float* b2, int32_t d, int32_t dff, float prob, double* out) {
    static double h[65536];
    for (int32_t m = 0; m < dff; ++m) {
        const float* w = w1 + (int64_t)m * d;
        double acc = 0.0;
        for (int32_t k = 0; k < d; ++k) acc += (double)x[k] * (double)w[k];
        h[m] = gelu_erf(acc + (double)b1[m]);
    }
    for (int32_t n = 0; n < d; ++n) {
        const float* w = w2 + (int64_t)n * dff;
        double acc = 0.0;
        for (int32_t m = 0; m < dff; ++m) acc += h[m] * (double)w[m];
        out[n] = (double)x[n] + (double)prob * (acc + (double)b2[n]);
    }
}

int orc_gate_top1(const float* logits, int32_t E, float* prob) {
    int32_t best = 0;
    for (int32_t e = 1; e < E; ++e)
        if (logits[e] > logits[best]) best = e;
    float s = 0.0f;
    for (int32_t e = 0; e < E; ++e) s += expf(logits[e] - logits[best]);
    if (prob) *prob = 1.0f / s;
    return best;
}


void orc_expert_ffn(const uint16_t* x, const uint16_t* w1, const uint16_t* b1,
                    const uint16_t* w2, const uint16_t* b2, int32_t d, int32_t dff,
                    float prob, uint16_t* out, float* out_f32) {
    float xf[8192];
    float hf[32768];
    for (int32_t k = 0; k < d; ++k) xf[k] = orc_bf16_to_f32(x[k]);
    for (int32_t m = 0; m < dff; ++m) {
        const uint16_t* w = w1 + (int64_t)m * d;
        double acc = 0.0;
        for (int32_t k = 0; k < d; ++k) acc += (double)xf[k] * orc_bf16_to_f32(w[k]);
        acc += orc_bf16_to_f32(b1[m]);
        hf[m] = orc_bf16_to_f32(orc_f32_to_bf16((float)gelu_erf(acc)));
    }
    for (int32_t n = 0; n < d; ++n) {
        const uint16_t* w = w2 + (int64_t)n * dff;
        double acc = 0.0;
        for (int32_t m = 0; m < dff; ++m) acc += (double)hf[m] * orc_bf16_to_f32(w[m]);
        acc += orc_bf16_to_f32(b2[n]);
        const float o = (float)((double)xf[n] + (double)prob * acc);
        if (out) out[n] = orc_f32_to_bf16(o);
        if (out_f32) out_f32[n] = o;
    }
}
