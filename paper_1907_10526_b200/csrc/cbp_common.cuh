// cbp_common.cuh -- device-side geometry record, per-geometry tables (row a1)
// and the Eq. 14 weight evaluation shared by the FP and BP kernels.
//
// Citations: P:n = PAPER.md line, ledger #k = DESIGN.md section 3 reading.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cbp {

// Geometry as the kernels see it (FP64 scalars + derived constants).
struct GeomDev {
    int n, n_views, n_det;
    double h, pitch, tau, sid, sdd;
    double c0;  // (n - 1) / 2: pixel-centre offset (ledger #13)
    double cs;  // (n_det - 1) / 2: bin-centre offset (ledger #10)
};

// Row a1: view-independent per-bin table and per-view rotation table, FP64,
// built once per (geometry, device) by cbp_tables_kernel.
struct Tables {
    const double2* view_cs;  // [n_views]  (cos theta_v, sin theta_v)
    const double2* bin_d;    // [n_det]    (s_j, 1 / L_j),  L_j = sqrt(D_ps^2 + s_j^2)
    const float4* bin_f;     // [n_det]    (sin phi_j, cos phi_j, g_j, 0)
};

// ---------------------------------------------------------------------------
// Eq. 14 in a form that is stable in FP32.
//
// M_{A,B,C}(x) = box_A * box_B * box_C (x) with A = max|zeta|, B = tau',
// C = min|zeta|, is evaluated as nested antiderivative differences:
//   R_C(z) = int_{-inf}^{z} H_C,  H_C the CDF of the centred box of width C
//          = max(z', 0) + (C/2) sat(z'/C + 1)^2,        z' = z - C/2
//   G(y)   = [R_C(y + B/2) - R_C(y - B/2)] / B           (CDF of box_B * box_C)
//   M(x)   = [G(x + A/2) - G(x - A/2)] / A
// which is algebraically Delta_A Delta_B Delta_C (x + sigma)_+^2 / (2! A B C)
// (Eq. 14) but never divides by the possibly vanishing C: C = 0 gives
// invC = +inf, sat() maps +-inf to {0, 1} and NaN to +0, and (C/2) t^2 = 0,
// i.e. the delta direction is eliminated exactly as P:347 prescribes.
//
// cnsf_num returns A B M(x) = R(z11) - R(z12) - R(z21) + R(z22); the caller
// multiplies by h^2 / A (per bin) and 1 / B.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float sat_fma(float a, float b, float c)
{
    float d;
    asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

__device__ __forceinline__ float rcp_approx(float x)
{
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// hAmC = (A - C)/2, hApC = (A + C)/2, invC = 1/C, hC = C/2
__device__ __forceinline__ float cnsf_num(float x, float B, float hAmC, float hApC, float invC,
                                          float hC)
{
    const float hb = 0.5f * B;
    const float y1 = x + hAmC;  // (x + A/2) - C/2
    const float y2 = x - hApC;  // (x - A/2) - C/2
    const float z11 = y1 + hb, z12 = y1 - hb, z21 = y2 + hb, z22 = y2 - hb;
    const float t11 = sat_fma(z11, invC, 1.0f);
    const float t12 = sat_fma(z12, invC, 1.0f);
    const float t21 = sat_fma(z21, invC, 1.0f);
    const float t22 = sat_fma(z22, invC, 1.0f);
    const float m = (fmaxf(z11, 0.0f) - fmaxf(z12, 0.0f)) - (fmaxf(z21, 0.0f) - fmaxf(z22, 0.0f));
    const float T = fmaf(t11, t11, -t12 * t12) - fmaf(t21, t21, -t22 * t22);
    return fmaf(hC, T, m);
}

}  // namespace cbp
