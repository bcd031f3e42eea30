// cbp_common.cuh -- device-side geometry record, per-geometry tables (row a1)
// and the Eq. 14 weight evaluation shared by the FP and BP kernels.
//
// Citations: P:n = PAPER.md line, ledger #k = DESIGN.md section 3 reading.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// Device-side index checks for the debug build (libcbp_debug.so, built with
// -DCBP_DEBUG_CHECKS): print the violated condition; no-ops otherwise.
#ifdef CBP_DEBUG_CHECKS
#include <cstdio>
#define CBP_CHECK(cond, ...)                                              \
    do {                                                                  \
        if (!(cond)) {                                                    \
            printf("CBP_CHECK %s:%d %s | ", __FILE__, __LINE__, #cond);   \
            printf(__VA_ARGS__);                                          \
        }                                                                 \
    } while (0)
#else
#define CBP_CHECK(cond, ...) \
    do {                     \
    } while (0)
#endif

namespace cbp {

// Geometry as the kernels see it (FP64 scalars + derived constants).
struct GeomDev {
    int n, n_views, n_det;
    int parallel;  // kind == CBP_PARALLEL (row f3): rays along -u, s' = s_j - k.e, tau' = tau
    int arc;       // kind == CBP_FAN_ARC (row f3): bin j is the ray at angle (j - cs) pitch / sdd
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
// Eq. 14 in a form that is stable in FP32 and cheap on the FP32 pipe
// (pinned on CPU by tests/test_weight_form.py).
//
// M_{A,B,C}(x) = box_A * box_B * box_C (x) with A = max|zeta|, B = tau',
// C = min|zeta| (Eq. 12-14) is evaluated as nested antiderivative differences
// of R_C(z) = int_{-inf}^z H_C (H_C the CDF of the centred box of width C):
//   A B M(x) = sum_{a = +-A/2, b = +-B/2} +- R_C(x + a + b)
// With z' = z - C/2, R_C = max(z', 0) + (C/2) sat(z'/C + 1)^2, and since the
// four shifted knots pair up as z11 - z12 = z21 - z22 = B:
//   sum +- max(z', 0) = clamp(z11, 0, B) - clamp(z21, 0, B)
//                     = max(0, min(z11, A, B, A + B - z11))   (a trapezoid in z11)
//   sum +- (C/2) t^2  = (C/2) (t11^2 - t12^2 - t21^2 + t22^2)
// where z11 = x + (A - C)/2 + B/2, z21 = z11 - A, t1. = sat(z11/C + {1, w1}),
// t2. = sat(z21/C + {1, w1}), w1 = 1 - B/C.  Never divides by a vanishing C:
// C = 0 gives 1/C = +inf, sat() maps +-inf to {0, 1} and NaN to +0, and
// (C/2) T = 0 -- the delta direction is eliminated exactly as P:347 says.
// W = h^2 M = (h^2 / A) * num / B.
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

__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }

// 3-input minimum (FMNMX3 on sm_100a)
__device__ __forceinline__ float fmin3(float a, float b, float c)
{
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// Two weights at once (packed FFMA2 / FADD2 / FMUL2 on sm_100a): lanes share
// the per-bin constants A, invC and hC = C/2.  Returns num = A B M for both.
// The trapezoid part clamp(z11,0,B) - clamp(z21,0,B) is written as
// max(0, min(z11, min(A, B), B - z21)), one 3-input min and two 2-input ops.
__device__ __forceinline__ float2 cnsf_num2(float2 z11, float2 z21, float2 B, float2 w1, float A,
                                            float invC, float hC)
{
    const float2 t11 = make_float2(sat_fma(z11.x, invC, 1.0f), sat_fma(z11.y, invC, 1.0f));
    const float2 t12 = make_float2(sat_fma(z11.x, invC, w1.x), sat_fma(z11.y, invC, w1.y));
    const float2 t21 = make_float2(sat_fma(z21.x, invC, 1.0f), sat_fma(z21.y, invC, 1.0f));
    const float2 t22 = make_float2(sat_fma(z21.x, invC, w1.x), sat_fma(z21.y, invC, w1.y));
    float2 T = __fmul2_rn(t11, t11);
    T = __ffma2_rn(neg2(t12), t12, T);
    T = __ffma2_rn(neg2(t21), t21, T);
    T = __ffma2_rn(t22, t22, T);
    const float2 r = __fadd2_rn(B, neg2(z21));  // A + B - z11
    const float2 M2 = make_float2(fmaxf(fmin3(z11.x, fminf(A, B.x), r.x), 0.0f),
                                  fmaxf(fmin3(z11.y, fminf(A, B.y), r.y), 0.0f));
    return __ffma2_rn(make_float2(hC, hC), T, M2);
}

// ---------------------------------------------------------------------------
// Eq. 14 for narrow bins (the precise mode).  The FP32 form
// above carries s' and the knot z11 = s' + (A - C)/2 + tau'/2 as FP32 values
// of size ~A, so their absolute rounding (~ulp(h), several ulp after the
// kernels' affine steps) shifts a ramp of width tau' + C by a relative
// ~1e-7 h / (tau' + C): past the parity bar once tau' ~ 0.01 h on views where
// C -> 0.  Here s' and A come in FP64 and the four knot arguments
//   k1 = z11, k2 = z11 - b, k3 = z11 - A, k4 = z11 - A - b
// are formed in FP64 before the single rounding to FP32, so each is exact to
// ~ulp of its own (small, near its knot) value.  The two widths besides A are
// nested smallest-innermost, b = max(tau', C), c = min(tau', C) (the spline
// box_A * box_tau' * box_C is symmetric in its widths): with c
// innermost the (c/2) T correction's FP32 rounding is ~1e-7 c / b <= 1e-7 of
// the plateau b (tau' innermost with C ~ h would give ~1e-7 h / tau').
// Returns num / b = A M (W = h^2 / A times it), pinned on CPU by
// tests/test_weight_form.py (<= 2e-7 of the peak for tau' / A down to 1e-4).
// tau' <= 0 only occurs in the FP's zero border: b, c are kept finite there.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float cnsf_prec(double s, double A, float tau, float Cz)
{
    const float b = fmaxf(fmaxf(tau, Cz), 1e-30f), c = fmaxf(fminf(tau, Cz), 0.0f);
    const double D = fma(0.5, A + (double)(b - c), s);  // z11 = s' + (A + b - c) / 2
    const double D3 = D - A;
    const float k1 = (float)D, k2 = (float)(D - (double)b), k3 = (float)D3, k4 = (float)(D3 - (double)b);
    const float ic = rcp_approx(c);  // c = 0: +inf, sat() eliminates the direction
    const float t11 = sat_fma(k1, ic, 1.0f), t12 = sat_fma(k2, ic, 1.0f);
    const float t21 = sat_fma(k3, ic, 1.0f), t22 = sat_fma(k4, ic, 1.0f);
    float T = t11 * t11;
    T = fmaf(-t12, t12, T);
    T = fmaf(-t21, t21, T);
    T = fmaf(t22, t22, T);
    const float trap = fmaxf(fmin3(k1, fminf((float)A, b), -k4), 0.0f);
    return fmaf(0.5f * c, T, trap) * rcp_approx(b);
}

// the multimem reduction (accumulate mode CBP_ACC_MULTIMEM): `mc` is a
// multicast address (an NVLink/NVSwitch multicast object bound to one buffer
// on every rank); the add is performed in the switch on every rank's copy
__device__ __forceinline__ void mc_red_add(float* mc, float v)
{
    asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}
__device__ __forceinline__ void mc_red_add4(float4* mc, float4 v)
{
    asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-stream-serialization attribute may start while its stream
// predecessor finishes; it runs griddep_wait() before touching anything the
// predecessor produced (or memory the predecessor's stream-ordered frees may
// hand out).  griddep_launch_dependents() lets the NEXT kernel launch once
// every CTA of this grid has called it.  Both are no-ops without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__device__ __forceinline__ float2 rcp2(float2 b) { return make_float2(rcp_approx(b.x), rcp_approx(b.y)); }

}  // namespace cbp
