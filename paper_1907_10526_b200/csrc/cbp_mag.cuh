// cbp_mag.cuh -- row f3: the magnified-footprint weight model
// (cbp_geometry_t.model = CBP_MODEL_MAG), FP and BP kernels.
//
// The pixel-driven reading of the method (BASELINE.json's prose, SURVEY
// §8(f) f3; the oracle's weight_mag_f): the detector coordinate of a point
// x is P(x) (Eq. 4; on the arc the angle times D_ps; parallel
// beam x.e).  Linearising P at the pixel centre k maps the pixel's edge
// vectors xi1 = (h, 0), xi2 = (0, h) to detector lengths
// zeta_i = h dP/dx_i(k), so the pixel's projection is the 2-direction box
// spline M_{|zeta1|,|zeta2|} around P(k) (Eq. 12's form), which
// the detector cell blurs with M_tau (unit mass, ledger #3):
//   W(v, j, k) = h^2 m(k) M_{|zeta1|, |zeta2|, tau}(s_j - P(k))
// with m(k) the pixel's detector-integrated chord length per unit area at
// its centre: (D_ps^2 + P^2) / (D_ps |k - p|) on the flat detector, D_ps / |k - p|
// on the arc, 1 in parallel beam.  Unlike the paper's CNSF weight (per bin
// ray, effective blur tau' in the object plane, Eq. 13) every (view, pixel)
// pair has ONE footprint that all its bins share, so the footprint is
// computed once per (view, pixel) -- FP64, the precision-critical P(k) and
// s_j - P(k) included -- and the bins evaluate only the nested FP32 form of
// Eq. 14 at x = s_j - P(k).
//
// FP: one thread per (slice, view, bin) gathers over the image lines the
// bin's footprint band crosses (no atomics, fixed order); BP: one thread per
// (slice, pixel) gathers over views and the bins of its footprint.  Both call
// mag_footprint / mag_weight for a (view, bin, pixel): the same arithmetic.
#pragma once

#include "cbp_common.cuh"

namespace cbp {

constexpr int MAG_FP_BLOCK = 128;
constexpr int MAG_BP_BLOCK = 128;

struct MagFootprint {
    double P;      // detector coordinate of the pixel centre, P(k) (FP64: s_j - P(k) cancels)
    float sigma;   // support half-width (A + B + C) / 2
    float A, C;    // max / min |zeta| (C = 0: eliminated)
    float wscale;  // h^2 m(k) / (A B)
};

// lateral offset k.e and depth D_po - k.u of the pixel centre k in view (cu, su)
__device__ __forceinline__ void mag_frame(const GeomDev& g, double cu, double su, double kx, double ky,
                                          double& lat, double& dep)
{
    lat = __fma_rn(ky, cu, -(kx * su));
    dep = g.sid - __fma_rn(kx, cu, ky * su);
}

// P(k) in FP64 (the flat detector's 1 / depth from the FP32 reciprocal and
// one Newton step, relative error ~1e-14); the footprint's shape (zeta, the
// magnification m) in FP32.  Ledger #7: |zeta| < 1e-6 h is eliminated.
__device__ __forceinline__ MagFootprint mag_footprint(const GeomDev& g, double cu, double su, double kx,
                                                      double ky)
{
    double lat, dep;
    mag_frame(g, cu, su, kx, ky, lat, dep);
    const float cuf = (float)cu, suf = (float)su, sdd = (float)g.sdd;
    const float latf = (float)lat, depf = (float)dep;
    double P;
    float gx, gy, m;
    if (g.parallel) {
        P = lat;
        gx = -suf;
        gy = cuf;
        m = 1.0f;
    } else {
        float f;
        const float r2 = __fmaf_rn(depf, depf, latf * latf);
        if (g.arc) {
            P = g.sdd * atan2(lat, dep);
            f = __fdiv_rn(sdd, r2);
            m = sdd * rsqrtf(r2);
        } else {
            const float invf = __frcp_rn(depf);
            double r = (double)invf;
            r = __fma_rn(r, __fma_rn(-dep, r, 1.0), r);
            P = g.sdd * lat * r;
            f = sdd * invf * invf;
            const float Pf = (float)P;
            m = __fdiv_rn(__fmaf_rn(Pf, Pf, sdd * sdd), sdd * sqrtf(r2));
        }
        // grad P = f (dep e + lat u)
        gx = f * __fmaf_rn(depf, -suf, latf * cuf);
        gy = f * __fmaf_rn(depf, cuf, latf * suf);
    }
    const float h = (float)g.h, tau = (float)g.tau;
    float a1 = fabsf(h * gx), a2 = fabsf(h * gy);
    const float eps = 1e-6f * h;
    if (a1 < eps) a1 = 0.0f;
    if (a2 < eps) a2 = 0.0f;
    MagFootprint fp;
    fp.P = P;
    fp.A = fmaxf(a1, a2);
    fp.C = fminf(a1, a2);
    fp.sigma = 0.5f * (fp.A + tau + fp.C);
    fp.wscale = __fdiv_rn(h * h * m, fp.A * tau);
    return fp;
}

// W at detector coordinate s (exactly 0 outside the open support, ledger #15):
// the scalar form of cnsf_num2 with B = tau
__device__ __forceinline__ float mag_weight(const MagFootprint& fp, double s, float B)
{
    const float x = (float)(s - fp.P);
    if (!(fabsf(x) < fp.sigma)) return 0.0f;
    const float A = fp.A, C = fp.C;
    const float invC = __frcp_rn(C);  // C = 0 -> +inf: sat() eliminates the direction
    const float w1 = __fmaf_rn(-B, invC, 1.0f);
    const float z11 = x + 0.5f * (A - C) + 0.5f * B;
    const float z21 = z11 - A;
    const float t11 = sat_fma(z11, invC, 1.0f), t12 = sat_fma(z11, invC, w1);
    const float t21 = sat_fma(z21, invC, 1.0f), t22 = sat_fma(z21, invC, w1);
    float T = t11 * t11;
    T = __fmaf_rn(-t12, t12, T);
    T = __fmaf_rn(-t21, t21, T);
    T = __fmaf_rn(t22, t22, T);
    const float trap = fmaxf(fmin3(z11, fminf(A, B), B - z21), 0.0f);
    return fp.wscale * __fmaf_rn(0.5f * C, T, trap);
}

__device__ __forceinline__ double mag_bin_s(const GeomDev& g, int j) { return ((double)j - g.cs) * g.pitch; }

struct MagParams {
    GeomDev g;
    const double2* view_cs;
    const float* image;    // FP: [batch][n][n]
    float* sino;           // FP: [batch][view_count][n_det] out
    const float* sino_in;  // BP: [batch][view_count][n_det]
    float* image_out;      // BP: [batch][n][n]
    int view_begin, view_count, batch, accumulate;
    double sigma_max;  // upper bound of every pixel's support half-width
};

// The pixels k with P(k) > s' are those with G(k) = alpha lat(k) - beta dep(k) > 0
// (every pixel is in front of the source, dep > 0): flat (alpha, beta) = (D_ps, s');
// arc (cos g, sin g), g = s'/D_ps, and beyond +-90 degrees every pixel or none;
// parallel (1, s') with dep = 1.  G is affine in (col, row).
struct MagEdge {
    double G00, Gr, Gc;  // G = G00 + Gr row + Gc col
};

__device__ __forceinline__ MagEdge mag_edge(const GeomDev& g, double cu, double su, double sp)
{
    double alpha, beta;
    if (g.parallel) {
        alpha = 1.0;
        beta = sp;
    } else if (g.arc) {
        const double gam = sp / g.sdd;
        if (gam <= -1.5707963267948966) {
            alpha = 0.0;
            beta = -1.0;  // G = dep > 0: every pixel is beyond the lower edge
        } else if (gam >= 1.5707963267948966) {
            alpha = 0.0;
            beta = 1.0;  // G = -dep < 0: no pixel is beyond the upper edge
        } else {
            sincos(gam, &beta, &alpha);
        }
    } else {
        alpha = g.sdd;
        beta = sp;
    }
    // k = ((col - c0) h, (c0 - row) h): lat = -kx su + ky cu, dep = sid - kx cu - ky su
    const double hc = g.h, c0h = g.c0 * g.h;
    const double lat00 = c0h * su + c0h * cu, dlat_c = -hc * su, dlat_r = -hc * cu;
    double dep00 = g.sid + c0h * cu - c0h * su, ddep_c = -hc * cu, ddep_r = hc * su;
    if (g.parallel) {
        dep00 = 1.0;
        ddep_c = 0.0;
        ddep_r = 0.0;
    }
    MagEdge E;
    E.G00 = alpha * lat00 - beta * dep00;
    E.Gc = alpha * dlat_c - beta * ddep_c;
    E.Gr = alpha * dlat_r - beta * ddep_r;
    return E;
}

// restrict [lo, hi] (pixel index units along the line) to G0 + G1 i > 0,
// widened by 1e-3 pixel against rounding (the exact test decides)
__device__ __forceinline__ void mag_halfline(double G0, double G1, double& lo, double& hi)
{
    if (G1 > 0.0)
        lo = fmax(lo, -G0 / G1 - 1e-3);
    else if (G1 < 0.0)
        hi = fmin(hi, -G0 / G1 + 1e-3);
    else if (!(G0 > -1e-12))
        hi = -1e30;
}

// FP: y[b][v][j] = sum_k c[b][k] W(v, j, k).  The pixels whose footprint can
// reach bin j have P(k) in (s_j - sigma_max, s_j + sigma_max): on each image
// line (rows when the bin's ray is within 45 degrees of the y axis, else
// columns) that is an index interval, from the two affine edge functions of
// mag_edge; the exact open-support test of mag_weight decides.
__global__ void __launch_bounds__(MAG_FP_BLOCK) cbp_mag_fp_kernel(MagParams p)
{
    const GeomDev& g = p.g;
    const int j = blockIdx.x * MAG_FP_BLOCK + threadIdx.x;
    const int vl = blockIdx.y, b = blockIdx.z;
    if (j >= g.n_det) return;
    const double2 cs = p.view_cs[p.view_begin + vl];
    const double cu = cs.x, su = cs.y;
    const double s = mag_bin_s(g, j);
    const float B = (float)g.tau;
    const MagEdge lo_e = mag_edge(g, cu, su, s - p.sigma_max), hi_e = mag_edge(g, cu, su, s + p.sigma_max);
    // direction of the bin-centre ray
    double dx, dy;
    if (g.parallel) {
        dx = -cu;
        dy = -su;
    } else if (g.arc) {
        double sg, cg;
        sincos(s / g.sdd, &sg, &cg);
        dx = -cg * cu - sg * su;
        dy = -cg * su + sg * cu;
    } else {
        dx = -g.sdd * cu - s * su;
        dy = -g.sdd * su + s * cu;
    }
    const bool rows = fabs(dy) >= fabs(dx);
    const int n = g.n;
    const float* img = p.image + (size_t)b * n * n;
    float acc = 0.0f;
    for (int l = 0; l < n; ++l) {
        double lo = -0.5, hi = (double)n - 0.5;
        // P > s - sigma_max: G_lo > 0;  P < s + sigma_max: -G_hi > 0
        if (rows) {
            mag_halfline(lo_e.G00 + lo_e.Gr * l, lo_e.Gc, lo, hi);
            mag_halfline(-(hi_e.G00 + hi_e.Gr * l), -hi_e.Gc, lo, hi);
        } else {
            mag_halfline(lo_e.G00 + lo_e.Gc * l, lo_e.Gr, lo, hi);
            mag_halfline(-(hi_e.G00 + hi_e.Gc * l), -hi_e.Gr, lo, hi);
        }
        if (!(hi >= lo)) continue;
        const int i0 = max(0, (int)ceil(lo)), i1 = min(n - 1, (int)floor(hi));
        for (int i = i0; i <= i1; ++i) {
            const int row = rows ? l : i, col = rows ? i : l;
            const double kx = ((double)col - g.c0) * g.h, ky = (g.c0 - (double)row) * g.h;
            const MagFootprint fp = mag_footprint(g, cu, su, kx, ky);
            const float wgt = mag_weight(fp, s, B);
            if (wgt != 0.0f) acc = __fmaf_rn(__ldg(img + (size_t)row * n + col), wgt, acc);
        }
    }
    p.sino[((size_t)b * p.view_count + vl) * g.n_det + j] = acc;
}

// BP: c[b][k] = sum_{v, j} y[b][v][j] W(v, j, k) over the bins of k's footprint
__global__ void __launch_bounds__(MAG_BP_BLOCK) cbp_mag_bp_kernel(MagParams p)
{
    const GeomDev& g = p.g;
    const int n = g.n;
    const int k = blockIdx.x * MAG_BP_BLOCK + threadIdx.x;
    const int b = blockIdx.y;
    if (k >= n * n) return;
    const int row = k / n, col = k - row * n;
    const double kx = ((double)col - g.c0) * g.h, ky = (g.c0 - (double)row) * g.h;
    const float B = (float)g.tau;
    const double inv_pitch = 1.0 / g.pitch;
    const float* y = p.sino_in + (size_t)b * p.view_count * g.n_det;
    float acc = 0.0f;
    for (int vl = 0; vl < p.view_count; ++vl) {
        const double2 cs = p.view_cs[p.view_begin + vl];
        const MagFootprint fp = mag_footprint(g, cs.x, cs.y, kx, ky);
        const double jc = fp.P * inv_pitch + g.cs, jw = (double)fp.sigma * inv_pitch;
        const double jlo = fmax(jc - jw, -2.0), jhi = fmin(jc + jw, (double)g.n_det + 1.0);
        const int j0 = max(0, (int)ceil(jlo) - 1), j1 = min(g.n_det - 1, (int)floor(jhi) + 1);
        const float* yv = y + (size_t)vl * g.n_det;
        for (int j = j0; j <= j1; ++j) {
            const float wgt = mag_weight(fp, mag_bin_s(g, j), B);
            if (wgt != 0.0f) acc = __fmaf_rn(__ldg(yv + j), wgt, acc);
        }
    }
    float* out = p.image_out + (size_t)b * n * n + k;
    *out = p.accumulate ? *out + acc : acc;
}

}  // namespace cbp
