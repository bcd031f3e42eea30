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
// pair has ONE footprint that all its bins share: it is computed once per
// (view, pixel) -- P(k) in FP64, since s_j - P(k) cancels -- and the bins
// evaluate only the nested FP32 form of Eq. 14 at
// x = s_j - P(k), rounded to FP32 from FP64.
//
// FP: a CTA per (slice, view, 128-bin tile) walks the image lines (rows or
// columns, whichever the tile's rays cross more steeply); per line the
// footprints of the pixels the tile's band covers are staged in shared
// memory (each computed once) and each bin sums over the index interval of
// its own band -- no atomics, a fixed order.  cbp_mag_fpw_kernel (default)
// gives the lines to the CTA's warps round-robin with warp-private staging;
// cbp_mag_fp_kernel stages each line for the whole CTA.  BP: threads per
// (slice, pixel) -- or per pixel of a symmetry domain and its 4 / 8 frames
// -- gather over views and the bins of the footprint.  All use mag_footprint
// and mag_weight_x; x differs only by the FP64 rounding of s_j (direct in
// the FP, incremental in the BP), far below FP32's.
#pragma once

#include "cbp_common.cuh"

namespace cbp {

#ifndef CBP_MAG_BRANCHLESS  // A/B knob: the FP walk's weight as a select (1) or an early-out (0)
#define CBP_MAG_BRANCHLESS 1
#endif
#ifndef CBP_MAG_BP_BRANCHLESS  // the same for the BP's bin loop, 4 frames only (measured: config 2,
#define CBP_MAG_BP_BRANCHLESS 1   // 4 frames, 0.528 -> 0.507 ms; config 3, 8 frames, 3.60 -> 4.38 ms)
#endif
constexpr int MAG_FP_BLOCK = 128;
constexpr int MAG_BP_BLOCK = 128;

struct MagFootprint {
    double P;  // detector coordinate of the pixel centre, P(k) (FP64: s_j - P(k) cancels)
    // FP32 shape, with the per-footprint constants of the nested form hoisted:
    float A;       // max |zeta|
    float invC;    // 1 / min |zeta| (+inf when eliminated)
    float w1;      // 1 - B / C
    float zoff;    // (A - C) / 2 + B / 2: z11 = x + zoff
    float minAB;   // min(A, B)
    float hC;      // C / 2
    float sigma;   // support half-width (A + B + C) / 2
    float wscale;  // h^2 m(k) / (A B)  (precise mode: h^2 m(k) / A)
    double Ad;     // precise mode only: max |zeta| in FP64
    float Cz;      // precise mode only: min |zeta|
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
            f = sdd * rcp_approx(r2);
            m = sdd * rsqrtf(r2);
        } else {
            const float invf = rcp_approx(depf);  // refined in FP64 below for P
            double r = (double)invf;
            r = __fma_rn(r, __fma_rn(-dep, r, 1.0), r);
            P = g.sdd * lat * r;
            f = sdd * invf * invf;
            const float Pf = (float)P;
            m = __fmaf_rn(Pf, Pf, sdd * sdd) * rcp_approx(sdd * sqrtf(r2));
        }
        // grad P = f (dep e + lat u)
        gx = f * __fmaf_rn(depf, -suf, latf * cuf);
        gy = f * __fmaf_rn(depf, cuf, latf * suf);
    }
    const float h = (float)g.h, B = (float)g.tau;
    float a1 = fabsf(h * gx), a2 = fabsf(h * gy);
    const float eps = 1e-6f * h;
    if (a1 < eps) a1 = 0.0f;
    if (a2 < eps) a2 = 0.0f;
    const float A = fmaxf(a1, a2), C = fminf(a1, a2);
    MagFootprint fp;
    fp.P = P;
    fp.A = A;
    fp.invC = rcp_approx(C);  // C = 0 -> +inf: sat() eliminates the direction
    fp.w1 = __fmaf_rn(-B, fp.invC, 1.0f);
    fp.zoff = 0.5f * (A - C) + 0.5f * B;
    fp.minAB = fminf(A, B);
    fp.hC = 0.5f * C;
    fp.sigma = 0.5f * (A + B + C);
    fp.wscale = h * h * m * rcp_approx(A * B);
    return fp;
}

// The precise mode (narrow bins, cbp_common.cuh cnsf_prec): the footprint's
// shape in FP64 too, since A enters the knot z11 - A (an FP32 A would shift it
// by ~1e-7 A against a ramp of width tau + C).
__device__ __forceinline__ MagFootprint mag_footprint_prec(const GeomDev& g, double cu, double su, double kx,
                                                           double ky)
{
    double lat, dep;
    mag_frame(g, cu, su, kx, ky, lat, dep);
    double P, gx, gy;
    float m;
    if (g.parallel) {
        P = lat;
        gx = -su;
        gy = cu;
        m = 1.0f;
    } else {
        const double r2 = fma(dep, dep, lat * lat);
        double f;
        if (g.arc) {
            P = g.sdd * atan2(lat, dep);
            f = g.sdd / r2;
            m = (float)(g.sdd / sqrt(r2));
        } else {
            const double r = 1.0 / dep;
            P = g.sdd * lat * r;
            f = g.sdd * r * r;
            m = (float)((P * P + g.sdd * g.sdd) / (g.sdd * sqrt(r2)));
        }
        gx = f * fma(dep, -su, lat * cu);  // grad P = f (dep e + lat u)
        gy = f * fma(dep, cu, lat * su);
    }
    double a1 = fabs(g.h * gx), a2 = fabs(g.h * gy);
    if (a1 < 1e-6 * g.h) a1 = 0.0;  // ledger #7
    if (a2 < 1e-6 * g.h) a2 = 0.0;
    const double A = fmax(a1, a2), C = fmin(a1, a2);
    MagFootprint fp;
    fp.P = P;
    fp.Ad = A;
    fp.Cz = (float)C;
    fp.A = (float)A;
    fp.sigma = (float)(0.5 * (A + g.tau + C));
    fp.wscale = (float)(g.h * g.h / A) * m;
    return fp;
}

__device__ __forceinline__ float mag_weight_prec(const MagFootprint& fp, double x, float B)
{
    if (!(fabs(x) < (double)fp.sigma)) return 0.0f;  // sigma rounded up or down: exact 0 there
    return fp.wscale * cnsf_prec(x, fp.Ad, B, fp.Cz);
}

// W at x = s - P(k) (exactly 0 outside the open support, ledger #15): the
// scalar form of cnsf_num2 with B = tau.  BRANCHLESS: the
// support test selects the result instead of returning early (the FP's
// lanes walk different candidate counts; a divergent early-out costs more
// than the ~20 instructions it skips)
template <bool BRANCHLESS = false>
__device__ __forceinline__ float mag_weight_x(const MagFootprint& fp, float x, float B)
{
    const bool in = fabsf(x) < fp.sigma;
    if (!BRANCHLESS && !in) return 0.0f;
    const float z11 = x + fp.zoff;
    const float z21 = z11 - fp.A;
    const float t11 = sat_fma(z11, fp.invC, 1.0f), t12 = sat_fma(z11, fp.invC, fp.w1);
    const float t21 = sat_fma(z21, fp.invC, 1.0f), t22 = sat_fma(z21, fp.invC, fp.w1);
    float T = t11 * t11;
    T = __fmaf_rn(-t12, t12, T);
    T = __fmaf_rn(-t21, t21, T);
    T = __fmaf_rn(t22, t22, T);
    const float trap = fmaxf(fmin3(z11, fp.minAB, B - z21), 0.0f);
    const float w = fp.wscale * __fmaf_rn(fp.hC, T, trap);
    return BRANCHLESS ? (in ? w : 0.0f) : w;
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
    int vg;            // BP: view groups per pixel (1, 2, 4)
    double sigma_max;  // upper bound of every pixel's support half-width
    // FP over a full scan (F = 4): the image's 4 rotations interleaved per pixel,
    // [n][n][4] (cbp_pad_sym4_kernel with no border): one coalesced float4 per
    // staged pixel instead of 4 loads, two of them walking a column per warp
    const float* pad4;
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

// The band P in (s_lo, s_hi) on line l as index bounds linear in l:
// G0(l) + G1 i > 0 with G0(l) = G00 + Gl l is i > -(G00 + Gl l) / G1 for
// G1 > 0 (a lower bound), i < ... for G1 < 0 (an upper one); G1 = 0 (the
// edge ray parallel to the lines) leaves the line unrestricted (a superset:
// the exact test decides).  FP32 coefficients, widened by 0.01 pixel plus
// their rounding.
struct MagBand {
    float loA, loB, hiA, hiB;  // lo(l) = loA + loB l, hi(l) = hiA + hiB l
};

__device__ __forceinline__ void mag_band_edge(double G00, double Gl, double G1, float& loA, float& loB, float& hiA,
                                              float& hiB, bool& has_lo, bool& has_hi)
{
    if (G1 == 0.0) return;
    const double A = -G00 / G1, Bl = -Gl / G1;
    if (G1 > 0.0) {
        if (!has_lo || A > (double)loA) {  // two bounds on one side: either one is a superset
            loA = (float)A;
            loB = (float)Bl;
        }
        has_lo = true;
    } else {
        if (!has_hi || A < (double)hiA) {
            hiA = (float)A;
            hiB = (float)Bl;
        }
        has_hi = true;
    }
}

__device__ __forceinline__ MagBand mag_band(const MagEdge& lo_e, const MagEdge& hi_e, bool rows, int n)
{
    // P > s_lo: G_lo > 0;  P < s_hi: -G_hi > 0
    float loA = -1e30f, loB = 0.0f, hiA = 1e30f, hiB = 0.0f;
    bool has_lo = false, has_hi = false;
    if (rows) {
        mag_band_edge(lo_e.G00, lo_e.Gr, lo_e.Gc, loA, loB, hiA, hiB, has_lo, has_hi);
        mag_band_edge(-hi_e.G00, -hi_e.Gr, -hi_e.Gc, loA, loB, hiA, hiB, has_lo, has_hi);
    } else {
        mag_band_edge(lo_e.G00, lo_e.Gc, lo_e.Gr, loA, loB, hiA, hiB, has_lo, has_hi);
        mag_band_edge(-hi_e.G00, -hi_e.Gc, -hi_e.Gr, loA, loB, hiA, hiB, has_lo, has_hi);
    }
    MagBand B;
    if (has_lo) {
        const float w = 0.01f + 1e-6f * (fabsf(loA) + fabsf(loB) * (float)n);
        B.loA = loA - w;
        B.loB = loB;
    } else {
        B.loA = -1e30f;
        B.loB = 0.0f;
    }
    if (has_hi) {
        const float w = 0.01f + 1e-6f * (fabsf(hiA) + fabsf(hiB) * (float)n);
        B.hiA = hiA + w;
        B.hiB = hiB;
    } else {
        B.hiA = 1e30f;
        B.hiB = 0.0f;
    }
    return B;
}

// index interval [i0, i1] of the band on line l
__device__ __forceinline__ void mag_band_range(const MagBand& B, int l, int n, int& i0, int& i1)
{
    const float lo = fmaxf(fmaf(B.loB, (float)l, B.loA), -1.0f);
    const float hi = fminf(fmaf(B.hiB, (float)l, B.hiA), (float)n);
    i0 = max(0, (int)ceilf(lo));
    i1 = min(n - 1, (int)floorf(hi));
}

// the staged footprint of one pixel of a line, with its F image values
// (F = 4: the pixel's values in the 4 rotated frames)
template <int F, bool PREC = false>
struct MagStaged {
    double P;
    float A, invC, w1, zoff, minAB, hC, sigma, wscale;
    float val[F];
};
template <int F>
struct MagStaged<F, true> {
    double P, Ad;
    float Cz, sigma, wscale;
    float val[F];
};

// pixel R^q (row, col) of the n x n grid, R(r, c) = (n-1-c, r) (+90 degrees,
// DESIGN.md 5.6): W(v + q N_v/4, j, R^q k) = W(v, j, k)
__device__ __forceinline__ void mag_rot(int n, int q, int& r, int& c)
{
    for (int t = 0; t < q; ++t) {
        const int nr = n - 1 - c;
        c = r;
        r = nr;
    }
}

// FP: y[b][v][j] = sum_k c[b][k] W(v, j, k).  The pixels whose footprint can
// reach bin j have P(k) in (s_j - sigma_max, s_j + sigma_max): on each image
// line that is an index interval, from the two affine edge functions of
// mag_edge (per thread for its bin, per CTA for the tile's band); the exact
// open-support test of mag_weight_x decides.
// F = 4 (one image, a full scan, N_v % 4 == 0): blockIdx.y is a base view
// v < N_v/4 and each weight serves the 4 views v + q N_v/4, reading the image
// at R^q k and writing the natural sinogram rows.
template <int F, bool PREC = false>
__global__ void __launch_bounds__(MAG_FP_BLOCK) cbp_mag_fp_kernel(MagParams p)
{
    __shared__ MagStaged<F, PREC> st[MAG_FP_BLOCK];
    const GeomDev& g = p.g;
    const int j0 = blockIdx.x * MAG_FP_BLOCK;
    const int j = j0 + threadIdx.x, jl = min(j0 + MAG_FP_BLOCK, g.n_det) - 1;
    const int vl = blockIdx.y, b = blockIdx.z;
    const double2 cs = p.view_cs[p.view_begin + vl];
    const double cu = cs.x, su = cs.y;
    const double s = mag_bin_s(g, min(j, g.n_det - 1));
    const float B = (float)g.tau;
    // lines: rows when the tile's middle ray is within 45 degrees of the y axis
    const double sm = 0.5 * (mag_bin_s(g, j0) + mag_bin_s(g, jl));
    double dx, dy;
    if (g.parallel) {
        dx = -cu;
        dy = -su;
    } else if (g.arc) {
        double sg, cg;
        sincos(sm / g.sdd, &sg, &cg);
        dx = -cg * cu - sg * su;
        dy = -cg * su + sg * cu;
    } else {
        dx = -g.sdd * cu - sm * su;
        dy = -g.sdd * su + sm * cu;
    }
    const bool rows = fabs(dy) >= fabs(dx);
    const int n = g.n;
    // the tile's band (uniform over the CTA), and this bin's
    const MagBand tband = mag_band(mag_edge(g, cu, su, mag_bin_s(g, j0) - p.sigma_max),
                                   mag_edge(g, cu, su, mag_bin_s(g, jl) + p.sigma_max), rows, n);
    const MagBand band = mag_band(mag_edge(g, cu, su, s - p.sigma_max), mag_edge(g, cu, su, s + p.sigma_max), rows, n);
    const float* img = p.image + (size_t)b * n * n;
    float acc[F];
#pragma unroll
    for (int q = 0; q < F; ++q) acc[q] = 0.0f;
    for (int l = 0; l < n; ++l) {
        int I0, I1, i0, i1;
        mag_band_range(tband, l, n, I0, I1);
        if (I1 < I0) continue;
        mag_band_range(band, l, n, i0, i1);
        for (int base = I0; base <= I1; base += MAG_FP_BLOCK) {
            const int i = base + threadIdx.x;
            if (i <= I1) {
                const int row = rows ? l : i, col = rows ? i : l;
                const double kx = ((double)col - g.c0) * g.h, ky = (g.c0 - (double)row) * g.h;
                MagStaged<F, PREC> m;
                if constexpr (PREC) {
                    const MagFootprint fp = mag_footprint_prec(g, cu, su, kx, ky);
                    m.P = fp.P;
                    m.Ad = fp.Ad;
                    m.Cz = fp.Cz;
                    m.sigma = fp.sigma;
                    m.wscale = fp.wscale;
                } else {
                    const MagFootprint fp = mag_footprint(g, cu, su, kx, ky);
                    m.P = fp.P;
                    m.A = fp.A;
                    m.invC = fp.invC;
                    m.w1 = fp.w1;
                    m.zoff = fp.zoff;
                    m.minAB = fp.minAB;
                    m.hC = fp.hC;
                    m.sigma = fp.sigma;
                    m.wscale = fp.wscale;
                }
#pragma unroll
                for (int q = 0; q < F; ++q) {
                    int r = row, c = col;
                    mag_rot(n, q, r, c);
                    m.val[q] = __ldg(img + (size_t)r * n + c);
                }
                st[threadIdx.x] = m;
            }
            __syncthreads();
            const int a = max(i0, base), e = min(i1, min(I1, base + MAG_FP_BLOCK - 1));
            for (int q = a; q <= e; ++q) {
                const MagStaged<F, PREC>& m = st[q - base];
                if constexpr (PREC) {
                    MagFootprint fp;
                    fp.Ad = m.Ad;
                    fp.Cz = m.Cz;
                    fp.sigma = m.sigma;
                    fp.wscale = m.wscale;
                    const float wgt = mag_weight_prec(fp, s - m.P, B);
#pragma unroll
                    for (int f = 0; f < F; ++f) acc[f] = __fmaf_rn(m.val[f], wgt, acc[f]);
                } else {
                    MagFootprint fp;
                    fp.P = m.P;
                    fp.A = m.A;
                    fp.invC = m.invC;
                    fp.w1 = m.w1;
                    fp.zoff = m.zoff;
                    fp.minAB = m.minAB;
                    fp.hC = m.hC;
                    fp.sigma = m.sigma;
                    fp.wscale = m.wscale;
                    const float wgt = mag_weight_x(fp, (float)(s - fp.P), B);
#pragma unroll
                    for (int f = 0; f < F; ++f) acc[f] = __fmaf_rn(m.val[f], wgt, acc[f]);
                }
            }
            __syncthreads();
        }
    }
    if (j < g.n_det) {
        if (F == 1) {
            p.sino[((size_t)b * p.view_count + vl) * g.n_det + j] = acc[0];
        } else {
#pragma unroll
            for (int q = 0; q < F; ++q)
                p.sino[((size_t)(p.view_begin + vl) + (size_t)q * (g.n_views / 4)) * g.n_det + j] = acc[q];
        }
    }
}

// FP, warp-per-line form (no CTA barriers in the walk): the CTA's 4 warps
// take the image lines round-robin; a warp stages the footprints of its
// line's band in its own shared memory (each footprint once per CTA, as in
// cbp_mag_fp_kernel) and each lane sums the candidates of its 4 bins
// j0 + lane + 32 r; the warps' partial sums are added in warp order at the end.
constexpr int MAG_FPW_STAGE = 160;  // staged pixels per warp and pass

template <int F>
__global__ void __launch_bounds__(MAG_FP_BLOCK, 5) cbp_mag_fpw_kernel(MagParams p)
{
    constexpr int NW = MAG_FP_BLOCK / 32, R = MAG_FP_BLOCK / 32;  // warps; bins per lane
    __shared__ MagStaged<F> st_all[NW][MAG_FPW_STAGE];
    __shared__ float comb[NW][F][MAG_FP_BLOCK];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    MagStaged<F>* st = st_all[warp];
    const GeomDev& g = p.g;
    const int j0 = blockIdx.x * MAG_FP_BLOCK;
    const int jl = min(j0 + MAG_FP_BLOCK, g.n_det) - 1;
    const int vl = blockIdx.y, b = blockIdx.z;
    const double2 cs = p.view_cs[p.view_begin + vl];
    const double cu = cs.x, su = cs.y;
    const float B = (float)g.tau;
    const double sm = 0.5 * (mag_bin_s(g, j0) + mag_bin_s(g, jl));
    double dx, dy;
    if (g.parallel) {
        dx = -cu;
        dy = -su;
    } else if (g.arc) {
        double sg, cg;
        sincos(sm / g.sdd, &sg, &cg);
        dx = -cg * cu - sg * su;
        dy = -cg * su + sg * cu;
    } else {
        dx = -g.sdd * cu - sm * su;
        dy = -g.sdd * su + sm * cu;
    }
    const bool rows = fabs(dy) >= fabs(dx);
    const int n = g.n;
    const MagBand tband = mag_band(mag_edge(g, cu, su, mag_bin_s(g, j0) - p.sigma_max),
                                   mag_edge(g, cu, su, mag_bin_s(g, jl) + p.sigma_max), rows, n);
    double s[R];
    MagBand band[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        s[r] = mag_bin_s(g, min(j0 + lane + 32 * r, g.n_det - 1));
        band[r] = mag_band(mag_edge(g, cu, su, s[r] - p.sigma_max), mag_edge(g, cu, su, s[r] + p.sigma_max), rows, n);
    }
    const float* img = p.image + (size_t)b * n * n;
    float acc[R][F];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int q = 0; q < F; ++q) acc[r][q] = 0.0f;
    for (int l = warp; l < n; l += NW) {
        int I0, I1;
        mag_band_range(tband, l, n, I0, I1);
        for (int base = I0; base <= I1; base += MAG_FPW_STAGE) {
            const int cnt = min(MAG_FPW_STAGE, I1 - base + 1);
            for (int t = lane; t < cnt; t += 32) {
                const int i = base + t;
                const int row = rows ? l : i, col = rows ? i : l;
                float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);  // issued before the footprint maths
                if (F == 4 && p.pad4) v4 = __ldg(reinterpret_cast<const float4*>(p.pad4) + (size_t)row * n + col);
                const double kx = ((double)col - g.c0) * g.h, ky = (g.c0 - (double)row) * g.h;
                const MagFootprint fp = mag_footprint(g, cu, su, kx, ky);
                MagStaged<F> m;
                m.P = fp.P;
                m.A = fp.A;
                m.invC = fp.invC;
                m.w1 = fp.w1;
                m.zoff = fp.zoff;
                m.minAB = fp.minAB;
                m.hC = fp.hC;
                m.sigma = fp.sigma;
                m.wscale = fp.wscale;
                if constexpr (F == 4) {
                    if (p.pad4) {
                        m.val[0] = v4.x;
                        m.val[1] = v4.y;
                        m.val[2] = v4.z;
                        m.val[3] = v4.w;
                        st[t] = m;
                        continue;
                    }
                }
#pragma unroll
                for (int q = 0; q < F; ++q) {
                    int rr = row, cc = col;
                    mag_rot(n, q, rr, cc);
                    m.val[q] = __ldg(img + (size_t)rr * n + cc);
                }
                st[t] = m;
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < R; ++r) {
                int i0, i1;
                mag_band_range(band[r], l, n, i0, i1);
                const int a = max(i0, base), e = min(i1, base + cnt - 1);
                for (int q = a; q <= e; ++q) {
                    const MagStaged<F>& m = st[q - base];
                    MagFootprint fp;
                    fp.P = m.P;
                    fp.A = m.A;
                    fp.invC = m.invC;
                    fp.w1 = m.w1;
                    fp.zoff = m.zoff;
                    fp.minAB = m.minAB;
                    fp.hC = m.hC;
                    fp.sigma = m.sigma;
                    fp.wscale = m.wscale;
                    const float wgt = mag_weight_x<CBP_MAG_BRANCHLESS>(fp, (float)(s[r] - fp.P), B);
#pragma unroll
                    for (int f = 0; f < F; ++f) acc[r][f] = __fmaf_rn(m.val[f], wgt, acc[r][f]);
                }
            }
            __syncwarp();
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int f = 0; f < F; ++f) comb[warp][f][lane + 32 * r] = acc[r][f];
    __syncthreads();
    const int jj = threadIdx.x, j = j0 + jj;  // one output bin per thread, warps summed in order
    if (j >= g.n_det) return;
#pragma unroll
    for (int f = 0; f < F; ++f) {
        float t = comb[0][f][jj];
        for (int w = 1; w < NW; ++w) t += comb[w][f][jj];
        if (F == 1)
            p.sino[((size_t)b * p.view_count + vl) * g.n_det + j] = t;
        else
            p.sino[((size_t)(p.view_begin + vl) + (size_t)f * (g.n_views / 4)) * g.n_det + j] = t;
    }
}

// BP: c[b][k] = sum_{v, j} y[b][v][j] W(v, j, k) over the bins of k's footprint
// (|j - P/Delta_s - c_s| < sigma/Delta_s, widened by 1e-3 bin; the exact test decides).
// F = 8 (one image, a full scan, N_v % 4 == 0, n even): the dihedral group of
// the square grid, frames g = R^q M^m (R(r, c) = (n-1-c, r), M(r, c) =
// (n-1-r, c)) with W(view_g(v), bin_g(j), g k) = W(v, j, k),
// view_g(v) = (m ? N_v - v : v) + q N_v/4 (mod N_v), bin_g(j) = m ? N_s-1-j : j.
// A thread per pixel k of the triangle r <= c of the top-left quadrant (a
// fundamental domain: its 8 images tile the grid; the transpose M R fixes
// its diagonal, whose pixels take the 4 rotations only) loops over all views
// and owns the 8 (4) output pixels g k: one footprint per 8 (view, pixel)
// pairs, no write conflicts.
// A CTA (MAG_BP_BLOCK threads) is 32 (4 / VG) pixels x VG view groups (views
// interleaved over the groups, for parallelism when the pixel domain is
// small; p.vg = VG in 1, 2, 4); the groups' partial sums are added in group
// order in shared memory.
constexpr int MAG_BP_VG = MAG_BP_BLOCK / 32;

template <int F, bool PREC = false>
__global__ void __launch_bounds__(MAG_BP_BLOCK) cbp_mag_bp_kernel(MagParams p)
{
    extern __shared__ float red[];  // VG > 1: [VG][F][MAG_BP_BLOCK / VG] (none for VG = 1: the L1 keeps it)
    const GeomDev& g = p.g;
    const int n = g.n;
    const int VG = p.vg, warp = threadIdx.x >> 5, vg = warp % VG;
    const int slot = (warp / VG) * 32 + (threadIdx.x & 31);  // pixel of the CTA
    const int t = blockIdx.x * (MAG_BP_BLOCK / VG) + slot;
    const int b = blockIdx.y;
    int row = 0, col = 0;
    bool valid;
    if (F == 1) {
        valid = t < n * n;
        row = t / n;
        col = t - row * n;
    } else if (F == 4) {  // the top-left quadrant (its 4 rotations tile the grid)
        const int half = n / 2;
        valid = t < half * half;
        row = min(t / half, half - 1);
        col = t - (t / half) * half;
    } else {
        // triangle index t -> (row, col), row <= col < half; row r starts at r half - r (r - 1) / 2
        const int half = n / 2;
        valid = t < half * (half + 1) / 2;
        const float tw = (float)(2 * half + 1);
        int r = (int)floorf(0.5f * (tw - sqrtf(fmaxf(tw * tw - 8.0f * (float)t, 0.0f))));
        r = max(0, min(r, half - 1));
        while (r > 0 && r * half - r * (r - 1) / 2 > t) --r;
        while (r + 1 < half && (r + 1) * half - (r + 1) * r / 2 <= t) ++r;
        row = r;
        col = min(half - 1, r + (t - (r * half - r * (r - 1) / 2)));
    }
    const bool diag = F == 8 && row == col;
    const double kx = ((double)col - g.c0) * g.h, ky = (g.c0 - (double)row) * g.h;
    const float B = (float)g.tau;
    const double inv_pitch = 1.0 / g.pitch;
    const int N = g.n_views, vq = N / 4;
    const float* y = p.sino_in + (size_t)b * p.view_count * g.n_det;
    float acc[F];
#pragma unroll
    for (int q = 0; q < F; ++q) acc[q] = 0.0f;
    for (int vl = vg; valid && vl < p.view_count; vl += VG) {
        const double2 cs = p.view_cs[p.view_begin + vl];
        const MagFootprint fp = PREC ? mag_footprint_prec(g, cs.x, cs.y, kx, ky) : mag_footprint(g, cs.x, cs.y, kx, ky);
        const double jc = fp.P * inv_pitch + g.cs, jw = (double)fp.sigma * inv_pitch + 1e-3;
        const double jlo = fmax(jc - jw, -1.0), jhi = fmin(jc + jw, (double)g.n_det);
        const int ja = max(0, (int)ceil(jlo)), jb = min(g.n_det - 1, (int)floor(jhi));
        // sinogram rows of the frames (mirrored frames read their rows backwards)
        const float* yq[F];
#pragma unroll
        for (int q = 0; q < F; ++q) {
            int v = F == 1 ? vl : ((q >= 4) ? N - vl : vl) + (q & 3) * vq;  // < 2 N
            if (v >= N) v -= N;
            yq[q] = y + (size_t)v * g.n_det + ((q >= 4) ? g.n_det - 1 : 0);
        }
        double sj = mag_bin_s(g, ja);
        for (int j = ja; j <= jb; ++j, sj += g.pitch) {
            const float wgt = PREC ? mag_weight_prec(fp, sj - fp.P, B)
                                   : mag_weight_x<CBP_MAG_BP_BRANCHLESS && F == 4>(fp, (float)(sj - fp.P), B);
#pragma unroll
            for (int q = 0; q < F; ++q) {
                if (q < 4 || !diag) acc[q] = __fmaf_rn(__ldg(yq[q] + (q >= 4 ? -j : j)), wgt, acc[q]);
            }
        }
    }
    if (VG > 1) {
        const int per = MAG_BP_BLOCK / VG;
#pragma unroll
        for (int q = 0; q < F; ++q) red[(vg * F + q) * per + slot] = acc[q];
        __syncthreads();
        if (vg != 0) return;
#pragma unroll
        for (int q = 0; q < F; ++q) {
            float sum = red[q * per + slot];
            for (int gg = 1; gg < VG; ++gg) sum += red[(gg * F + q) * per + slot];
            acc[q] = sum;
        }
    }
    if (!valid) return;
#pragma unroll
    for (int q = 0; q < F; ++q) {
        if (q >= 4 && diag) continue;  // the transpose repeats the rotations' pixels
        int r = row, c = col;
        if (q >= 4) r = n - 1 - r;  // M, then R^(q mod 4)
        mag_rot(n, q & 3, r, c);
        float* out = p.image_out + (size_t)b * n * n + (size_t)r * n + c;
        if (p.accumulate == 2)
            mc_red_add(out, acc[q]);  // multicast address (CBP_ACC_MULTIMEM)
        else
            *out = p.accumulate ? *out + acc[q] : acc[q];
    }
}

}  // namespace cbp
