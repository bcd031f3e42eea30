// cbp_fp.cuh -- rows a2-a5: forward projection y = A c (Eq. 6) as an
// atomics-free per-(view, bin) gather over the pixel strip the fan ray covers.
//
// Thread = one detector bin j of one view v of one image.  For the ray of bin
// j everything of Eq. 11-13 that does not depend on the pixel is a constant:
// the ray frame r_j, v_j, the projected pixel directions zeta1 = h r_x,
// zeta2 = h r_y (Eq. 12) and the effective-blur gain g_j.  The
// pixel-dependent quantities are affine in (row, col):
//   s'(k)  = r_j . (p - k)       (Eq. 11 with the pixel moved to the origin, Eq. 4)
//   tau'(k)= g_j (k - p) . v_j    (Eq. 13 on the plane through k, ledger #1)
// so the thread walks the image along the axis most parallel to the ray
// ("lines" i) and, on each line, visits the K pixels q whose blurred support
// can contain the ray: |s'| < (A + B + C)/2.  The crossing position q*(i) of
// the ray on line i is carried in 32.32 fixed point, which keeps s' exact to
// ~1e-7 h at any image size (an FP32 absolute coordinate would lose
// log2(n) bits).  Each output is written once (no atomics,
// deterministic; the paper's FP used atomic adds).
#pragma once

#include "cbp_common.cuh"

namespace cbp {

struct FPParams {
    GeomDev g;
    Tables t;
    const float* image;  // [batch][n][n]
    float* sino;         // [batch][view_count][n_det]
    int view_begin, view_count;
};

constexpr int FP_BLOCK = 64;

__global__ void __launch_bounds__(FP_BLOCK) cbp_fp_kernel(const FPParams P)
{
    const GeomDev& g = P.g;
    const int j = blockIdx.x * FP_BLOCK + threadIdx.x;
    const int vl = blockIdx.y;
    const int b = blockIdx.z;
    if (j >= g.n_det) return;
    const int v = P.view_begin + vl;
    const int n = g.n;

    // ---- per-ray constants (FP64): Eq. 11 frame, Eq. 12 directions, Eq. 13 gain
    const double2 cs = P.t.view_cs[v];
    const double2 bd = P.t.bin_d[j];
    const double cth = cs.x, sth = cs.y, s = bd.x, invL = bd.y;
    const double sphi = s * invL, cphi = g.sdd * invL;
    const double rx = sphi * cth - cphi * sth;  // r_j = (D_ps e + s_j u) / L_j
    const double ry = cphi * cth + sphi * sth;
    const double vx = -ry, vy = rx;             // v_j = (-D_ps u + s_j e) / L_j
    const double h = g.h, c0 = g.c0;
    // s'(row, col) = X00 + col * bcol + row * brow   (r.p = s_j D_po / L_j)
    const double X00 = s * g.sid * invL + h * c0 * (rx - ry);
    const double bcol = -rx * h, brow = ry * h;
    // d(row, col) = (k - p).v = D00 + col * dcol + row * drow  (p.v = -D_po D_ps / L_j)
    const double D00 = g.sid * g.sdd * invL + h * c0 * (vy - vx);
    const double dcol = vx * h, drow = -vy * h;
    const double gj = (double)P.t.bin_f[j].z;

    const bool rows_major = fabs(rx) >= fabs(ry);
    const double a_i = rows_major ? brow : bcol;  // step of s' along the line index
    const double b_q = rows_major ? bcol : brow;  // step of s' along the line (|b_q| = A)
    const double t_i = gj * (rows_major ? drow : dcol);
    const double t_q = gj * (rows_major ? dcol : drow);
    const size_t stride_i = rows_major ? (size_t)n : 1;
    const size_t stride_q = rows_major ? 1 : (size_t)n;

    const double A = fabs(b_q), C = fabs(a_i);
    double dmax = D00;
    dmax = fmax(dmax, D00 + (n - 1) * dcol);
    dmax = fmax(dmax, D00 + (n - 1) * drow);
    dmax = fmax(dmax, D00 + (n - 1) * (dcol + drow));
    const double sig_q = 0.5 * (A + C + gj * dmax) / A;  // support half-width in pixels
    const int K = (int)floor(2.0 * sig_q) + 1;          // max candidates per line

    // crossing of the ray with line i: q*(i) = Q0 + i m
    const double Q0 = -X00 / b_q, m = -a_i / b_q;
    double ilo, ihi;
    if (fabs(m) < 1e-15) {
        const bool hit = Q0 > -sig_q && Q0 < (n - 1) + sig_q;
        ilo = hit ? 0.0 : 1.0;
        ihi = hit ? (double)(n - 1) : 0.0;
    } else {
        double a = (-sig_q - Q0) / m, c = ((n - 1) + sig_q - Q0) / m;
        if (a > c) {
            const double tmp = a;
            a = c;
            c = tmp;
        }
        ilo = fmax(0.0, floor(a));
        ihi = fmin((double)(n - 1), ceil(c));
    }

    const float* img = P.image + (size_t)b * n * n;
    const float bq_fx = (float)(b_q * 0x1p-32);
    const float bq = (float)b_q, tq = (float)t_q, ti = (float)t_i;
    const float T00 = (float)(gj * D00);
    const float hA = (float)A, hC_ = (float)C;
    const float hAmC = 0.5f * (hA - hC_), hApC = 0.5f * (hA + hC_);
    const float invC = 1.0f / hC_;  // +inf when C == 0 (handled by sat)
    const float hC = 0.5f * hC_;

    const int64_t Q0fx = (int64_t)llrint(Q0 * 0x1p32);
    const int64_t Mfx = (int64_t)llrint(m * 0x1p32);
    const int64_t Sfx = (int64_t)llrint(sig_q * 0x1p32);

    double acc = 0.0;
    if (ilo <= ihi) {
        const int i0 = (int)ilo, i1 = (int)ihi;
        int64_t Qi = Q0fx + (int64_t)i0 * Mfx;
        for (int i = i0; i <= i1; ++i, Qi += Mfx) {
            const int q_lo = (int)((Qi - Sfx) >> 32) + 1;  // first pixel past q* - sigma
            const int64_t dq = (int64_t)q_lo * 4294967296LL - Qi;  // (q_lo - q*) in 32.32
            const float x0 = (float)dq * bq_fx;           // s' at pixel q_lo
            const float tau0 = fmaf((float)q_lo, tq, fmaf((float)i, ti, T00));
            const float* line = img + (size_t)i * stride_i;
            float part = 0.0f;
            for (int k = 0; k < K; ++k) {
                const int q = q_lo + k;
                const float x = fmaf((float)k, bq, x0);
                const float B = fmaf((float)k, tq, tau0);
                const float c = ((unsigned)q < (unsigned)n) ? __ldg(line + (size_t)q * stride_q) : 0.0f;
                const float num = cnsf_num(x, B, hAmC, hApC, invC, hC);
                const bool in = fabsf(x) < fmaf(0.5f, B, hApC);  // open support (ledger #15)
                part = fmaf(in ? c : 0.0f, num * rcp_approx(B), part);
            }
            acc += (double)part;
        }
    }
    // W = h^2 M = (h^2 / A) * num / B
    P.sino[((size_t)b * P.view_count + vl) * g.n_det + j] = (float)(acc * (h * h / A));
}

}  // namespace cbp
