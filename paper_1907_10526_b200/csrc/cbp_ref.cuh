// cbp_ref.cuh -- row f2: the paper's reference projector "Ref"
// on the GPU, in FP64.
//
//   y[v][j] = sum_k c_k (1/tau) int_{s_j - tau/2}^{s_j + tau/2} chord_k(s) ds
//
// chord_k(s) is the length that the ray from the source to detector point s
// cuts through the indicator pixel k: Eq. 10, the exact fan-beam X-ray
// transform of the pixel basis without detector blur.  The paper integrated
// it symbolically to 1e-12 absolute; here the integrand is split at the
// perspective images (Eq. 4) of the four pixel corners -- between them the
// ray enters and leaves through fixed edges and the chord is a smooth
// (rational x sqrt) function of s -- and each piece gets an 8-point
// Gauss-Legendre rule.
//
// Thread = one (view, bin).  It walks the image lines (rows or columns, the
// axis most perpendicular to the bin's central ray); on each line the wedge
// of rays s in [s_j - tau/2, s_j + tau/2] crosses the line's band of pixels
// between its two edge rays, which bounds the candidate pixels.  One write
// per output, no atomics.  This is an accuracy reference, not a hot path:
// it costs ~100x the CNSF projector.
#pragma once

#include "cbp_common.cuh"

namespace cbp {

struct RefParams {
    GeomDev g;
    Tables t;
    const float* img;  // [batch][n][n]
    double* sino;      // [batch][view_count][n_det]
    int view_begin, view_count, batch;
};

constexpr int REF_BLOCK = 128;

// 8-point Gauss-Legendre on [-1, 1]
__device__ __forceinline__ double gl8_x(int i)
{
    constexpr double X[4] = {0.1834346424956498049395, 0.5255324099163289858177,
                             0.7966664774136267395916, 0.9602898564975362316836};
    return i < 4 ? -X[3 - i] : X[i - 4];
}
__device__ __forceinline__ double gl8_w(int i)
{
    constexpr double Wt[4] = {0.3626837833783619829652, 0.3137066458778872873380,
                              0.2223810344533744705444, 0.1012285362903762591525};
    return i < 4 ? Wt[3 - i] : Wt[i - 4];
}

// chord of the line p + t d (|d| = len) with the box [x0, x1] x [y0, y1]
__device__ __forceinline__ double ref_chord(double px, double py, double dx, double dy, double len,
                                            double x0, double x1, double y0, double y1)
{
    double t0 = -1e300, t1 = 1e300;
    if (dx != 0.0) {
        const double inv = 1.0 / dx;
        const double ta = (x0 - px) * inv, tb = (x1 - px) * inv;
        t0 = fmax(t0, fmin(ta, tb));
        t1 = fmin(t1, fmax(ta, tb));
    } else if (px <= x0 || px >= x1) {
        return 0.0;
    }
    if (dy != 0.0) {
        const double inv = 1.0 / dy;
        const double ta = (y0 - py) * inv, tb = (y1 - py) * inv;
        t0 = fmax(t0, fmin(ta, tb));
        t1 = fmin(t1, fmax(ta, tb));
    } else if (py <= y0 || py >= y1) {
        return 0.0;
    }
    return t1 > t0 ? (t1 - t0) * len : 0.0;
}

struct RefView {
    double ux, uy, ex, ey, px, py, dps;
    int parallel, arc;  // geometry kind (row f3)
};

__device__ __forceinline__ RefView ref_view(const GeomDev& g, double2 cs)
{
    RefView V;
    V.ux = cs.x;
    V.uy = cs.y;
    V.ex = -cs.y;
    V.ey = cs.x;
    V.px = g.sid * cs.x;
    V.py = g.sid * cs.y;
    V.dps = g.sdd;
    V.parallel = g.parallel;
    V.arc = g.arc;
    return V;
}

// the ray of detector coordinate s: a point on it, its direction, |direction|
//   flat: from the source to -D_so u + s e;  arc: from the source at angle
//   s / D_ps (radius D_ps);  parallel: through s e along -u (sign irrelevant)
__device__ __forceinline__ void ref_ray(const RefView& V, double s, double& ox, double& oy, double& dx,
                                        double& dy, double& len)
{
    if (V.parallel) {
        ox = s * V.ex;
        oy = s * V.ey;
        dx = V.ux;
        dy = V.uy;
        len = 1.0;
    } else if (V.arc) {
        double sg, cg;
        sincos(s / V.dps, &sg, &cg);
        ox = V.px;
        oy = V.py;
        dx = V.dps * (-cg * V.ux + sg * V.ex);
        dy = V.dps * (-cg * V.uy + sg * V.ey);
        len = V.dps;
    } else {
        ox = V.px;
        oy = V.py;
        dx = -V.dps * V.ux + s * V.ex;
        dy = -V.dps * V.uy + s * V.ey;
        len = sqrt(V.dps * V.dps + s * s);
    }
}

// detector coordinate of the ray through x: Eq. 4 on the flat detector,
// D_ps x angle on the arc, x.e in parallel beam
__device__ __forceinline__ double ref_project(const RefView& V, double x, double y)
{
    if (V.parallel) return x * V.ex + y * V.ey;
    const double ax = x - V.px, ay = y - V.py;
    const double lat = ax * V.ex + ay * V.ey, dep = -(ax * V.ux + ay * V.uy);
    return V.arc ? V.dps * atan2(lat, dep) : V.dps * lat / dep;
}

// (1/tau) int_a^b chord(s) ds for the pixel box [x0, x1] x [y0, y1]
__device__ double ref_weight(const RefView& V, double a, double b, double x0, double x1, double y0,
                             double y1)
{
    double c[4] = {ref_project(V, x0, y0), ref_project(V, x1, y0), ref_project(V, x0, y1),
                   ref_project(V, x1, y1)};
    // sort the four breakpoints (5-comparator network)
#define REF_SWAP(i, j)                 \
    if (c[i] > c[j]) {                 \
        const double tmp_ = c[i];      \
        c[i] = c[j];                   \
        c[j] = tmp_;                   \
    }
    REF_SWAP(0, 1) REF_SWAP(2, 3) REF_SWAP(0, 2) REF_SWAP(1, 3) REF_SWAP(1, 2)
#undef REF_SWAP
    if (c[3] <= a || c[0] >= b) return 0.0;  // the pixel's shadow misses the bin
    double sum = 0.0, lo = a;
#pragma unroll
    for (int piece = 0; piece < 5; ++piece) {
        const double hi = piece < 4 ? fmin(fmax(c[piece], a), b) : b;
        if (hi > lo) {
            const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
            double part = 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double ox, oy, dx, dy, len;
                ref_ray(V, mid + half * gl8_x(i), ox, oy, dx, dy, len);
                part += gl8_w(i) * ref_chord(ox, oy, dx, dy, len, x0, x1, y0, y1);
            }
            sum += part * half;
            lo = hi;
        }
    }
    return sum;
}

__global__ void __launch_bounds__(REF_BLOCK) cbp_ref_fp_kernel(const RefParams P)
{
    const GeomDev& g = P.g;
    const int j = blockIdx.x * REF_BLOCK + threadIdx.x;
    if (j >= g.n_det) return;
    const int vl = blockIdx.y, b = blockIdx.z;
    const int n = g.n;
    const RefView V = ref_view(g, P.t.view_cs[P.view_begin + vl]);
    const double sj = ((double)j - g.cs) * g.pitch;  // bin centre (arc length on the arc)
    const double a = sj - 0.5 * g.tau, bb = sj + 0.5 * g.tau;
    const double h = g.h, hh = 0.5 * g.h, c0 = g.c0;
    // central ray: walk rows (y const) if it is closer to the y axis
    double ocx, ocy, dcx, dcy, lc_;
    ref_ray(V, sj, ocx, ocy, dcx, dcy, lc_);
    const bool rows = fabs(dcy) >= fabs(dcx);
    // edge rays of the bin (each its own point and direction)
    double oax, oay, dax, day, oex, oey, dbx, dby, ln;
    ref_ray(V, a, oax, oay, dax, day, ln);
    ref_ray(V, bb, oex, oey, dbx, dby, ln);
    // slope of the edge rays along the walk (NaN-free only if the wedge
    // contains no ray parallel to the lines: else every pixel of a line is a candidate)
    const double da = rows ? day : dax, db = rows ? dby : dbx;
    const bool bounded = (da > 0.0 && db > 0.0) || (da < 0.0 && db < 0.0);
    const double ma = rows ? dax / day : day / dax, mb = rows ? dbx / dby : dby / dbx;
    // each edge ray's point: line coordinate, along-line coordinate
    const double pla = rows ? oay : oax, pqa = rows ? oax : oay;
    const double plb = rows ? oey : oex, pqb = rows ? oex : oey;
    const float* img = P.img + (size_t)b * n * n;
    double y = 0.0;
    for (int i = 0; i < n; ++i) {
        // line i: row i (y = (c0 - i) h) or column i (x = (i - c0) h)
        const double lc = rows ? (c0 - i) * h : (i - c0) * h;
        int q0 = 0, q1 = n - 1;
        if (bounded) {
            const double xa0 = pqa + (lc - hh - pla) * ma, xa1 = pqa + (lc + hh - pla) * ma;
            const double xb0 = pqb + (lc - hh - plb) * mb, xb1 = pqb + (lc + hh - plb) * mb;
            const double lo = fmin(fmin(xa0, xa1), fmin(xb0, xb1)), hi = fmax(fmax(xa0, xa1), fmax(xb0, xb1));
            // along-line pixel index of coordinate x: rows -> col = x/h + c0, columns -> row = c0 - y/h
            double ilo = rows ? lo / h + c0 : c0 - hi / h, ihi = rows ? hi / h + c0 : c0 - lo / h;
            ilo = fmax(-1.0, fmin((double)n, floor(ilo - 0.5)));
            ihi = fmax(-1.0, fmin((double)n, ceil(ihi + 0.5)));
            q0 = max(0, (int)ilo);
            q1 = min(n - 1, (int)ihi);
        }
        for (int q = q0; q <= q1; ++q) {
            const int row = rows ? i : q, col = rows ? q : i;
            const float cv = __ldg(img + (size_t)row * n + col);
            if (cv == 0.0f) continue;  // exact
            const double kx = (col - c0) * h, ky = (c0 - row) * h;
            y += (double)cv * ref_weight(V, a, bb, kx - hh, kx + hh, ky - hh, ky + hh);
        }
    }
    P.sino[((size_t)b * P.view_count + vl) * g.n_det + j] = y / g.tau;
}

// A_ref^T: thread = one pixel of one image; for every view the bins whose
// interval meets the pixel's projected corners (widened by tau/2 and one bin)
// -- a superset of the nonzero weights, so this is the exact transpose of
// cbp_ref_fp_kernel (weights outside the support are exactly 0 there too).
struct RefBackParams {
    GeomDev g;
    Tables t;
    const double* sino;  // [batch][view_count][n_det]
    double* img;         // [batch][n][n]
    int view_begin, view_count, batch;
};

__global__ void __launch_bounds__(REF_BLOCK) cbp_ref_bp_kernel(const RefBackParams P)
{
    const GeomDev& g = P.g;
    const int n = g.n;
    const int px = blockIdx.x * REF_BLOCK + threadIdx.x;
    if (px >= n * n) return;
    const int b = blockIdx.y;
    const int row = px / n, col = px % n;
    const double h = g.h, hh = 0.5 * g.h;
    const double kx = (col - g.c0) * h, ky = (g.c0 - row) * h;
    const double* y = P.sino + (size_t)b * P.view_count * g.n_det;
    double acc = 0.0;
    for (int vl = 0; vl < P.view_count; ++vl) {
        const RefView V = ref_view(g, P.t.view_cs[P.view_begin + vl]);
        const double s0 = ref_project(V, kx - hh, ky - hh), s1 = ref_project(V, kx + hh, ky - hh);
        const double s2 = ref_project(V, kx - hh, ky + hh), s3 = ref_project(V, kx + hh, ky + hh);
        const double smin = fmin(fmin(s0, s1), fmin(s2, s3)), smax = fmax(fmax(s0, s1), fmax(s2, s3));
        const double ip = 1.0 / g.pitch;
        const int jlo = max(0, (int)fmax(-1.0, ceil((smin - 0.5 * g.tau) * ip + g.cs - 1.0)));
        const int jhi = min(g.n_det - 1, (int)fmin((double)g.n_det, floor((smax + 0.5 * g.tau) * ip + g.cs + 1.0)));
        for (int j = jlo; j <= jhi; ++j) {
            const double yv = y[(size_t)vl * g.n_det + j];
            if (yv == 0.0) continue;  // exact
            const double sj = ((double)j - g.cs) * g.pitch;
            acc += yv * ref_weight(V, sj - 0.5 * g.tau, sj + 0.5 * g.tau, kx - hh, kx + hh, ky - hh, ky + hh);
        }
    }
    P.img[(size_t)b * n * n + px] = acc / g.tau;
}

}  // namespace cbp
