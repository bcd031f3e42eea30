// cbp_bp.cuh -- rows a2-a4, a6: back-projection c = A^T y as an atomics-free
// per-pixel gather over views, with the per-(view, bin) constants of the
// CTA's image tile staged in shared memory.
//
// CTA = a 16 x 16 pixel tile, thread = one pixel.  For a chunk of BP_VC views:
//  1. one thread per view builds the tile's view header in FP64: the
//     perspective map of the tile anchor k_a (Eq. 4), its linearisation over
//     the tile, and a proven bound on the half-width (in bins) of every
//     tile pixel's blurred support, which gives the tile's bin range;
//  2. the CTA builds one shared-memory entry per (view, bin) of that range:
//     s'(k) = r_j.(p - k) and tau'(k) = g_j (k - p).v_j are affine in the
//     pixel offset (dc, dr) from the anchor, so an entry holds their values
//     at k_a (s' anchored in FP64, so FP32 never sees absolute coordinates)
//     and their two slopes, the Eq. 12 directions (A, C) and y[v][j];
//  3. each pixel visits the bins of its own support interval and evaluates
//     Eq. 14 with the same nested form as the FP kernel.
// Each pixel is written once (no atomics, deterministic).
#pragma once

#include "cbp_common.cuh"

namespace cbp {

struct BPParams {
    GeomDev g;
    Tables t;
    const float* sino;  // [batch][view_count][n_det]
    float* image;       // [batch][n][n]
    int view_begin, view_count, accumulate;
};

constexpr int BP_TILE = 16;                    // pixels per tile side
constexpr int BP_THREADS = BP_TILE * BP_TILE;  // one pixel per thread
constexpr int BP_VC = 8;                       // views per chunk
constexpr int BP_NB = 64;                      // bins per view per pass

struct __align__(16) BPEntry {
    float4 a;  // s'(k_a), ds'/dcol, ds'/drow, tau'(k_a)
    float4 b;  // dtau'/dcol, dtau'/drow, (A - C)/2, (A + C)/2
    float4 c;  // 1/C, C/2, h^2/A, y[b][v][j]
};

struct BPHeader {
    int ja, jlo, jhi, npass;  // nearest bin of P(k_a); tile bin range; passes
    float urel, ux, uy, W;    // u(k) - ja ~ urel + dc ux + dr uy; support half-width bound
    double delta_a, f_a;      // depth of k_a; P(k_a) - s_ja
    double cth, sth, kae;
};

__device__ void bp_view_header(const GeomDev& g, const Tables& t, int v, double kax, double kay,
                               BPHeader& H)
{
    const double2 cs = t.view_cs[v];
    const double cth = cs.x, sth = cs.y;
    const double kau = kax * cth + kay * sth;   // k_a . u
    const double kae = -kax * sth + kay * cth;  // k_a . e
    const double delta = g.sid - kau;           // depth (p - k_a) . u
    const double Pa = g.sdd * kae / delta;      // Eq. 4
    const double ua = Pa / g.pitch + g.cs;      // continuous bin coordinate
    const double ja = floor(ua + 0.5);
    // d u / d(col), d u / d(row): dP/dk = D_ps (e delta + k_e u) / delta^2, dk = (h, 0) / (0, -h)
    const double s2 = g.sdd * g.h / (delta * delta * g.pitch);
    const double ux = s2 * (-sth * delta + kae * cth);
    const double uy = -s2 * (cth * delta + kae * sth);
    const double half = 0.5 * (BP_TILE - 1);
    const double Rt = (half + 0.5) * 1.4142135623730951 * g.h;  // tile radius (mm)
    const double dmin = delta - Rt;
    const double ext = half * (fabs(ux) + fabs(uy));
    // |u(k) - u_lin(k)| <= |u_lin - ua| * Rt / dmin  (second-order term of Eq. 4)
    const double lin = 2.0 * ext * Rt / dmin + 2e-3;
    // |s_j - P(k)| < sigma_j L_j / delta_k  <=>  W != 0   (s' = delta (s_j - P) / L_j)
    const double px = g.sid * cth - kax, py = g.sid * sth - kay;
    const double dmax = sqrt(px * px + py * py) + Rt;  // d_j(k) <= |k - p|
    const double taumax = g.tau / g.sdd * dmax;        // g_j <= g(0) = tau / D_ps
    const double smax_det = g.cs * g.pitch;
    double Lmax = sqrt(g.sdd * g.sdd + smax_det * smax_det);
    double w = 0.5 * (g.h * 1.4142135623730951 + taumax) * Lmax / (dmin * g.pitch) + lin;
    double jl = fmax(0.0, floor(ua - ext - w)), jh = fmin((double)(g.n_det - 1), ceil(ua + ext + w));
    if (jl <= jh) {
        // refine with the actual zeta range of these bins: A + C = h (|sin psi| + |cos psi|)
        const double s1 = (jl - g.cs) * g.pitch, s2b = (jh - g.cs) * g.pitch;
        const double L1 = sqrt(g.sdd * g.sdd + s1 * s1), L2 = sqrt(g.sdd * g.sdd + s2b * s2b);
        Lmax = fmax(L1, L2);
        const double sp1 = s1 / L1 * cth - g.sdd / L1 * sth, cp1 = g.sdd / L1 * cth + s1 / L1 * sth;
        const double sp2 = s2b / L2 * cth - g.sdd / L2 * sth, cp2 = g.sdd / L2 * cth + s2b / L2 * sth;
        const bool peak = (fabs(sp1) > fabs(cp1)) != (fabs(sp2) > fabs(cp2));
        const double fmax_ = peak ? 1.4142135623730951
                                  : fmax(fabs(sp1) + fabs(cp1), fabs(sp2) + fabs(cp2));
        w = 0.5 * (g.h * fmax_ + taumax) * Lmax / (dmin * g.pitch) + lin;
        jl = fmax(0.0, floor(ua - ext - w));
        jh = fmin((double)(g.n_det - 1), ceil(ua + ext + w));
    }
    H.ja = (int)ja;
    H.jlo = (int)jl;
    H.jhi = (int)jh;
    H.npass = jl <= jh ? ((int)(jh - jl) + BP_NB) / BP_NB : 0;
    H.urel = (float)(ua - ja);
    H.ux = (float)ux;
    H.uy = (float)uy;
    H.W = (float)w;
    H.delta_a = delta;
    H.f_a = Pa - (ja - g.cs) * g.pitch;
    H.cth = cth;
    H.sth = sth;
    H.kae = kae;
}

__device__ void bp_build_entry(const GeomDev& g, const Tables& t, const BPHeader& H, int j,
                               float y, BPEntry& E)
{
    const double2 bd = t.bin_d[j];
    const float gj = t.bin_f[j].z;
    const double invL = bd.y;
    const double sphi = bd.x * invL, cphi = g.sdd * invL;
    const double rx = sphi * H.cth - cphi * H.sth;  // r_j (Eq. 11)
    const double ry = cphi * H.cth + sphi * H.sth;
    // s'(k_a) = delta_a (s_j - P(k_a)) / L_j with s_j - P(k_a) = (j - ja) Delta_s - f_a
    const double xa = H.delta_a * ((double)(j - H.ja) * g.pitch - H.f_a) * invL;
    const double da = cphi * H.delta_a + sphi * H.kae;  // (k_a - p) . v_j
    const double h = g.h;
    const double arx = fabs(rx) * h, ary = fabs(ry) * h;
    const float A = (float)fmax(arx, ary), C = (float)fmin(arx, ary);
    E.a = make_float4((float)xa, (float)(-rx * h), (float)(ry * h), (float)(gj * da));
    E.b = make_float4((float)(-gj * ry * h), (float)(-gj * rx * h), 0.5f * (A - C), 0.5f * (A + C));
    E.c = make_float4(1.0f / C, 0.5f * C, (float)(h * h) / A, y);
}

__global__ void __launch_bounds__(BP_THREADS) cbp_bp_kernel(const BPParams P)
{
    __shared__ BPEntry tab[BP_VC][BP_NB];
    __shared__ BPHeader hdr[BP_VC];

    const GeomDev& g = P.g;
    const int tid = threadIdx.x;
    const int tx = tid % BP_TILE, ty = tid / BP_TILE;
    const int col0 = blockIdx.x * BP_TILE, row0 = blockIdx.y * BP_TILE;
    const int b = blockIdx.z;
    const int row = row0 + ty, col = col0 + tx;
    const bool active = row < g.n && col < g.n;
    const float half = 0.5f * (BP_TILE - 1);
    const float dc = (float)tx - half, dr = (float)ty - half;
    const double kax = ((double)col0 + half - g.c0) * g.h;  // tile anchor k_a
    const double kay = (g.c0 - (double)row0 - half) * g.h;
    const float* y = P.sino + (size_t)b * P.view_count * g.n_det;

    double total = 0.0;
    for (int vc = 0; vc < P.view_count; vc += BP_VC) {
        const int nvc = min(BP_VC, P.view_count - vc);
        if (tid < nvc) bp_view_header(g, P.t, P.view_begin + vc + tid, kax, kay, hdr[tid]);
        __syncthreads();
        int npass = 0;
        for (int vi = 0; vi < nvc; ++vi) npass = max(npass, hdr[vi].npass);
        float part = 0.0f;
        for (int pass = 0; pass < npass; ++pass) {
            for (int e = tid; e < BP_VC * BP_NB; e += BP_THREADS) {
                const int vi = e / BP_NB, jj = e % BP_NB;
                if (vi < nvc) {
                    const BPHeader& H = hdr[vi];
                    const int j = H.jlo + pass * BP_NB + jj;
                    if (j <= H.jhi)
                        bp_build_entry(g, P.t, H, j, __ldg(y + (size_t)(vc + vi) * g.n_det + j),
                                       tab[vi][jj]);
                }
            }
            __syncthreads();
            if (active) {
                for (int vi = 0; vi < nvc; ++vi) {
                    const BPHeader& H = hdr[vi];
                    const int base = H.jlo + pass * BP_NB;
                    const float u = fmaf(dr, H.uy, fmaf(dc, H.ux, H.urel));
                    int jl = H.ja + (int)floorf(u - H.W) + 1;
                    int jh = H.ja + (int)ceilf(u + H.W) - 1;
                    jl = max(jl, base);
                    jh = min(jh, min(H.jhi, base + BP_NB - 1));
                    for (int j = jl; j <= jh; ++j) {
                        const BPEntry& E = tab[vi][j - base];
                        const float4 ea = E.a, eb = E.b, ec = E.c;
                        const float x = fmaf(dr, ea.z, fmaf(dc, ea.y, ea.x));
                        const float B = fmaf(dr, eb.y, fmaf(dc, eb.x, ea.w));
                        const float num = cnsf_num(x, B, eb.z, eb.w, ec.x, ec.y);
                        const bool in = fabsf(x) < fmaf(0.5f, B, eb.w);
                        part = fmaf(in ? ec.w * ec.z : 0.0f, num * rcp_approx(B), part);
                    }
                }
            }
            __syncthreads();
        }
        total += (double)part;
    }
    if (active) {
        float* out = P.image + ((size_t)b * g.n + row) * g.n + col;
        *out = P.accumulate ? *out + (float)total : (float)total;
    }
}

}  // namespace cbp
