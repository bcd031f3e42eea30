// cbp_tables.cuh -- row a1: per-view rotation and view-independent per-bin
// tables, FP64 on the device (once per geometry and device, then cached).
#pragma once

#include "cbp_common.cuh"

namespace cbp {

// theta_v = 2 pi v / N_v (ledger #9); s_j = (j - (N_s - 1)/2) Delta_s
// (ledger #10); the bin-centre ray leaves the source at angle phi_j with
// tan phi_j = s_j / D_ps (the detector is rigid w.r.t. the source, so these
// are view-independent); g_j is the effective-blur gain of Eq. 13:
// tau'(k) = g_j * d_j(k), d_j(k) = (k - p) . v_j the pixel depth along the
// ray, g_j = tau D_ps L_j^2 / (L_j^4 - (tau s_j / 2)^2).
__global__ void cbp_tables_kernel(GeomDev g, double2* view_cs, double2* bin_d, float4* bin_f)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < g.n_views) {
        double s, c;
        sincospi(2.0 * (double)t / (double)g.n_views, &s, &c);
        view_cs[t] = make_double2(c, s);
    }
    if (t < g.n_det) {
        const double s = ((double)t - g.cs) * g.pitch;
        const double L2 = g.sdd * g.sdd + s * s;
        const double L = sqrt(L2);
        const double invL = 1.0 / L;
        const double hts = 0.5 * g.tau * s;
        const double gj = g.tau * g.sdd * L2 / (L2 * L2 - hts * hts);
        if (g.arc) {  // the arc ray at gamma is the flat ray at s = D_ps tan(gamma);
                      // its bin subtends tau / D_ps: g_j = 2 tan(tau / (2 D_ps))
            const double gam = ((double)t - g.cs) * g.pitch / g.sdd;
            double sg, cg;
            sincos(gam, &sg, &cg);
            bin_d[t] = make_double2(g.sdd * sg / cg, cg / g.sdd);
            bin_f[t] = make_float4((float)sg, (float)cg, (float)(2.0 * tan(0.5 * g.tau / g.sdd)), 0.0f);
        } else if (g.parallel) {  // every ray is perpendicular to the detector: phi = 0, tau' = tau
            bin_d[t] = make_double2(s, 1.0);
            bin_f[t] = make_float4(0.0f, 1.0f, 1.0f, 0.0f);
        } else {
            bin_d[t] = make_double2(s, invL);
            bin_f[t] = make_float4((float)(s * invL), (float)(g.sdd * invL), (float)gj, 0.0f);
        }
    }
}

}  // namespace cbp
