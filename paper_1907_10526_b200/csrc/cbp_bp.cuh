// cbp_bp.cuh -- rows a2-a4, a6: back-projection c = A^T y as an atomics-free
// per-pixel gather over views, with the per-(view, bin) constants of the
// CTA's image tile staged in shared memory.
//
// CTA = a 32 x 32 pixel tile and one group of views; thread = a 2 x 2 pixel
// quad.  For each chunk of BP_VC views:
//  1. one thread per view builds the tile's view header in FP64: the exact
//     perspective map (Eq. 4) of every tile pixel as a linear-fractional
//     function of its offset (dc, dr) from the tile anchor k_a, and a proven
//     bound on the half-width (in bins) of each pixel's blurred support,
//     which also gives the tile's bin range;
//  2. the CTA builds one shared-memory entry per (view, bin) of that range:
//     s'(k) = r_j.(p - k) and tau'(k) = g_j (k - p).v_j are affine in
//     (dc, dr), so an entry holds z11 = s' + (A - C)/2 + tau'/2 and tau' at
//     k_a (anchored in FP64: FP32 never sees absolute coordinates), their
//     slopes, the Eq. 12 directions (A, C) and y[v][j] h^2 / A;
//  3. each quad evaluates its pixels as two pairs along the axis most
//     parallel to the rays (those pixels share bins), in packed f32x2
//     arithmetic, over the union of the pair's support intervals.
// Views are split into groups across CTAs for occupancy; groups > 1 write
// FP32 partial images that cbp_reduce_kernel sums in a fixed order.  No
// atomics anywhere: the result is deterministic.
#pragma once

#include "cbp_common.cuh"

namespace cbp {

#ifdef CBP_DEBUG_CHECKS
#include <cstdio>
#define CBP_CHECK(cond, ...)                                   \
    do {                                                       \
        if (!(cond)) {                                         \
            printf("CBP_CHECK %s:%d " #cond "\n", __FILE__, __LINE__); \
            printf(__VA_ARGS__);                                \
        }                                                      \
    } while (0)
#else
#define CBP_CHECK(cond, ...) \
    do {                     \
    } while (0)
#endif

struct BPParams {
    GeomDev g;
    Tables t;
    const float* sino;  // [batch][view_count][n_det]
    float* out;         // groups == 1: image [batch][n][n]; else partials [groups][batch][n][n]
    int view_begin, view_count;
    int groups, views_per_group, batch;
    int accumulate;     // groups == 1 only
};

constexpr int BP_TILE = 32;     // pixels per tile side
constexpr int BP_QUADS = 16;    // quads per tile side
constexpr int BP_THREADS = BP_QUADS * BP_QUADS;
constexpr int BP_VC = 8;        // views per chunk
constexpr int BP_NB = 64;       // bins per view per pass

struct __align__(16) BPEntry {
    float4 a;  // z11(k_a), dz11/dc, dz11/dr, tau'(k_a)
    float4 b;  // dtau'/dc, dtau'/dr, z11 step, tau' step along the pair direction
    float4 c;  // A, 1/C, C/2, y[b][v][j] h^2 / A
};

struct BPHeader {
    int ja, jlo, jhi, horiz;  // nearest bin of P(k_a); tile bin range; pair direction
    float urel, nx, ny, cW;   // u(k) - ja = urel + (nx dc + ny dr) / den;  W(k) = cW / den
    float dena, dx, dy, npass_f;  // den = delta_k = dena + dx dc + dy dr
    double delta_a, f_a, cth, sth, kae;
};

// (hcx, hcy): half-extents, in pixels, of the tile's valid pixel centres
// around the anchor k_a (tiles are clipped by the image border).
__device__ void bp_view_header(const GeomDev& g, const Tables& t, int v, double kax, double kay,
                               double hcx, double hcy, BPHeader& H)
{
    CBP_CHECK(v >= 0 && v < g.n_views, "header v=%d\n", v);
    const double2 cs = t.view_cs[v];
    const double cth = cs.x, sth = cs.y;
    const double kau = kax * cth + kay * sth;   // k_a . u
    const double kae = -kax * sth + kay * cth;  // k_a . e
    const double delta = g.sid - kau;           // depth (p - k_a) . u
    const double Pa = g.sdd * kae / delta;      // Eq. 4
    const double ua = Pa / g.pitch + g.cs;      // continuous bin coordinate
    const double ja = floor(ua + 0.5);
    // P(k) - P(k_a) = (D_ps dk_e + P_a dk_u) / (delta_a - dk_u), dk = (dc h, -dr h)
    const double nx = g.h * (-g.sdd * sth + Pa * cth) / g.pitch;
    const double ny = g.h * (-g.sdd * cth - Pa * sth) / g.pitch;
    const double dx = -g.h * cth, dy = g.h * sth;
    // extremes of the linear-fractional map over the tile are at its corners
    double umin = 1e300, umax = -1e300;
    for (int c = 0; c < 4; ++c) {
        const double dc = (c & 1) ? hcx : -hcx, dr = (c & 2) ? hcy : -hcy;
        const double du = (nx * dc + ny * dr) / (delta + dx * dc + dy * dr);
        umin = fmin(umin, du);
        umax = fmax(umax, du);
    }
    umin += ua;
    umax += ua;
    // |s_j - P(k)| < sigma_j L_j / delta_k  <=>  W != 0   (s' = delta (s_j - P) / L_j)
    const double Rt = sqrt((hcx + 0.5) * (hcx + 0.5) + (hcy + 0.5) * (hcy + 0.5)) * g.h;
    const double dmin = delta - Rt;  // > 0: every pixel is inside the FOV circle < sid
    const double px = g.sid * cth - kax, py = g.sid * sth - kay;
    const double dmax = sqrt(px * px + py * py) + Rt;  // d_j(k) <= |k - p|
    const double taumax = g.tau / g.sdd * dmax;        // g_j <= g(0) = tau / D_ps
    const double sedge = g.cs * g.pitch;
    double Lmax = sqrt(g.sdd * g.sdd + sedge * sedge);
    double cW = 0.5 * (g.h * 1.4142135623730951 + taumax) * Lmax / g.pitch;
    double jl = fmax(0.0, floor(umin - cW / dmin)), jh = fmin((double)(g.n_det - 1), ceil(umax + cW / dmin));
    if (jl <= jh) {
        // refine with the actual zeta range of these bins: A + C = h (|sin psi| + |cos psi|)
        const double s1 = (jl - g.cs) * g.pitch, s2 = (jh - g.cs) * g.pitch;
        const double L1 = sqrt(g.sdd * g.sdd + s1 * s1), L2 = sqrt(g.sdd * g.sdd + s2 * s2);
        Lmax = fmax(L1, L2);
        const double sp1 = (s1 * cth - g.sdd * sth) / L1, cp1 = (g.sdd * cth + s1 * sth) / L1;
        const double sp2 = (s2 * cth - g.sdd * sth) / L2, cp2 = (g.sdd * cth + s2 * sth) / L2;
        const bool peak = (fabs(sp1) > fabs(cp1)) != (fabs(sp2) > fabs(cp2));
        const double fmx = peak ? 1.4142135623730951
                                : fmax(fabs(sp1) + fabs(cp1), fabs(sp2) + fabs(cp2));
        cW = 0.5 * (g.h * fmx + taumax) * Lmax / g.pitch * (1.0 + 1e-6);
        jl = fmax(0.0, floor(umin - cW / dmin - 2e-3));
        jh = fmin((double)(g.n_det - 1), ceil(umax + cW / dmin + 2e-3));
    }
    H.ja = (int)ja;
    H.jlo = (int)jl;
    H.jhi = (int)jh;
    H.horiz = fabs(nx) <= fabs(ny);  // pair the pixels whose projections nearly coincide
    H.urel = (float)(ua - ja);
    H.nx = (float)nx;
    H.ny = (float)ny;
    H.cW = (float)cW;
    H.dena = (float)delta;
    H.dx = (float)dx;
    H.dy = (float)dy;
    H.npass_f = jl <= jh ? (float)(((int)(jh - jl) + BP_NB) / BP_NB) : 0.0f;
    H.delta_a = delta;
    H.f_a = Pa - (ja - g.cs) * g.pitch;
    H.cth = cth;
    H.sth = sth;
    H.kae = kae;
}

__device__ void bp_build_entry(const GeomDev& g, const Tables& t, const BPHeader& H, int j, float y,
                               BPEntry& E)
{
    CBP_CHECK(j >= 0 && j < g.n_det, "build j=%d\n", j);
    const double2 bd = t.bin_d[j];
    const double gj = (double)t.bin_f[j].z;
    const double invL = bd.y;
    const double sphi = bd.x * invL, cphi = g.sdd * invL;
    const double rx = sphi * H.cth - cphi * H.sth;  // r_j (Eq. 11)
    const double ry = cphi * H.cth + sphi * H.sth;
    // s'(k_a) = delta_a (s_j - P(k_a)) / L_j with s_j - P(k_a) = (j - ja) Delta_s - f_a
    const double xa = H.delta_a * ((double)(j - H.ja) * g.pitch - H.f_a) * invL;
    const double da = cphi * H.delta_a + sphi * H.kae;  // (k_a - p) . v_j
    const double h = g.h;
    const double A = fmax(fabs(rx), fabs(ry)) * h, C = fmin(fabs(rx), fabs(ry)) * h;
    const double Ba = gj * da;
    const double tx = -gj * ry * h, ty = -gj * rx * h;  // dtau'/dc, dtau'/dr
    const double zsx = -rx * h + 0.5 * tx, zsy = ry * h + 0.5 * ty;
    const float Cf = (float)C;
    E.a = make_float4((float)(xa + 0.5 * (A - C) + 0.5 * Ba), (float)zsx, (float)zsy, (float)Ba);
    E.b = make_float4((float)tx, (float)ty, (float)(H.horiz ? zsx : zsy), (float)(H.horiz ? tx : ty));
    E.c = make_float4((float)A, 1.0f / Cf, 0.5f * Cf, (float)((double)y * h * h / A));
}

// support interval of one pixel pair (exact projection, per-pixel bound)
__device__ __forceinline__ void pair_range(const BPHeader& H, float ua, float wa, float ub, float wb,
                                           int base, int& jl, int& jh)
{
    const float lo = fminf(ua - wa, ub - wb), hi = fmaxf(ua + wa, ub + wb);
    jl = max(H.ja + __float2int_rd(lo) + 1, base);
    jh = min(H.ja + __float2int_ru(hi) - 1, min(H.jhi, base + BP_NB - 1));
}

// entries row[jl - base .. jh - base]; empty when jh < jl (no pointer is
// formed outside the row: the trip count is an integer)
__device__ __forceinline__ float2 bp_pair(const BPEntry* row, int jl, int jh, int base, float dc,
                                          float dr, float2 acc)
{
    const int cnt = jh - jl + 1;
    if (cnt <= 0) return acc;
    const BPEntry* e = row + (jl - base);
    for (int k = 0; k < cnt; ++k, ++e) {
        const float4 ea = e->a, eb = e->b, ec = e->c;
        const float za = fmaf(dr, ea.z, fmaf(dc, ea.y, ea.x));
        const float Ba = fmaf(dr, eb.y, fmaf(dc, eb.x, ea.w));
        const float2 z11 = make_float2(za, za + eb.z);
        const float2 B = make_float2(Ba, Ba + eb.w);
        const float2 z21 = __fadd2_rn(z11, make_float2(-ec.x, -ec.x));
        const float2 w1 = __ffma2_rn(neg2(B), make_float2(ec.y, ec.y), make_float2(1.0f, 1.0f));
        const float2 num = cnsf_num2(z11, z21, B, w1, ec.x, ec.y, ec.z);
        acc = __ffma2_rn(__fmul2_rn(make_float2(ec.w, ec.w), rcp2(B)), num, acc);
    }
    return acc;
}

__global__ void __launch_bounds__(BP_THREADS, 2) cbp_bp_kernel(const BPParams P)
{
    __shared__ BPEntry tab[BP_VC][BP_NB];
    __shared__ BPHeader hdr[BP_VC];

    const GeomDev& g = P.g;
    const int tid = threadIdx.x;
    const int qx = tid % BP_QUADS, qy = tid / BP_QUADS;
    const int col0 = blockIdx.x * BP_TILE, row0 = blockIdx.y * BP_TILE;
    const int grp = blockIdx.z % P.groups, b = blockIdx.z / P.groups;
    const int vg0 = grp * P.views_per_group;
    const int vgn = min(P.views_per_group, P.view_count - vg0);
    // anchor k_a = centre of the tile's valid pixels (clipped at the border)
    const float hcx = 0.5f * (float)(min(BP_TILE, g.n - col0) - 1);
    const float hcy = 0.5f * (float)(min(BP_TILE, g.n - row0) - 1);
    const double kax = ((double)col0 + hcx - g.c0) * g.h;
    const double kay = (g.c0 - (double)row0 - hcy) * g.h;
    const float dc0 = (float)(2 * qx) - hcx, dr0 = (float)(2 * qy) - hcy;  // quad pixel (0, 0)
    const float* y = P.sino + (size_t)b * P.view_count * g.n_det;

    float2 accH0 = make_float2(0.f, 0.f), accH1 = accH0, accV0 = accH0, accV1 = accH0;
    double tot[4] = {0.0, 0.0, 0.0, 0.0};
    for (int vc = 0; vc < vgn; vc += BP_VC) {
        const int nvc = min(BP_VC, vgn - vc);
        if (tid < nvc)
            bp_view_header(g, P.t, P.view_begin + vg0 + vc + tid, kax, kay, hcx, hcy, hdr[tid]);
        __syncthreads();
        int npass = 0;
        for (int vi = 0; vi < nvc; ++vi) npass = max(npass, (int)hdr[vi].npass_f);
        for (int pass = 0; pass < npass; ++pass) {
            for (int e = tid; e < BP_VC * BP_NB; e += BP_THREADS) {
                const int vi = e / BP_NB, jj = e % BP_NB;
                if (vi < nvc) {
                    const BPHeader& H = hdr[vi];
                    const int j = H.jlo + pass * BP_NB + jj;
                    CBP_CHECK(vg0 + vc + vi < P.view_count, "view %d\n", vg0 + vc + vi);
                    CBP_CHECK(j > H.jhi || (j >= 0 && j < g.n_det), "entry j=%d jlo=%d jhi=%d\n", j, H.jlo, H.jhi);
                    if (j <= H.jhi)
                        bp_build_entry(g, P.t, H, j,
                                       __ldg(y + (size_t)(vg0 + vc + vi) * g.n_det + j), tab[vi][jj]);
                }
            }
            __syncthreads();
            for (int vi = 0; vi < nvc; ++vi) {
                const BPHeader& H = hdr[vi];
                const int base = H.jlo + pass * BP_NB;
                if (base > H.jhi) continue;
                // exact bin coordinates and bounds of the quad's 4 pixels
                const float2 dcp = make_float2(dc0, dc0 + 1.0f);
                const float2 num0 = __ffma2_rn(make_float2(dr0, dr0), make_float2(H.ny, H.ny),
                                               __fmul2_rn(dcp, make_float2(H.nx, H.nx)));
                const float2 num1 = __fadd2_rn(num0, make_float2(H.ny, H.ny));
                const float2 den0 = __ffma2_rn(make_float2(dr0, dr0), make_float2(H.dy, H.dy),
                                               __ffma2_rn(dcp, make_float2(H.dx, H.dx),
                                                          make_float2(H.dena, H.dena)));
                const float2 den1 = __fadd2_rn(den0, make_float2(H.dy, H.dy));
                const float2 i0 = rcp2(den0), i1 = rcp2(den1);
                const float2 u0 = __ffma2_rn(num0, i0, make_float2(H.urel, H.urel));  // row 0
                const float2 u1 = __ffma2_rn(num1, i1, make_float2(H.urel, H.urel));  // row 1
                const float2 w0 = __ffma2_rn(make_float2(H.cW, H.cW), i0, make_float2(2e-3f, 2e-3f));
                const float2 w1 = __ffma2_rn(make_float2(H.cW, H.cW), i1, make_float2(2e-3f, 2e-3f));
                const BPEntry* row = tab[vi];
                int jl, jh;
                if (H.horiz) {  // pairs (0,0)-(1,0) and (0,1)-(1,1)
                    pair_range(H, u0.x, w0.x, u0.y, w0.y, base, jl, jh);
                    CBP_CHECK(jl > jh || (jl >= base && jh < base + BP_NB), "H0 jl=%d jh=%d base=%d u=%f %f w=%f %f\n", jl, jh, base, u0.x, u0.y, w0.x, w0.y);
                    accH0 = bp_pair(row, jl, jh, base, dc0, dr0, accH0);
                    pair_range(H, u1.x, w1.x, u1.y, w1.y, base, jl, jh);
                    accH1 = bp_pair(row, jl, jh, base, dc0, dr0 + 1.0f, accH1);
                } else {        // pairs (0,0)-(0,1) and (1,0)-(1,1)
                    pair_range(H, u0.x, w0.x, u1.x, w1.x, base, jl, jh);
                    CBP_CHECK(jl > jh || (jl >= base && jh < base + BP_NB), "V0 jl=%d jh=%d base=%d\n", jl, jh, base);
                    accV0 = bp_pair(row, jl, jh, base, dc0, dr0, accV0);
                    pair_range(H, u0.y, w0.y, u1.y, w1.y, base, jl, jh);
                    accV1 = bp_pair(row, jl, jh, base, dc0 + 1.0f, dr0, accV1);
                }
            }
            __syncthreads();
        }
        // two-level accumulation: FP32 over a chunk of views, FP64 across chunks
        tot[0] += (double)(accH0.x + accV0.x);
        tot[1] += (double)(accH0.y + accV1.x);
        tot[2] += (double)(accH1.x + accV0.y);
        tot[3] += (double)(accH1.y + accV1.y);
        accH0 = accH1 = accV0 = accV1 = make_float2(0.f, 0.f);
    }
    const size_t plane = (size_t)g.n * g.n;
    float* out = P.out + (P.groups > 1 ? ((size_t)grp * P.batch + b) : (size_t)b) * plane;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int col = col0 + 2 * qx + (q & 1), row = row0 + 2 * qy + (q >> 1);
        if (col < g.n && row < g.n) {
            CBP_CHECK(grp < P.groups && b < P.batch, "out grp=%d b=%d\n", grp, b);
            float* o = out + (size_t)row * g.n + col;
            *o = (P.groups == 1 && P.accumulate) ? *o + (float)tot[q] : (float)tot[q];
        }
    }
}

// out[b][p] = (accumulate ? out[b][p] : 0) + sum_g part[g][b][p], fixed order
__global__ void cbp_reduce_kernel(const float* __restrict__ part, float* __restrict__ out,
                                  size_t count, int groups, int accumulate)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x) {
        float s = accumulate ? out[i] : 0.0f;
        CBP_CHECK(i < count, "reduce i\n");
        for (int gi = 0; gi < groups; ++gi) s += part[(size_t)gi * count + i];
        out[i] = s;
    }
}

}  // namespace cbp
