// cbp_bp.cuh -- rows a2-a4, a6: back-projection c = A^T y as an atomics-free
// per-pixel gather over views, with the per-(view, bin) constants of the
// CTA's image tile staged in shared memory.
//
// CTA = a 32 x 32 pixel tile and one group of views.  For each chunk of BP_VC
// views:
//  1. one thread per view builds the tile's view header: the exact
//     perspective map (Eq. 4) of every tile pixel as a linear-fractional
//     function of its offset (dc, dr) from the tile anchor k_a, and a proven
//     bound on the half-width (in bins) of each pixel's blurred support,
//     which also gives the tile's bin range;
//  2. the CTA builds one shared-memory entry per (view, bin) of that range:
//     s'(k) = r_j.(p - k) and tau'(k) = g_j (k - p).v_j are affine in
//     (dc, dr), so an entry holds z11 = s' + (A - C)/2 + tau'/2 and tau' at
//     k_a (anchored in FP64: FP32 never sees absolute coordinates), their
//     slopes, the Eq. 12 directions (A, C) and y[v][j] h^2 / A;
//  3. every thread evaluates two pixel PAIRS, each pair two pixels adjacent
//     along the image axis most parallel to this view's rays (they share
//     bins), in packed f32x2 arithmetic over the union of their support
//     intervals.  Which pairs a thread owns depends on the rays' direction
//     through the tile, quantised to BP_BUCKETS directions over [0, pi):
//     for each direction the 512 pairs are sorted by their lateral
//     coordinate (perpendicular to the rays) and dealt out in that order, so
//     the 32 lanes of a warp hold a thin strip of pairs along the rays --
//     they read the same few entries (shared-memory broadcast) and have
//     nearly equal trip counts (little divergence).  Partial sums live in
//     registers for a run of views with the same direction bucket and are
//     flushed to a per-tile FP64 accumulator in shared memory.
// Views are split into groups across CTAs for occupancy; groups > 1 write
// FP32 partial images that cbp_reduce_kernel sums in a fixed order.  No
// atomics anywhere: the result is deterministic.
#pragma once

#include <cooperative_groups.h>
#include <type_traits>

#include "cbp_common.cuh"

namespace cbp {

struct BPParams {
    GeomDev g;
    Tables t;
    const uint16_t* pairs;  // [BP_BUCKETS][512] tile pair order per ray direction (r * 32 + c)
    const struct BPHeader* hdrs;  // [tiles_y][tiles_x][view_count] from cbp_bp_header_kernel
    const float* sino;  // [batch][view_count][n_det]
    float* out;         // groups == 1: image [batch][n][n]; else partials [groups][batch][n][n]
    int view_begin, view_count;
    int groups, views_per_group, batch;
    int accumulate;     // groups == 1 only
    // > 0: 4-fold rotational symmetry: slice q reads sinogram rows
    // vl + q sym_stride of batch 0 and accumulates the image in the frame
    // rotated by q (written in output orientation, summed by cbp_reduce_kernel)
    int sym_stride;
    // 8: dihedral symmetry, S = 8 frames g = R^q M^m over base views
    // [0, n_views/8] of the natural sinogram; with `images` > 1 slice group sg
    // is image sg of a batch ([images][n_views][n_det] in, partial planes
    // [images][groups][8] out)
    int sym_mode;
    int images;
    // 1: the view-sharded all-reduce fused into the epilogue (CBP_ACC_MULTIMEM):
    // `out` is a multicast image address and every CTA adds its finished tile of
    // every frame / view group with multimem.red (no partial planes, no reduce
    // kernel): the NVSwitch sums the tiles of all CTAs and ranks while the
    // remaining tiles still compute
    int mc_fused;
    // orbit clusters (cbp_bp_kernel<8, false, true>, n a multiple of BP_TILE):
    // cluster k of 8 CTAs covers the orbit of tile orbit_reps[k] (x, y) under
    // the 8 frames on the orbit_T x orbit_T tile grid
    const int2* orbit_reps;
    int orbit_T;
    // persistent segments (cbp_bp_kernel<8, false, false, true>):
    // the (tile, view) pairs of one image, tile-major, are cut into gridDim.x
    // runs of equal estimated cost (cbp_bp_plan_kernel); CTA b walks segments
    // cta_seg[b] .. cta_seg[b + 1] - 1 (a segment: one tile, views
    // seg_idx[s] .. seg_idx[s + 1] - 1 of it, as tile * view_count + view) and
    // writes each segment's S frame accumulators as a compact block
    // out[image][seg][S][BP_TILE^2] (tile orientation) that cbp_seg_reduce_kernel
    // maps onto the image
    const int* seg_idx;
    const int* cta_seg;
    int seg_max;  // block slots per image (>= segments)
    // 1: the headers are the library's cached set (written by an earlier,
    // completed call), so the staged BP reads them -- and builds chunk 0's
    // geometry-only entries -- before waiting on the FP (programmatic launch)
    int hdr_ready;
    // CBP_BP_PROF (diagnostics, a -DCBP_BP_PROFILE build): per CTA start / end ns, SM,
    // segments, header features
    unsigned long long* prof;
};

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid()
{
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}

constexpr int BP_TILE = 32;       // pixels per tile side
constexpr int BP_THREADS = 256;   // 8 warps x 2 pairs x 2 pixels x 32 lanes = 32 x 32
#ifndef CBP_BP_VC  // (compile-time knobs for A/B builds)
#define CBP_BP_VC 8
#endif
#ifndef CBP_BP_NB
#define CBP_BP_NB 80
#endif
constexpr int BP_VC = CBP_BP_VC;  // views per chunk
constexpr int BP_NB = CBP_BP_NB;  // bins per view per pass (a 32-pixel tile spans <= ~64 at config 2)
// the chunk shape of the staged BP: W = 0 the default (8 views x 80 bins);
// W = 1 for wide projected tiles (4 views x 128 bins: the paper's timing
// shapes, where a tile spans 64-90+ bins and 80-bin passes split views in
// two) -- the same shared memory budget
template <int W>
struct BPShape {
    static constexpr int VC = W ? 4 : BP_VC;
    static constexpr int NB = W ? 128 : BP_NB;
};
#ifndef CBP_BP_BUCKETS  // (compile-time knobs for A/B builds)
#define CBP_BP_BUCKETS 32
#endif
#ifndef CBP_BP_RUN_CHUNKS
#define CBP_BP_RUN_CHUNKS 4
#endif
constexpr int BP_BUCKETS = CBP_BP_BUCKETS;        // ray directions over [0, pi) for the pair order
constexpr int BP_RUN_CHUNKS = CBP_BP_RUN_CHUNKS;  // register partial sums span at most 4 chunks (32 views)
constexpr int BP_PAIRS = BP_TILE * BP_TILE / 2;

struct __align__(16) BPEntry {
    float4 a;  // z11(k_a), dz11/dc, dz11/dr, tau'(k_a)
    float4 b;  // dtau'/dc, dtau'/dr, z11 step, tau' step along the pair direction
    float4 c;  // A, 1/C, C/2, y[b][v][j] h^2 / A
};

struct __align__(16) BPHeader {
    int ja, jlo, jhi, bucket;  // nearest bin of P(k_a); tile bin range; ray-direction bucket
    float urel, nx, ny, cW;    // u(k) - ja = urel + (nx dc + ny dr) / den;  W(k) = cW / den
    float dena, dx, dy, npass_f;  // den = delta_k = dena + dx dc + dy dr
    double delta_a, f_a, cth, sth, kae;
};

// (hcx, hcy): half-extents, in pixels, of the tile's valid pixel centres
// around the anchor k_a (tiles are clipped by the image border).
__device__ void bp_view_header(const GeomDev& g, const Tables& t, int v, double kax, double kay,
                               float hcx, float hcy, BPHeader& H)
{
    const double2 cs = t.view_cs[v];
    const double cth = cs.x, sth = cs.y;
    const double kau = kax * cth + kay * sth;   // k_a . u
    const double kae = -kax * sth + kay * cth;  // k_a . e
    if (g.parallel) {  // row f3: P(k) = k.e, linear in (dc, dr); no depth, tau' = tau
        const double ua = kae / g.pitch + g.cs;
        const double ja = floor(ua + 0.5);
        const float h = (float)g.h, ip = (float)(1.0 / g.pitch), fc = (float)cth, fs = (float)sth;
        const float nx = -h * fs * ip, ny = -h * fc * ip;  // dk = (dc h, -dr h)
        const float umin = -fabsf(nx) * hcx - fabsf(ny) * hcy, umax = -umin;
        const float urel = (float)(ua - ja);
        // |s_j - P(k)| < (A + C + tau)/2, A + C = h (|sin| + |cos|) for every ray of the view
        const float cW = 0.5f * (h * (fabsf(fs) + fabsf(fc)) + (float)g.tau) * ip * (1.0f + 1e-5f);
        const float jsh = (float)ja;
        const float jl = fmaxf(0.0f, floorf(jsh + urel + umin - cW - 0.01f));
        const float jh = fminf((float)(g.n_det - 1), ceilf(jsh + urel + umax + cW + 0.01f));
        H.ja = (int)ja;
        H.jlo = (int)jl;
        H.jhi = (int)jh;
        float phi = atan2f(-fs, -fc);  // the rays run along -u
        if (phi < 0.0f) phi += 3.14159265f;
        H.bucket = min(BP_BUCKETS - 1, max(0, (int)(phi * (BP_BUCKETS / 3.14159265f))));
        H.urel = urel;
        H.nx = nx;
        H.ny = ny;
        H.cW = cW;
        H.dena = 1.0f;
        H.dx = 0.0f;
        H.dy = 0.0f;
        H.npass_f = jl <= jh ? (float)(((int)(jh - jl) + BP_NB) / BP_NB) : 0.0f;
        H.delta_a = 1.0;  // s'(k_a) = (j - ja) Delta_s - f_a (with 1/L_j = 1 in the tables)
        H.f_a = kae - (ja - g.cs) * g.pitch;
        H.cth = cth;
        H.sth = sth;
        H.kae = kae;
        return;
    }
    const double delta = g.sid - kau;           // depth (p - k_a) . u
    const double Pa = g.sdd * kae / delta;      // Eq. 4
    const double ua = Pa / g.pitch + g.cs;      // continuous bin coordinate
    const double ja = floor(ua + 0.5);
    // everything below only bounds ranges: FP32 with explicit guards
    const float h = (float)g.h, ip = (float)(1.0 / g.pitch), sdd = (float)g.sdd;
    const float fc = (float)cth, fs = (float)sth, fPa = (float)Pa, fd = (float)delta;
    // P(k) - P(k_a) = (D_ps dk_e + P_a dk_u) / (delta_a - dk_u), dk = (dc h, -dr h)
    const float nx = h * (-sdd * fs + fPa * fc) * ip;
    const float ny = h * (-sdd * fc - fPa * fs) * ip;
    const float dx = -h * fc, dy = h * fs;
    // extremes of the linear-fractional map over the tile are at its corners
    float umin = 3.0e38f, umax = -3.0e38f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float dc = (c & 1) ? hcx : -hcx, dr = (c & 2) ? hcy : -hcy;
        const float du = (nx * dc + ny * dr) / (fd + dx * dc + dy * dr);
        umin = fminf(umin, du);
        umax = fmaxf(umax, du);
    }
    if (g.arc) {  // row f3, arc detector: bin coordinate gamma(k) / dgam with tan gamma = k_e / delta
        const double ta = kae / delta, gam_a = atan(ta), dgam = g.pitch / g.sdd;
        const double uaa = gam_a / dgam + g.cs, jaa = floor(uaa + 0.5);
        // linearise atan over the tile: gamma - gamma_a ~ (t - t_a) / (1 + t_a^2); the flat map
        // (P - P_a) / Delta_s = D_ps (t - t_a) / Delta_s, so the slopes scale by 1 / (1 + t_a^2)
        const float sc = (float)(1.0 / (1.0 + ta * ta));
        const float dt = fmaxf(fabsf(umin), fabsf(umax)) * (float)(g.pitch / g.sdd);  // max |t - t_a|
        const float E = 0.5f * 0.65f * dt * dt / (float)dgam * 1.1f + 1e-4f;  // |atan''| <= 0.65, in bins
        const float Rt = sqrtf((hcx + 0.5f) * (hcx + 0.5f) + (hcy + 0.5f) * (hcy + 0.5f)) * h;
        const float dmin = fd - fabsf(dx) * (hcx + 0.5f) - fabsf(dy) * (hcy + 0.5f);
        const double dist_a = sqrt(delta * delta + kae * kae);
        const float sigma = 0.5f * (h * 1.41421356f + (float)(2.0 * tan(0.5 * g.tau / g.sdd)) * ((float)dist_a + Rt));
        // |gamma - gamma(k)| < asin(sigma / |k - p|) <= asin(x), x = sigma / delta(k)
        // <= x / sqrt(1 - x^2) (x < 1; x >= 1: any angle) -- the small-angle 1.01 x
        // undercounts for a source within a few pixels (found by tools/fuzz_wide.py);
        // den = delta(k) <= fd + Rt
        const float xs = sigma / fmaxf(dmin, 1e-30f);
        const float fac = xs < 0.999f ? fmaxf(1.01f, rsqrtf(1.0f - xs * xs)) * 1.0001f : 1e7f;
        const float cW = fac * sigma / (float)dgam + E * (fd + Rt);
        const float urel = (float)(uaa - jaa);
        const float jsh = (float)jaa;
        const float jl = fmaxf(0.0f, floorf(jsh + urel + umin * sc - cW / dmin - 0.01f));
        const float jh = fminf((float)(g.n_det - 1), ceilf(jsh + urel + umax * sc + cW / dmin + 0.01f));
        H.ja = (int)jaa;
        H.jlo = (int)jl;
        H.jhi = (int)jh;
        float phi = atan2f((float)(kay - g.sid * sth), (float)(kax - g.sid * cth));
        if (phi < 0.0f) phi += 3.14159265f;
        H.bucket = min(BP_BUCKETS - 1, max(0, (int)(phi * (BP_BUCKETS / 3.14159265f))));
        H.urel = urel;
        H.nx = nx * sc;
        H.ny = ny * sc;
        H.cW = cW;
        H.dena = fd;
        H.dx = dx;
        H.dy = dy;
        H.npass_f = jl <= jh ? (float)(((int)(jh - jl) + BP_NB) / BP_NB) : 0.0f;
        H.delta_a = delta;  // depth; s'(k_a) = |p - k_a| sin(gamma_j - gamma_a) in bp_build_entry
        H.f_a = gam_a - (jaa - g.cs) * dgam;
        H.cth = cth;
        H.sth = sth;
        H.kae = kae;
        return;
    }
    const float urel = (float)(ua - ja);
    // |s_j - P(k)| < sigma_j L_j / delta_k  <=>  W != 0   (s' = delta (s_j - P) / L_j),
    // sigma_j = (A + C + tau') / 2 <= (h (|sin psi| + |cos psi|) + tau'_max) / 2
    const float Rt = sqrtf((hcx + 0.5f) * (hcx + 0.5f) + (hcy + 0.5f) * (hcy + 0.5f)) * h;
    // least depth over the tile's pixels (depth is affine: extremes at the corners); > 0
    // because every pixel is inside the FOV circle < sid.  (fd - Rt, the circumscribed
    // circle, is far too low for a ragged tile near the source.)
    const float dmin = fd - fabsf(dx) * (hcx + 0.5f) - fabsf(dy) * (hcy + 0.5f);
    const float px = (float)(g.sid * cth - kax), py = (float)(g.sid * sth - kay);
    const float taumax = (float)(g.tau / g.sdd) * (sqrtf(px * px + py * py) + Rt);  // g_j <= tau/D_ps
    const float sedge = (float)(g.cs * g.pitch);
    float Lmax = sqrtf(sdd * sdd + sedge * sedge);
    float cW = 0.5f * (h * 1.41421356f + taumax) * Lmax * ip;
    const float jsh = (float)ja;
    float jl = fmaxf(0.0f, floorf(jsh + urel + umin - cW / dmin)),
          jh = fminf((float)(g.n_det - 1), ceilf(jsh + urel + umax + cW / dmin));
    if (jl <= jh) {
        // refine with the actual zeta range of these bins: A + C = h (|sin psi| + |cos psi|)
        const float s1 = (jl - (float)g.cs) * (float)g.pitch, s2 = (jh - (float)g.cs) * (float)g.pitch;
        const float L1 = sqrtf(sdd * sdd + s1 * s1), L2 = sqrtf(sdd * sdd + s2 * s2);
        Lmax = fmaxf(L1, L2);
        const float sp1 = (s1 * fc - sdd * fs) / L1, cp1 = (sdd * fc + s1 * fs) / L1;
        const float sp2 = (s2 * fc - sdd * fs) / L2, cp2 = (sdd * fc + s2 * fs) / L2;
        // a diagonal (|sin| = |cos|) lies between the two end rays: one crossing flips the
        // dominant axis; two need an angular span >= 90 degrees (cos(span) <= 0)
        const bool peak = ((fabsf(sp1) > fabsf(cp1)) != (fabsf(sp2) > fabsf(cp2))) ||
                          (sp1 * sp2 + cp1 * cp2 < 0.01f);
        const float fmx = peak ? 1.41421356f
                               : fmaxf(fabsf(sp1) + fabsf(cp1), fabsf(sp2) + fabsf(cp2));
        cW = 0.5f * (h * fmx + taumax) * Lmax * ip * (1.0f + 1e-5f);
        jl = fmaxf(0.0f, floorf(jsh + urel + umin - cW / dmin - 0.01f));
        jh = fminf((float)(g.n_det - 1), ceilf(jsh + urel + umax + cW / dmin + 0.01f));
    }
    H.ja = (int)ja;
    H.jlo = (int)jl;
    H.jhi = (int)jh;
    // direction of the rays through the tile (source -> anchor), modulo pi
    float phi = atan2f((float)(kay - g.sid * sth), (float)(kax - g.sid * cth));
    if (phi < 0.0f) phi += 3.14159265f;
    H.bucket = min(BP_BUCKETS - 1, max(0, (int)(phi * (BP_BUCKETS / 3.14159265f))));
    H.urel = urel;
    H.nx = nx;
    H.ny = ny;
    H.cW = cW;
    H.dena = fd;
    H.dx = dx;
    H.dy = dy;
    H.npass_f = jl <= jh ? (float)(((int)(jh - jl) + BP_NB) / BP_NB) : 0.0f;
    H.delta_a = delta;
    H.f_a = Pa - (ja - g.cs) * g.pitch;
    H.cth = cth;
    H.sth = sth;
    H.kae = kae;
}

// anchor of a tile: centre of its valid pixels (tiles are clipped by the border)
__device__ __forceinline__ void bp_tile_anchor(const GeomDev& g, int tx, int ty, float& hcx,
                                               float& hcy, double& kax, double& kay)
{
    const int col0 = tx * BP_TILE, row0 = ty * BP_TILE;
    hcx = 0.5f * (float)(min(BP_TILE, g.n - col0) - 1);
    hcy = 0.5f * (float)(min(BP_TILE, g.n - row0) - 1);
    kax = ((double)col0 + hcx - g.c0) * g.h;
    kay = (g.c0 - (double)row0 - hcy) * g.h;
}

// all (tile, view) headers of one BP launch, ahead of the BP kernel (so the
// FP64 header chain is off the BP kernel's critical path)
__global__ void __launch_bounds__(128) cbp_bp_header_kernel(GeomDev g, Tables t, int view_begin,
                                                            int view_count, int tiles_x,
                                                            BPHeader* __restrict__ out)
{
    const int tile = blockIdx.x;
    const int vl = blockIdx.y * blockDim.x + threadIdx.x;
    if (vl >= view_count) return;
    float hcx, hcy;
    double kax, kay;
    bp_tile_anchor(g, tile % tiles_x, tile / tiles_x, hcx, hcy, kax, kay);
    BPHeader H;
    bp_view_header(g, t, view_begin + vl, kax, kay, hcx, hcy, H);
    out[(size_t)tile * view_count + vl] = H;
}

// pairs along x for ray directions within 45 degrees of the x axis
__host__ __device__ inline bool bucket_horiz(int b) { return b < BP_BUCKETS / 4 || b >= 3 * BP_BUCKETS / 4; }

// PAR (parallel beam, tau' = tau): b.x, b.y carry 1 - tau / C and 1 / tau in
// place of the tau' slopes (zero there), for bp_weight<true>
template <bool PAR = false>
__device__ void bp_build_entry(const GeomDev& g, const Tables& t, const BPHeader& H, int j, float y,
                               BPEntry& E)
{
    const double2 bd = t.bin_d[j];
    const float4 bf = t.bin_f[j];
    const double invL = bd.y;  // parallel: 1
    const double sphi = g.parallel ? 0.0 : bd.x * invL, cphi = g.parallel ? 1.0 : g.sdd * invL;
    const double rxd = sphi * H.cth - cphi * H.sth;  // r_j (Eq. 11)
    const double ryd = cphi * H.cth + sphi * H.sth;
    // s'(k_a) = delta_a (s_j - P(k_a)) / L_j with s_j - P(k_a) = (j - ja) Delta_s - f_a  (FP64)
    const double xa = g.arc ? sqrt(H.delta_a * H.delta_a + H.kae * H.kae) *
                                  sin((double)(j - H.ja) * (g.pitch / g.sdd) - H.f_a)
                            : H.delta_a * ((double)(j - H.ja) * g.pitch - H.f_a) * invL;
    const float rx = (float)rxd, ry = (float)ryd;
    const float da = bf.y * (float)H.delta_a + bf.x * (float)H.kae;  // (k_a - p) . v_j
    const float h = (float)g.h, gj = g.parallel ? 0.0f : bf.z;
    const float A = fmaxf(fabsf(rx), fabsf(ry)) * h, C = fminf(fabsf(rx), fabsf(ry)) * h;
    const float Ba = g.parallel ? (float)g.tau : gj * da;  // parallel: tau' = tau, no slopes
    const float tx = -gj * ry * h, ty = -gj * rx * h;  // dtau'/dc, dtau'/dr
    const float zsx = -rx * h + 0.5f * tx, zsy = ry * h + 0.5f * ty;
    E.a = make_float4((float)(xa + 0.5 * ((double)A - (double)C) + 0.5 * (double)Ba), zsx, zsy, Ba);
    const bool horiz = bucket_horiz(H.bucket);
    E.b = make_float4(tx, ty, horiz ? zsx : zsy, horiz ? tx : ty);
    E.c = make_float4(A, 1.0f / C, 0.5f * C, y * (h * h / A));
    if constexpr (PAR) E.b = make_float4(fmaf(-Ba, E.c.y, 1.0f), 1.0f / Ba, E.b.z, 0.0f);
}

// The precise mode (narrow bins, cbp_common.cuh cnsf_prec): s' at the anchor,
// its slopes and A in FP64, so s'(k) and the knots are exact to ~ulp of
// their own size (S = 1 only; the symmetric and batched paths stay FP32).
struct __align__(16) BPEntryP {
    double xa, sc, sr;  // s'(k_a), ds'/dc, ds'/dr
    double A;           // max |zeta|
    float Ba, tx, ty;   // tau'(k_a), dtau'/dc, dtau'/dr
    float Cz;           // min |zeta|
    float yw;           // y[v][j] h^2 / A
};

__device__ void bp_build_entry_prec(const GeomDev& g, const Tables& t, const BPHeader& H, int j, float y,
                                    BPEntryP& E)
{
    const double2 bd = t.bin_d[j];
    const float4 bf = t.bin_f[j];
    const double invL = bd.y;
    const double sphi = g.parallel ? 0.0 : bd.x * invL, cphi = g.parallel ? 1.0 : g.sdd * invL;
    const double rxd = sphi * H.cth - cphi * H.sth, ryd = cphi * H.cth + sphi * H.sth;
    E.xa = g.arc ? sqrt(H.delta_a * H.delta_a + H.kae * H.kae) * sin((double)(j - H.ja) * (g.pitch / g.sdd) - H.f_a)
                 : H.delta_a * ((double)(j - H.ja) * g.pitch - H.f_a) * invL;
    E.sc = -rxd * g.h;  // dk = (dc h, -dr h), s' = r_j . (p - k)
    E.sr = ryd * g.h;
    const double Ad = fmax(fabs(rxd), fabs(ryd)) * g.h;
    E.A = Ad;
    const float rx = (float)rxd, ry = (float)ryd, h = (float)g.h, gj = g.parallel ? 0.0f : bf.z;
    const float da = bf.y * (float)H.delta_a + bf.x * (float)H.kae;  // (k_a - p) . v_j
    E.Ba = g.parallel ? (float)g.tau : gj * da;
    E.tx = -gj * ry * h;
    E.ty = -gj * rx * h;
    E.Cz = (float)(fmin(fabs(rxd), fabs(ryd)) * g.h);
    E.yw = y * (float)(g.h * g.h / Ad);
}

// entries row[jl - base .. jh - base] for one pixel pair (dc, dr).{x, y}
__device__ __forceinline__ void bp_pair_prec(const BPEntryP* row, int jl, int jh, int base, float2 dc, float2 dr,
                                             float2& acc)
{
    if (jh < jl) return;
    CBP_CHECK(jl >= base && jh - base < 128, "bp_pair_prec jl=%d jh=%d base=%d\n", jl, jh, base);
    const BPEntryP* e = row + (jl - base);
    for (int k = jl; k <= jh; ++k, ++e) {
        const double xa = e->xa, sc = e->sc, sr = e->sr, A = e->A;
        const float Ba = e->Ba, tx = e->tx, ty = e->ty, Cz = e->Cz, yw = e->yw;
        const float wa = cnsf_prec(fma((double)dr.x, sr, fma((double)dc.x, sc, xa)), A,
                                   fmaf(dr.x, ty, fmaf(dc.x, tx, Ba)), Cz);
        const float wb = cnsf_prec(fma((double)dr.y, sr, fma((double)dc.y, sc, xa)), A,
                                   fmaf(dr.y, ty, fmaf(dc.y, tx, Ba)), Cz);
        acc.x = fmaf(yw, wa, acc.x);
        acc.y = fmaf(yw, wb, acc.y);
    }
}

// one entry, one pixel pair (lane b = lane a + one pixel along the pair axis):
// returns num / tau' for both pixels (the weight without the h^2/A factor)
template <bool PAR = false>
__device__ __forceinline__ float2 bp_weight(const BPEntry* e, float dc, float dr)
{
    const float4 ea = e->a, eb = e->b, ec = e->c;
    if constexpr (PAR) {  // parallel beam: tau' = tau (ea.w), w1 and 1 / tau from the entry
        const float za = fmaf(dr, ea.z, fmaf(dc, ea.y, ea.x));
        const float2 z11 = make_float2(za, za + eb.z);
        const float2 B = make_float2(ea.w, ea.w);
        const float2 z21 = __fadd2_rn(z11, make_float2(-ec.x, -ec.x));
        const float2 num = cnsf_num2(z11, z21, B, make_float2(eb.x, eb.x), ec.x, ec.y, ec.z);
        return __fmul2_rn(num, make_float2(eb.y, eb.y));
    }
    const float za = fmaf(dr, ea.z, fmaf(dc, ea.y, ea.x));
    const float Ba = fmaf(dr, eb.y, fmaf(dc, eb.x, ea.w));
    const float2 z11 = make_float2(za, za + eb.z);
    const float2 B = make_float2(Ba, Ba + eb.w);
    const float2 z21 = __fadd2_rn(z11, make_float2(-ec.x, -ec.x));
    const float2 w1 = __ffma2_rn(neg2(B), make_float2(ec.y, ec.y), make_float2(1.0f, 1.0f));
    const float2 num = cnsf_num2(z11, z21, B, w1, ec.x, ec.y, ec.z);
    return __fmul2_rn(num, rcp2(B));
}

// entries row[jl - base .. jh - base]; empty when jh < jl (no pointer is
// formed outside the row: the trip count is an integer).  S == 1: the entry's
// c.w is y h^2/A.  S > 1: c.w is h^2/A and the S raw y values of the entry
// are yrow[entry * S + q] (staged from the sinogram by bp_y_load).
template <int S, bool PAR = false>
__device__ __forceinline__ void bp_pair(const BPEntry* row, const float* yrow, int jl, int jh,
                                        int base, float dc, float dr, float2 (&acc)[S])
{
    if (jh < jl) return;
    CBP_CHECK(jl >= base && jh - base < 128, "bp_pair jl=%d jh=%d base=%d\n", jl, jh, base);
    const int cnt = jh - jl + 1;
    const BPEntry* e = row + (jl - base);
    const float* ys = yrow + (jl - base) * S;
    for (int k = 0; k < cnt; ++k, ++e, ys += S) {
        if constexpr (S == 1) {
            const float2 w = bp_weight<PAR>(e, dc, dr);
            const float yw = e->c.w;
            acc[0] = __ffma2_rn(make_float2(yw, yw), w, acc[0]);
        } else {
            const float hA = e->c.w;
            const float2 w = __fmul2_rn(bp_weight<PAR>(e, dc, dr), make_float2(hA, hA));
            if constexpr (S == 2) {
                const float2 y2 = *reinterpret_cast<const float2*>(ys);
                acc[0] = __ffma2_rn(make_float2(y2.x, y2.x), w, acc[0]);
                acc[1] = __ffma2_rn(make_float2(y2.y, y2.y), w, acc[1]);
            } else {
                static_assert(S % 4 == 0, "S is 1, 2 or a multiple of 4");
#pragma unroll
                for (int q = 0; q < S; q += 4) {
                    const float4 y4 = *reinterpret_cast<const float4*>(ys + q);
                    acc[q] = __ffma2_rn(make_float2(y4.x, y4.x), w, acc[q]);
                    acc[q + 1] = __ffma2_rn(make_float2(y4.y, y4.y), w, acc[q + 1]);
                    acc[q + 2] = __ffma2_rn(make_float2(y4.z, y4.z), w, acc[q + 2]);
                    acc[q + 3] = __ffma2_rn(make_float2(y4.w, y4.w), w, acc[q + 3]);
                }
            }
        }
    }
}

// per-tile accumulators: FP64 for S <= 2, FP32 for S >= 4 (shared-memory
// budget; each term is already a partial over a run of views)
// one loop for both of a lane's pixel pairs (see cbp_bp_kernel)
#ifndef CBP_BP_EARLY  // A/B knob: chunk 0's headers and entries before the wait on the FP
#define CBP_BP_EARLY 1
#endif
#ifndef CBP_BP_UNION8  // A/B knob: 0 = two exact-window loops at S = 8 as well
#define CBP_BP_UNION8 1
#endif
template <int S>
constexpr bool BP_UNION = S == 8 && CBP_BP_UNION8;

// two pixel pairs over the same entries [jl, jh] (one set of shared loads,
// two independent weight chains)
template <int S, bool PAR = false>
__device__ __forceinline__ void bp_pair2(const BPEntry* row, const float* yrow, int jl, int jh, int base,
                                         float dc0, float dr0, float dc1, float dr1, float2 (&a0)[S],
                                         float2 (&a1)[S])
{
    if (jh < jl) return;
    CBP_CHECK(jl >= base && jh - base < 128, "bp_pair2 jl=%d jh=%d base=%d\n", jl, jh, base);
    const int cnt = jh - jl + 1;
    const BPEntry* e = row + (jl - base);
    const float* ys = yrow + (jl - base) * S;
    for (int k = 0; k < cnt; ++k, ++e, ys += S) {
        if constexpr (S == 1) {
            const float yw = e->c.w;
            const float2 w0 = bp_weight<PAR>(e, dc0, dr0), w1 = bp_weight<PAR>(e, dc1, dr1);
            a0[0] = __ffma2_rn(make_float2(yw, yw), w0, a0[0]);
            a1[0] = __ffma2_rn(make_float2(yw, yw), w1, a1[0]);
        } else {
            const float hA = e->c.w;
            const float2 w0 = __fmul2_rn(bp_weight<PAR>(e, dc0, dr0), make_float2(hA, hA));
            const float2 w1 = __fmul2_rn(bp_weight<PAR>(e, dc1, dr1), make_float2(hA, hA));
            if constexpr (S == 2) {
                const float2 y2 = *reinterpret_cast<const float2*>(ys);
                a0[0] = __ffma2_rn(make_float2(y2.x, y2.x), w0, a0[0]);
                a0[1] = __ffma2_rn(make_float2(y2.y, y2.y), w0, a0[1]);
                a1[0] = __ffma2_rn(make_float2(y2.x, y2.x), w1, a1[0]);
                a1[1] = __ffma2_rn(make_float2(y2.y, y2.y), w1, a1[1]);
            } else {
#pragma unroll
                for (int q = 0; q < S; q += 4) {
                    const float4 y4 = *reinterpret_cast<const float4*>(ys + q);
                    a0[q] = __ffma2_rn(make_float2(y4.x, y4.x), w0, a0[q]);
                    a0[q + 1] = __ffma2_rn(make_float2(y4.y, y4.y), w0, a0[q + 1]);
                    a0[q + 2] = __ffma2_rn(make_float2(y4.z, y4.z), w0, a0[q + 2]);
                    a0[q + 3] = __ffma2_rn(make_float2(y4.w, y4.w), w0, a0[q + 3]);
                    a1[q] = __ffma2_rn(make_float2(y4.x, y4.x), w1, a1[q]);
                    a1[q + 1] = __ffma2_rn(make_float2(y4.y, y4.y), w1, a1[q + 1]);
                    a1[q + 2] = __ffma2_rn(make_float2(y4.z, y4.z), w1, a1[q + 2]);
                    a1[q + 3] = __ffma2_rn(make_float2(y4.w, y4.w), w1, a1[q + 3]);
                }
            }
        }
    }
}

template <int S>
using bp_acc_t = typename std::conditional<(S >= 4), float, double>::type;

template <int S>
__device__ __forceinline__ void bp_flush(bp_acc_t<S>* acc_s, int horiz, int e0, int e1,
                                         float2 (&a0)[S], float2 (&a1)[S])
{
    constexpr int LD = BP_TILE + 1, PL = BP_TILE * LD;
    const int i0 = (e0 >> 5) * LD + (e0 & 31), i1 = (e1 >> 5) * LD + (e1 & 31);
    const int st = horiz ? 1 : LD;  // second pixel of a pair
#pragma unroll
    for (int q = 0; q < S; ++q) {
        acc_s[q * PL + i0] += (bp_acc_t<S>)a0[q].x;
        acc_s[q * PL + i0 + st] += (bp_acc_t<S>)a0[q].y;
        acc_s[q * PL + i1] += (bp_acc_t<S>)a1[q].x;
        acc_s[q * PL + i1 + st] += (bp_acc_t<S>)a1[q].y;
        a0[q] = a1[q] = make_float2(0.f, 0.f);
    }
}

// header buffers: S > 1 keeps three chunks of headers in flight (current,
// next, the one after), S == 1 one
__host__ __device__ constexpr int bp_hdr_bufs(int S) { return S > 1 ? 3 : 1; }

// Symmetry frames on pixel (r, c) of the n x n grid:
// g = R^q M^m with R(r, c) = (n-1-c, r) (+90 degrees) and M(r, c) = (n-1-r, c).
__device__ __forceinline__ void frame_fwd(int n, int q, int m, int& r, int& c)
{
    if (m) r = n - 1 - r;
    for (int t = 0; t < q; ++t) {
        const int nr = n - 1 - c;
        c = r;
        r = nr;
    }
}
__device__ __forceinline__ void frame_inv(int n, int q, int m, int& r, int& c)
{
    for (int t = 0; t < q; ++t) {  // R^-1 (r, c) = (c, n-1-r)
        const int nr = c;
        c = n - 1 - r;
        r = nr;
    }
    if (m) r = n - 1 - r;
}

// Orbit clusters.  With n = 32 T the 8 frames map tiles
// onto tiles: tile (ty, tx) -> frame_fwd(T, ...) on tile coordinates.  The
// orbit of a tile has 8, 4 (a diagonal tile: the transpose fixes it) or 1
// (the centre tile of an odd T) distinct tiles; its members are listed in
// frame order without repeats, identically by every CTA.
__device__ __forceinline__ int bp_orbit_members(int T, int2 rep, int (&mem)[8])
{
    int size = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        int r = rep.y, c = rep.x;
        frame_fwd(T, q & 3, q >> 2, r, c);
        const int t = r * T + c;
        bool seen = false;
        for (int i = 0; i < size; ++i) seen |= mem[i] == t;
        if (!seen) mem[size++] = t;
    }
    return size;
}

// dynamic shared memory of the BP kernel for S slices: entries, headers,
// (S > 1) two y buffers [2][VC][NB][S], tile accumulators [S][32][33]
__host__ __device__ constexpr size_t bp_smem_bytes(int S, bool prec = false, int W = 0)
{
    return (prec ? sizeof(BPEntryP) : sizeof(BPEntry)) * (W ? BPShape<1>::VC * BPShape<1>::NB : BP_VC * BP_NB) +
           sizeof(BPHeader) * (W ? BPShape<1>::VC : BP_VC) * bp_hdr_bufs(S) +
           (S > 1 ? 2 * sizeof(float) * (W ? BPShape<1>::VC * BPShape<1>::NB : BP_VC * BP_NB) * S : 0) +
           (S >= 4 ? sizeof(float) : sizeof(double)) * S * BP_TILE * (BP_TILE + 1);
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// S > 1: the raw y values of one chunk (views vl0 .. vl0 + nvc - 1 of this
// CTA, bins jlo + pass NB + jj of each, all S frames / slices) into
// ybuf[VC][NB][S] -- asynchronously (cp.async, overlapping the previous
// chunk's compute) or with plain loads (later passes of a wide bin range).
// Four .. sixteen threads per (view, slice) walk its bins.
template <int S, int W = 0>
__device__ __forceinline__ void bp_y_load(const BPParams& P, int vl0, int nvc, int pass,
                                          const BPHeader* H, float* ybuf, bool async)
{
    constexpr int BP_VC = BPShape<W>::VC, BP_NB = BPShape<W>::NB;
    const GeomDev& g = P.g;
    constexpr int TPC = BP_THREADS / (BP_VC * S);  // threads per (view, slice)
    static_assert(TPC >= 1 && BP_THREADS % (BP_VC * S) == 0, "BP_VC * S must divide the CTA");
    const int tid = threadIdx.x;
    const int combo = tid / TPC, sub = tid % TPC;
    const int vi = combo / S, q = combo % S;
    if (vi >= nvc) return;
    const BPHeader& h = H[vi];
    const int j0 = h.jlo + pass * BP_NB;
    const int cnt = min(h.jhi - j0 + 1, BP_NB);
    const int vl = vl0 + vi;
    const float* src = nullptr;
    int dir = 1;
    if (P.sym_mode == 8) {  // frame (qq, m) of base view v: view_g(v), bin_m(j)
        const int N = g.n_views, v = P.view_begin + vl, m = q >> 2, qq = q & 3;
        const size_t img = blockIdx.z / P.groups;  // image of the batch (slice group)
        int view = (m ? N - v : v) + qq * (N / 4);
        if (view >= N) view -= N;  // 0 <= v <= N/8
        if (!(m && (v == 0 || 8 * v == N))) {  // else the mirrored frame repeats a rotation: y = 0
            src = P.sino + (img * N + view) * g.n_det + (m ? g.n_det - 1 - j0 : j0);
            dir = m ? -1 : 1;
        }
    } else if (P.sym_stride > 0) {
        src = P.sino + ((size_t)q * P.sym_stride + vl) * g.n_det + j0;
    } else {
        const int b = blockIdx.z / P.groups * S + q;
        if (b < P.batch) src = P.sino + ((size_t)b * P.view_count + vl) * g.n_det + j0;
    }
    float* dst = ybuf + (size_t)vi * BP_NB * S + q;
    for (int jj = sub; jj < cnt; jj += TPC) {
        CBP_CHECK(j0 + jj >= 0 && j0 + jj < g.n_det, "y_load j=%d\n", j0 + jj);
        if (!src)
            dst[jj * S] = 0.0f;
        else if (async)
            cp_async4(dst + jj * S, src + dir * jj);
        else
            dst[jj * S] = __ldg(src + dir * jj);
    }
}

// The orbit cluster's epilogue: every CTA of the cluster holds the 8 frame
// accumulators of its member tile; output tile U (member rank mod size) is
// the sum, over the cluster's CTAs i and the frames q with g_q(S_i) = U, of
// CTA i's frame q read through distributed shared memory in U's orientation
// -- in (i, q) order, so the result is deterministic, with no partial frame
// planes and no reduce kernel.  A member tile shared by 8 / size CTAs (a
// smaller orbit) has its rows split among them.  Output: the image (one view
// group; accumulate adds), the multicast image (mc_fused: red.add), or the
// group's partial plane [images][groups] (cbp_reduce_kernel sums the groups).
__device__ void bp_orbit_epilogue(const BPParams& P, float* acc_s, const int (&mem)[8], int size, int grp, int sg)
{
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int LD = BP_TILE + 1, PL = BP_TILE * LD;
    const int T = P.orbit_T, n = P.g.n, tid = threadIdx.x;
    const int rank = (int)cluster.block_rank();
    const int U = mem[rank % size], ur = U / T, uc = U % T;
    const int parts = 8 / size, part = rank / size;
    const int rlo = part * (BP_TILE / parts), rhi = rlo + BP_TILE / parts;
    __shared__ int4 contrib[64];  // (cluster rank i, base index in its acc_s, col step, row step)
    __shared__ int ncontrib;
    if (tid == 0) {
        int k = 0;
        for (int i = 0; i < 8; ++i) {
            const int S0 = mem[i % size], sr0 = (S0 / T) * BP_TILE, sc0 = (S0 % T) * BP_TILE;
            for (int q = 0; q < 8; ++q) {
                int tr = S0 / T, tc = S0 % T;
                frame_fwd(T, q & 3, q >> 2, tr, tc);
                if (tr * T + tc != U) continue;
                // source pixel of output pixels (ur 32, uc 32) + {(0, 0), (0, 1), (1, 0)}
                int k0r = ur * BP_TILE, k0c = uc * BP_TILE, k1r = k0r, k1c = k0c + 1, k2r = k0r + 1, k2c = k0c;
                frame_inv(n, q & 3, q >> 2, k0r, k0c);
                frame_inv(n, q & 3, q >> 2, k1r, k1c);
                frame_inv(n, q & 3, q >> 2, k2r, k2c);
                contrib[k++] = make_int4(i, q * PL + (k0r - sr0) * LD + (k0c - sc0), (k1r - k0r) * LD + (k1c - k0c),
                                         (k2r - k0r) * LD + (k2c - k0c));
            }
        }
        ncontrib = k;
    }
    cluster.sync();  // every CTA's accumulators are final (and contrib is ready)
    const int nc = ncontrib;
    const size_t plane = (size_t)n * n;
    float* out = P.groups > 1 && !P.mc_fused ? P.out + ((size_t)sg * P.groups + grp) * plane
                                             : P.out + (size_t)sg * plane;
    const bool add = P.groups == 1 && P.accumulate;
    for (int i = tid; i < (rhi - rlo) * (BP_TILE / 4); i += BP_THREADS) {
        const int r = rlo + i / (BP_TILE / 4), c = (i % (BP_TILE / 4)) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k = 0; k < nc; ++k) {
            const int4 cb = contrib[k];
            const float* a = cluster.map_shared_rank(acc_s, cb.x);
            const int si = cb.y + r * cb.w + c * cb.z;
            v.x += a[si];
            v.y += a[si + cb.z];
            v.z += a[si + 2 * cb.z];
            v.w += a[si + 3 * cb.z];
        }
        float4* o = reinterpret_cast<float4*>(out + (size_t)(ur * BP_TILE + r) * n + uc * BP_TILE + c);
        if (P.mc_fused) {
            mc_red_add4(o, v);
        } else {
            if (add) {
                const float4 w = *o;
                v.x += w.x;
                v.y += w.y;
                v.z += w.z;
                v.w += w.w;
            }
            *o = v;
        }
    }
    cluster.sync();  // the other CTAs' reads of this CTA's accumulators are done
}

// One CTA's work on one tile over views [vg0, vg0 + vgn) of the launch (view
// group grp, slice group sg; seg: the segment of a persistent launch).
template <int S, bool PREC, bool ORB, bool SEG, int W = 0, bool PAR = false>
__device__ __forceinline__ void bp_body(const BPParams& P, int tile_x, int tile_y, int tiles_x, int vg0, int vgn,
                                        int grp, int sg, int seg, const int (&omem)[8], int osize)
{
    constexpr int BP_VC = BPShape<W>::VC, BP_NB = BPShape<W>::NB;  // the chunk shape
    static_assert(!PREC || S == 1, "the precise mode runs one slice per weight");
    static_assert(!ORB || (S == 8 && !PREC), "orbit clusters carry the 8 dihedral frames");
    using Ent = typename std::conditional<PREC, BPEntryP, BPEntry>::type;
    constexpr bool STAGE = S > 1;  // y staged asynchronously one chunk ahead
    constexpr int HB = bp_hdr_bufs(S);
    extern __shared__ __align__(16) unsigned char smem[];
    Ent(*tab)[BP_NB] = reinterpret_cast<Ent(*)[BP_NB]>(smem);
    BPHeader* hdr_all = reinterpret_cast<BPHeader*>(smem + sizeof(Ent) * BP_VC * BP_NB);  // [HB][VC]
    float* ytab_all = reinterpret_cast<float*>(hdr_all + HB * BP_VC);  // [2][VC][NB][S] (S > 1)
    bp_acc_t<S>* acc_s = reinterpret_cast<bp_acc_t<S>*>(
        smem + bp_smem_bytes(S, PREC, W) - sizeof(bp_acc_t<S>) * S * BP_TILE * (BP_TILE + 1));

    const GeomDev& g = P.g;
    const int tid = threadIdx.x;
    const int col0 = tile_x * BP_TILE, row0 = tile_y * BP_TILE;
    const int nchunks = (vgn + BP_VC - 1) / BP_VC;
    float hcx, hcy;  // anchor k_a = centre of the tile's valid pixels
    double kax, kay;
    bp_tile_anchor(g, tile_x, tile_y, hcx, hcy, kax, kay);
    const BPHeader* hsrc = P.hdrs + ((size_t)tile_y * tiles_x + tile_x) * P.view_count + vg0;
    const size_t sino_plane = (size_t)P.view_count * g.n_det;
    constexpr int HW = sizeof(BPHeader) / 16;  // 16-byte words per header
    auto hdr_buf = [&](int c) { return hdr_all + (c % HB) * BP_VC; };
    auto y_buf = [&](int c) { return ytab_all + (c & 1) * (BP_VC * BP_NB * S); };
    auto hdr_copy = [&](int c) {  // chunk c's headers (async)
        const int nvc = min(BP_VC, vgn - c * BP_VC);
        if (tid < nvc * HW)
            cp_async16(reinterpret_cast<int4*>(hdr_buf(c)) + tid, reinterpret_cast<const int4*>(hsrc + c * BP_VC) + tid);
    };

    // the S entries of chunk views vc .. vc + nvc - 1, pass `pass`, into tab
    auto build_entries = [&](const BPHeader* hdr, int vc, int nvc, int pass) {
#pragma unroll 3
        for (int e = tid; e < BP_VC * BP_NB; e += BP_THREADS) {
            const int vi = e / BP_NB, jj = e % BP_NB;
            if (vi < nvc) {
                const BPHeader& H = hdr[vi];
                const int j = H.jlo + pass * BP_NB + jj;
                CBP_CHECK(j > H.jhi || (j >= 0 && j < g.n_det), "entry j=%d jlo=%d jhi=%d\n", j, H.jlo, H.jhi);
                if (j <= H.jhi) {
                    if constexpr (PREC) {
                        const size_t yo = (size_t)(vg0 + vc + vi) * g.n_det + j;
                        bp_build_entry_prec(g, P.t, H, j, __ldg(P.sino + (size_t)sg * sino_plane + yo),
                                            tab[vi][jj]);
                    } else if constexpr (S == 1) {
                        const size_t yo = (size_t)(vg0 + vc + vi) * g.n_det + j;
                        bp_build_entry<PAR>(g, P.t, H, j, __ldg(P.sino + (size_t)sg * sino_plane + yo),
                                            tab[vi][jj]);
                    } else {
                        bp_build_entry<PAR>(g, P.t, H, j, 1.0f, tab[vi][jj]);  // c.w = h^2 / A
                    }
                }
            }
        }
    };

    for (int i = tid; i < S * BP_TILE * (BP_TILE + 1); i += BP_THREADS) acc_s[i] = 0;
    // staged BP with cached headers: chunk 0's headers and entries (geometry
    // only) before the wait on the FP, so they overlap its tail
    const bool early = STAGE && !SEG && CBP_BP_EARLY && P.hdr_ready && nchunks > 0;
    if (early) {
        hdr_copy(0);
        if (nchunks > 1) hdr_copy(1);
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
        build_entries(hdr_buf(0), 0, min(BP_VC, vgn), 0);
    }
    if constexpr (!SEG) {
        griddep_launch_dependents();  // the reduce may launch into this grid's tail
        griddep_wait();               // the sinogram, headers and pool memory are ready
    }

    if constexpr (STAGE) {
        if (nchunks > 0) {
            if (!early) {
                hdr_copy(0);
                if (nchunks > 1) hdr_copy(1);
                cp_async_commit();
                cp_async_wait_all();
                __syncthreads();
            }
            bp_y_load<S, W>(P, vg0, min(BP_VC, vgn), 0, hdr_buf(0), y_buf(0), true);
            cp_async_commit();
        }
    }
    // the thread's two pixel pairs (their order depends on the ray-direction
    // bucket) and their FP32 partial sums, carried across chunks and flushed
    // to acc_s when the bucket changes, every BP_RUN_CHUNKS chunks and at the end
    float2 a0[S], a1[S];
#pragma unroll
    for (int q = 0; q < S; ++q) a0[q] = a1[q] = make_float2(0.f, 0.f);
    int bucket = -1, horiz = 1, e0 = 0, e1 = 0, prev_npass = 1;
    float2 dc0, dr0, dc1, dr1;  // pixel offsets of the two pairs (lanes a, b)
    for (int c = 0; c < nchunks; ++c) {
        const int vc = c * BP_VC;
        const int nvc = min(BP_VC, vgn - vc);
        BPHeader* hdr = hdr_buf(c);
        float* ytab = y_buf(c);
        if constexpr (STAGE) {
            // chunk c's headers and y, chunk c+1's headers have landed, and every
            // thread is done with chunk c-1 (whose buffers are refilled next)
            cp_async_wait_all();
            __syncthreads();
            if (c + 2 < nchunks) hdr_copy(c + 2);
            if (c + 1 < nchunks)
                bp_y_load<S, W>(P, vg0 + vc + BP_VC, min(BP_VC, vgn - vc - BP_VC), 0, hdr_buf(c + 1), y_buf(c + 1),
                             true);
            cp_async_commit();
        } else {
            // the single header buffer is rewritten here: every thread must be done
            // reading the previous chunk's headers.  A chunk with passes ends in a
            // barrier; one whose views all miss the tile (npass = 0: a tile the
            // detector does not cover for those views) does not -- without this
            // barrier a fast thread overwrote the headers a slow one was still
            // reading (found by tools/fuzz.py wide seeds 139 and 2189: ragged edge
            // tiles outside the detector, one slice per weight)
            if (c > 0 && prev_npass == 0) __syncthreads();
            if (tid < nvc * HW)
                reinterpret_cast<int4*>(hdr)[tid] = __ldg(reinterpret_cast<const int4*>(hsrc + vc) + tid);
            __syncthreads();
        }
        int npass = 0;
        for (int vi = 0; vi < nvc; ++vi)  // passes of BP_NB bins (the header's npass_f is for the default shape)
            npass = max(npass, W == 0 ? (int)hdr[vi].npass_f
                                      : (hdr[vi].jhi >= hdr[vi].jlo ? (hdr[vi].jhi - hdr[vi].jlo) / BP_NB + 1 : 0));
        prev_npass = npass;
        for (int pass = 0; pass < npass; ++pass) {
            if (STAGE && pass > 0) bp_y_load<S, W>(P, vg0 + vc, nvc, pass, hdr, ytab, false);
            if (!(early && c == 0 && pass == 0)) build_entries(hdr, vc, nvc, pass);
            __syncthreads();
            for (int vi = 0; vi < nvc; ++vi) {
                const BPHeader& H = hdr[vi];
                const int4 hi = *reinterpret_cast<const int4*>(&H.ja);  // ja, jlo, jhi, bucket
                // new pair order, or FP32 register sums over BP_RUN views: hand the pixels back
                // (S >= 4: the tile accumulator is FP32 too, so periodic flushes buy no
                // precision -- measured config 5 BP 9.69 -> 9.46 ms without them)
                const bool renew = hi.w != bucket ||
                                   (S <= 2 && vi == 0 && pass == 0 && c > 0 && c % BP_RUN_CHUNKS == 0);
                if (renew) {
                    if (bucket >= 0) {
                        bp_flush<S>(acc_s, horiz, e0, e1, a0, a1);
                        __syncthreads();
                    }
                    bucket = hi.w;
                    horiz = bucket_horiz(bucket);
                    // the lane's two pairs are neighbours in the lateral order: nearly the
                    // same bins, so one loop over the union of their ranges serves both
                    // (only at S = 8, measured: S = 4 spills under its 3-CTA register
                    // budget, S = 1 is 3% slower; they keep two loops with pairs 32 apart)
                    constexpr int PSTEP = BP_UNION<S> ? 1 : 32;
                    const uint16_t* order = P.pairs + bucket * BP_PAIRS + (tid >> 5) * 64 +
                                            (BP_UNION<S> ? 2 * (tid & 31) : (tid & 31));
                    CBP_CHECK(bucket >= 0 && bucket < BP_BUCKETS, "bucket %d\n", bucket);
                    e0 = __ldg(order);
                    e1 = __ldg(order + PSTEP);
                    const float sx = horiz ? 1.0f : 0.0f, sy = 1.0f - sx;  // pair step (dc, dr)
                    const float c0 = (float)(e0 & 31) - hcx, r0 = (float)(e0 >> 5) - hcy;
                    const float c1 = (float)(e1 & 31) - hcx, r1 = (float)(e1 >> 5) - hcy;
                    dc0 = make_float2(c0, c0 + sx);
                    dr0 = make_float2(r0, r0 + sy);
                    dc1 = make_float2(c1, c1 + sx);
                    dr1 = make_float2(r1, r1 + sy);
                }
                const int base = hi.y + pass * BP_NB;
                if (base > hi.z) continue;
                const Ent* row = tab[vi];
                const float* yrow = ytab + vi * BP_NB * S;
                const float4 hf = *reinterpret_cast<const float4*>(&H.urel);  // urel, nx, ny, cW
                const float4 hd = *reinterpret_cast<const float4*>(&H.dena);  // dena, dx, dy, -
                const int jmax = min(hi.z, base + BP_NB - 1);
                int jl2 = 1 << 30, jh2 = -(1 << 30);
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const float2 dcp = p ? dc1 : dc0, drp = p ? dr1 : dr0;
                    // exact bin coordinates of the two pixels, and their support bounds
                    const float2 num = __ffma2_rn(drp, make_float2(hf.z, hf.z),
                                                  __fmul2_rn(dcp, make_float2(hf.y, hf.y)));
                    const float2 den = __ffma2_rn(drp, make_float2(hd.z, hd.z),
                                                  __ffma2_rn(dcp, make_float2(hd.y, hd.y),
                                                             make_float2(hd.x, hd.x)));
                    const float2 inv = rcp2(den);
                    const float2 u = __ffma2_rn(num, inv, make_float2(hf.x, hf.x));
                    const float2 w = __ffma2_rn(make_float2(hf.w, hf.w), inv, make_float2(2e-3f, 2e-3f));
                    // clamp before the integer conversion: pixels of a ragged tile that lie
                    // outside the image can give inf / NaN here (their sums are discarded)
                    const float lo = fmaxf(fminf(fminf(u.x - w.x, u.y - w.y), 1e6f), -1e6f);
                    const float hi2 = fmaxf(fminf(fmaxf(u.x + w.x, u.y + w.y), 1e6f), -1e6f);
                    const int jl = max(hi.x + __float2int_rd(lo) + 1, base);
                    const int jh = min(hi.x + __float2int_ru(hi2) - 1, jmax);
                    if constexpr (PREC) {
                        bp_pair_prec(row, jl, jh, base, dcp, drp, p ? a1[0] : a0[0]);
                    } else if constexpr (BP_UNION<S>) {
                        jl2 = min(jl2, jl);
                        jh2 = max(jh2, jh);
                    } else if (p == 0) {
                        bp_pair<S, PAR>(row, yrow, jl, jh, base, dcp.x, drp.x, a0);
                    } else {
                        bp_pair<S, PAR>(row, yrow, jl, jh, base, dcp.x, drp.x, a1);
                    }
                }
                // both pairs over the union (weights outside a pixel's support are exactly 0)
                if constexpr (BP_UNION<S>)
                    bp_pair2<S, PAR>(row, yrow, jl2, jh2, base, dc0.x, dr0.x, dc1.x, dr1.x, a0, a1);
            }
            // the next pass rebuilds tab (the next chunk's top barrier covers S > 1)
            if (!STAGE || pass + 1 < npass) __syncthreads();
        }
    }
    if (bucket >= 0) bp_flush<S>(acc_s, horiz, e0, e1, a0, a1);
    if constexpr (STAGE) {
        cp_async_wait_all();
        __syncthreads();
    }
    if constexpr (ORB) {
        bp_orbit_epilogue(P, acc_s, omem, osize, grp, sg);
        return;
    }

    // Write the tile's sums.  With symmetry, slice q holds frame g_q = R^qq M^m
    // of the image; its values go straight to the output orientation (pixel
    // g_q(k)), so the partial planes are summed elementwise (cbp_reduce_kernel).
    // Threads walk the OUTPUT rectangle g_q(tile) row by row (coalesced
    // stores; the transposed shared-memory reads are conflict-free with the
    // 33-float row pitch).
    const int n = g.n;
    const size_t plane = (size_t)n * n;
    const int th = min(BP_TILE, n - row0), tw = min(BP_TILE, n - col0);
    const int fsym = P.sym_mode == 8 ? 8 : (P.sym_stride > 0 ? 4 : 0);
    constexpr int LD = BP_TILE + 1;
    __shared__ int4 ep[S][2];  // per slice: (OR, OC, oh, ow), (s0, sc, sr, -)
    if (tid < S) {
        const int q = tid;
        const int qq = fsym ? (q & 3) : 0, m = (fsym == 8 && q >= 4) ? 1 : 0;
        int ra = row0, ca = col0, rb = row0 + th - 1, cb = col0 + tw - 1;
        frame_fwd(n, qq, m, ra, ca);
        frame_fwd(n, qq, m, rb, cb);
        const int OR = min(ra, rb), OC = min(ca, cb);
        // tile pixel of output (OR, OC) and its step per output column / row
        int k0r = OR, k0c = OC, k1r = OR, k1c = OC + 1, k2r = OR + 1, k2c = OC;
        frame_inv(n, qq, m, k0r, k0c);
        frame_inv(n, qq, m, k1r, k1c);
        frame_inv(n, qq, m, k2r, k2c);
        ep[q][0] = make_int4(OR, OC, abs(ra - rb) + 1, abs(ca - cb) + 1);
        ep[q][1] = make_int4((k0r - row0) * LD + (k0c - col0), (k1r - k0r) * LD + (k1c - k0c),
                             (k2r - k0r) * LD + (k2c - k0c), 0);
    }
    __syncthreads();
    for (int q = 0; q < S; ++q) {
        const int b = fsym ? q : sg * S + q;
        if (b >= P.batch) break;
        // symmetric frames: plane (sg groups + grp) frames + q; batch: (grp batch + b)
        const size_t pi = fsym ? ((size_t)sg * P.groups + grp) * P.batch + q
                               : (P.groups > 1 ? (size_t)grp * P.batch + b : (size_t)b);
        // fused multicast reduction: every frame of every view group adds into the image
        float* out = P.mc_fused ? P.out + (fsym ? (size_t)sg : (size_t)b) * plane : P.out + pi * plane;
        const int4 e0 = ep[q][0], e1 = ep[q][1];
        const int OR = e0.x, OC = e0.y, oh = e0.z, ow = e0.w, s0 = e1.x, sc = e1.y, sr = e1.z;
        // the rectangle's origin and row pitch: the image, or (a persistent launch)
        // the segment's compact block [q][oh][ow], also in output orientation
        size_t pitch = n;
        float* dst = out + (size_t)OR * n + OC;
        if (SEG && !P.mc_fused) {
            pitch = ow;
            dst = P.out + (((size_t)sg * P.seg_max + seg) * S + q) * (BP_TILE * BP_TILE);
        }
        const bp_acc_t<S>* a = acc_s + q * BP_TILE * LD;
        const bool acc_out = P.groups == 1 && P.accumulate && !SEG;
        if (oh == BP_TILE && ow == BP_TILE && (pitch & 3) == 0 && !acc_out) {  // float4 stores
            for (int i = tid; i < BP_TILE * BP_TILE / 4; i += BP_THREADS) {
                const int r = i / (BP_TILE / 4), c = (i % (BP_TILE / 4)) * 4;
                const int si = s0 + r * sr + c * sc;
                const float4 v = make_float4((float)a[si], (float)a[si + sc], (float)a[si + 2 * sc],
                                             (float)a[si + 3 * sc]);
                float4* o = reinterpret_cast<float4*>(dst + r * pitch + c);
                if (P.mc_fused)
                    mc_red_add4(o, v);
                else
                    *o = v;
            }
        } else {
            for (int i = tid; i < BP_TILE * BP_TILE; i += BP_THREADS) {
                const int r = i / BP_TILE, c = i % BP_TILE;
                if (r < oh && c < ow) {
                    float* o = dst + r * pitch + c;
                    const float v = (float)a[s0 + r * sr + c * sc];
                    if (P.mc_fused)
                        mc_red_add(o, v);
                    else
                        *o = acc_out ? *o + v : v;
                }
            }
        }
    }
}

template <int S, bool PREC = false, bool ORB = false, bool SEG = false, int W = 0, bool PAR = false>
__global__ void __launch_bounds__(BP_THREADS, S == 1 ? 4 : (S == 4 ? 3 : 2)) cbp_bp_kernel(const BPParams P)
{
    int omem[8], osize = 1;
#ifdef CBP_BP_PROFILE
    const unsigned long long t_start = P.prof ? globaltimer() : 0;
    unsigned long long f_bins = 0, f_cov = 0, f_views = 0;  // the CTA's header features
    auto prof_feat = [&](int tile, int v0, int len) {
        if (P.prof && threadIdx.x == 0)
            for (int v = v0; v < v0 + len; ++v) {
                const BPHeader& H = P.hdrs[(size_t)tile * P.view_count + v];
                ++f_views;
                if (H.npass_f > 0.0f) {
                    ++f_cov;
                    f_bins += H.jhi - H.jlo + 1;
                }
            }
    };
    auto prof_end = [&](int segs) {
        if (P.prof && threadIdx.x == 0) {
            const size_t cta = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
            unsigned long long* r = P.prof + 8 * cta;
            r[0] = t_start;
            r[1] = globaltimer();
            r[2] = smid();
            r[3] = segs;
            r[4] = f_bins;
            r[5] = f_cov;
            r[6] = f_views;
        }
    };
#else
    auto prof_feat = [](int, int, int) {};
    auto prof_end = [](int) {};
#endif
    if constexpr (SEG) {
        static_assert(!ORB, "segments and orbit clusters are separate launch modes");
        griddep_launch_dependents();  // the reduce may launch into this grid's tail
        griddep_wait();               // the sinogram, headers, plan and pool memory are ready
        const int tiles_x = (P.g.n + BP_TILE - 1) / BP_TILE;
        const int s0 = P.cta_seg[blockIdx.x], s1 = P.cta_seg[blockIdx.x + 1];
        for (int s = s0; s < s1; ++s) {
            const int i0 = P.seg_idx[s], len = P.seg_idx[s + 1] - i0;
            const int tile = i0 / P.view_count, v0 = i0 - tile * P.view_count;
            if (s > s0) __syncthreads();  // the previous segment's epilogue is done with acc_s
            prof_feat(tile, v0, len);
            bp_body<S, PREC, ORB, SEG, W>(P, tile % tiles_x, tile / tiles_x, tiles_x, v0, len, 0, blockIdx.z, s,
                                          omem, osize);
        }
        prof_end(s1 - s0);
        return;
    }
    const int grp = blockIdx.z % P.groups, sg = blockIdx.z / P.groups;  // view group, slice group
    int vg0 = grp * P.views_per_group;
    int vgn = max(0, min(P.views_per_group, P.view_count - vg0));
    int tile_x = blockIdx.x, tile_y = blockIdx.y, tiles_x = gridDim.x;
    if constexpr (ORB) {
        // cluster rank r takes orbit member r mod size over part r / size of the
        // group's views (8 / size parts: a smaller orbit splits its views)
        tiles_x = P.orbit_T;
        osize = bp_orbit_members(P.orbit_T, P.orbit_reps[blockIdx.x / 8], omem);
        const int rank = blockIdx.x % 8, parts = 8 / osize, part = rank / osize;
        tile_x = omem[rank % osize] % tiles_x;
        tile_y = omem[rank % osize] / tiles_x;
        const int per = (vgn + parts - 1) / parts;
        vg0 += part * per;
        vgn = max(0, min(per, vgn - part * per));
    }
    if (!ORB) prof_feat(tile_y * tiles_x + tile_x, vg0, vgn);
    bp_body<S, PREC, ORB, SEG, W, PAR>(P, tile_x, tile_y, tiles_x, vg0, vgn, grp, sg, 0, omem, osize);
    prof_end(1);
}

// ---- the persistent BP's plan (per geometry and view range, cached with the
// headers).  Estimated cost of tile t, view v: the bins of its range plus a
// fixed per-view share (set-up, window, barriers), in bin units; a view that
// misses the tile costs little.
constexpr int BP_PLAN_VIEW = 12, BP_PLAN_MISS = 2;

__device__ __forceinline__ int bp_plan_cost(const BPHeader& H)
{
    return H.npass_f > 0.0f ? H.jhi - H.jlo + 1 + BP_PLAN_VIEW : BP_PLAN_MISS;
}

// one CTA per tile: cum[t][v] = inclusive prefix of the tile's view costs,
// tot[t] = the tile's total
__global__ void __launch_bounds__(256) cbp_bp_plan_cost_kernel(const BPHeader* __restrict__ hdrs, int nv,
                                                               int* __restrict__ cum, long long* __restrict__ tot)
{
    __shared__ int part[256];
    __shared__ int carry;
    const int t = blockIdx.x, tid = threadIdx.x;
    if (tid == 0) carry = 0;
    for (int v0 = 0; v0 < nv; v0 += 256) {
        const int v = v0 + tid;
        int c = v < nv ? bp_plan_cost(hdrs[(size_t)t * nv + v]) : 0;
        part[tid] = c;
        __syncthreads();
        for (int off = 1; off < 256; off <<= 1) {  // Hillis-Steele inclusive scan
            const int add = tid >= off ? part[tid - off] : 0;
            __syncthreads();
            part[tid] += add;
            __syncthreads();
        }
        if (v < nv) cum[(size_t)t * nv + v] = carry + part[tid];
        __syncthreads();
        if (tid == 255) carry += part[255];
        __syncthreads();
    }
    if (tid == 0) tot[t] = carry;
}

// one CTA: the segments of an NB-CTA persistent launch.  plan layout (ints):
// seg_idx[tiles + NB + 1] | cta_seg[NB + 1] | seg_first[tiles + 1] | D[NB] | starts[NB + 1]
// with pre[tiles + 1] (int64) the tiles' exclusive cost prefix.
__global__ void __launch_bounds__(1024) cbp_bp_plan_kernel(const int* __restrict__ cum, long long* __restrict__ pre,
                                                           int tiles, int nv, int NB, int* __restrict__ plan)
{
    int* seg_idx = plan;
    int* cta_seg = seg_idx + tiles + NB + 1;
    int* seg_first = cta_seg + NB + 1;
    int* D = seg_first + tiles + 1;
    int* starts = D + NB;
    __shared__ long long ssum[1024];
    __shared__ int nD;
    const int tid = threadIdx.x;
    // 1. exclusive prefix of the tile totals (pre holds the totals on entry)
    const int per = (tiles + 1023) / 1024, a = min(tiles, tid * per), b = min(tiles, a + per);
    long long s = 0;
    for (int i = a; i < b; ++i) s += pre[i];
    ssum[tid] = s;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const long long add = tid >= off ? ssum[tid - off] : 0;
        __syncthreads();
        ssum[tid] += add;
        __syncthreads();
    }
    long long run = ssum[tid] - s;
    for (int i = a; i < b; ++i) {
        const long long v = pre[i];
        pre[i] = run;
        run += v;
    }
    if (tid == 1023) pre[tiles] = ssum[1023];
    __syncthreads();
    const long long total = pre[tiles];
    const int T = tiles * nv;
    // 2. CTA b starts at the (tile, view) whose cost interval holds b total / NB
    for (int bb = tid; bb < NB; bb += 1024) {
        const long long target = (long long)bb * total / NB;
        int lo = 0, hi = tiles - 1;  // last tile with pre[t] <= target
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pre[mid] <= target) lo = mid; else hi = mid - 1;
        }
        const long long local = target - pre[lo];
        int vl = 0, vh = nv - 1;  // first view with cum > local
        const int* c = cum + (size_t)lo * nv;
        while (vl < vh) {
            const int mid = (vl + vh) >> 1;
            if (c[mid] > local) vh = mid; else vl = mid + 1;
        }
        starts[bb] = lo * nv + vl;
    }
    if (tid == 0) starts[NB] = T;
    __syncthreads();
    // 3. D = the distinct CTA starts inside a tile (tile starts are boundaries anyway)
    if (tid == 0) {
        int k = 0;
        for (int bb = 0; bb < NB; ++bb) {
            const int x = starts[bb];
            if (x % nv != 0 && (k == 0 || D[k - 1] != x)) D[k++] = x;
        }
        nD = k;
    }
    __syncthreads();
    const int nd = nD, nseg = tiles + nd;
    auto below = [&](int x) {  // #{d in D : d < x}
        int l = 0, h = nd;
        while (l < h) {
            const int m = (l + h) >> 1;
            if (D[m] < x) l = m + 1; else h = m;
        }
        return l;
    };
    for (int t = tid; t < tiles; t += 1024) {
        const int r = t + below(t * nv);
        seg_idx[r] = t * nv;
        seg_first[t] = r;
    }
    for (int i = tid; i < nd; i += 1024) seg_idx[(D[i] + nv - 1) / nv + i] = D[i];
    for (int bb = tid; bb < NB; bb += 1024) {
        const int x = starts[bb];
        cta_seg[bb] = (x + nv - 1) / nv + below(x);
    }
    if (tid == 0) {
        seg_idx[nseg] = T;
        cta_seg[NB] = nseg;
        seg_first[tiles] = nseg;
    }
}

// out[image][p] (+)= sum over frames q (fixed order) and the segments of the
// tile holding k = g_q^-1(p) (in order) of block[image][seg][q] at p: the
// persistent BP's reduction, deterministic.  Blocks are in output orientation
// (g_q of the tile's rectangle, row pitch = its width).  n a multiple of
// BP_TILE (frames map tiles onto tiles): one CTA per output tile, float4 rows;
// else one thread per pixel (cbp_seg_reduce_px_kernel).  S = 8: the dihedral
// frames.  mode 1 adds to out, 2 adds through a multicast address.
template <int S>
__global__ void __launch_bounds__(256) cbp_seg_reduce_kernel(const float* __restrict__ blocks, float* __restrict__ out,
                                                             const int* __restrict__ seg_first, int n, int seg_max,
                                                             int accumulate)
{
    griddep_wait();  // the BP's blocks
    constexpr int TT = BP_TILE * BP_TILE;
    const int T = n / BP_TILE, U = blockIdx.x, ur = U / T, uc = U % T, tid = threadIdx.x;
    __shared__ int2 segs[S];
    if (tid < S) {
        int tr = ur, tc = uc;  // the source tile of frame q on the T x T tile grid
        if constexpr (S == 8) frame_inv(T, tid & 3, tid >> 2, tr, tc);
        const int t = tr * T + tc;
        segs[tid] = make_int2(__ldg(seg_first + t), __ldg(seg_first + t + 1));
    }
    __syncthreads();
    blocks += (size_t)blockIdx.y * seg_max * S * TT;
    out += (size_t)blockIdx.y * n * n;
    const int r = tid / (BP_TILE / 4), c = (tid % (BP_TILE / 4)) * 4;  // 256 threads x 4 pixels
    float4* o = reinterpret_cast<float4*>(out + (size_t)(ur * BP_TILE + r) * n + uc * BP_TILE + c);
    float4 v = accumulate == 1 ? *o : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < S; ++q) {
        const int2 sr = segs[q];
        for (int s = sr.x; s < sr.y; ++s) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(blocks + ((size_t)s * S + q) * TT) + tid);
            v.x += b.x;
            v.y += b.y;
            v.z += b.z;
            v.w += b.w;
        }
    }
    if (accumulate == 2)
        mc_red_add4(o, v);
    else
        *o = v;
}

template <int S>
__global__ void __launch_bounds__(256) cbp_seg_reduce_px_kernel(const float* __restrict__ blocks,
                                                                float* __restrict__ out,
                                                                const int* __restrict__ seg_first, int n,
                                                                int seg_max, int accumulate)
{
    griddep_wait();  // the BP's blocks
    constexpr int TT = BP_TILE * BP_TILE;
    const int tiles_x = (n + BP_TILE - 1) / BP_TILE;
    const size_t plane = (size_t)n * n;
    blocks += (size_t)blockIdx.y * seg_max * S * TT;
    out += (size_t)blockIdx.y * plane;
    for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < plane; p += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(p / n), c = (int)(p % n);
        float v = accumulate == 1 ? out[p] : 0.0f;
#pragma unroll
        for (int q = 0; q < S; ++q) {
            int kr = r, kc = c;
            const int qq = S == 8 ? (q & 3) : 0, m = S == 8 ? (q >> 2) : 0;
            frame_inv(n, qq, m, kr, kc);
            const int tr = kr / BP_TILE, tc = kc / BP_TILE;
            // g_q of the source tile's rectangle: origin and width (as the BP's epilogue)
            const int row0 = tr * BP_TILE, col0 = tc * BP_TILE;
            int ra = row0, ca = col0, rb = min(row0 + BP_TILE, n) - 1, cb = min(col0 + BP_TILE, n) - 1;
            frame_fwd(n, qq, m, ra, ca);
            frame_fwd(n, qq, m, rb, cb);
            const int off = q * TT + (r - min(ra, rb)) * (abs(ca - cb) + 1) + (c - min(ca, cb));
            const int t = tr * tiles_x + tc, s1 = __ldg(seg_first + t + 1);
            for (int s = __ldg(seg_first + t); s < s1; ++s) v += __ldg(blocks + (size_t)s * S * TT + off);
        }
        if (accumulate == 2)
            mc_red_add(out + p, v);
        else
            out[p] = v;
    }
}

// out[p] = (mode 1 ? out[p] : 0) + sum_g part[g][p] over `groups` planes
// of `count` floats, fixed order (deterministic); float4 when aligned
// (blockIdx.y selects one of gridDim.y independent outputs: part + y groups count,
// out + y count).  mode 2: out is a multicast address and the sum is ADDED
// to every rank's copy by multimem.red (the view-sharded all-reduce of row a7
// fused into the BP's last kernel; order across ranks is the switch's).
#ifndef CBP_REDUCE_QUAD  // A/B knob: four lanes per float4 when there are many planes
#define CBP_REDUCE_QUAD 1
#endif
__global__ void cbp_reduce_kernel(const float* __restrict__ part, float* __restrict__ out,
                                  size_t count, int groups, int accumulate)
{
    griddep_wait();  // the BP's partial planes
    part += (size_t)blockIdx.y * groups * count;
    out += (size_t)blockIdx.y * count;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t t0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const bool aligned =
        ((count & 3) | (reinterpret_cast<uintptr_t>(part) & 15) | (reinterpret_cast<uintptr_t>(out) & 15)) == 0;
    if (aligned && CBP_REDUCE_QUAD && groups >= 16 && groups % 32 == 0) {
        // many planes: four lanes per float4, each summing a quarter of the
        // planes (8 loads in flight), combined as (q0 + q1) + (q2 + q3) --
        // a fixed order, so the result stays deterministic
        const size_t c4 = count / 4, total = 4 * c4;
        const float4* p4 = reinterpret_cast<const float4*>(part);
        float4* o4 = reinterpret_cast<float4*>(out);
        const int lane = threadIdx.x & 31, qq = lane & 3, per = groups / 4;
        for (size_t t = t0 - lane; t < total; t += stride) {  // warp-uniform trip count
            const size_t tt = t + lane, i = tt >> 2;
            const bool ok = tt < total;
            float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ok) {
                for (int gi = qq * per; gi < (qq + 1) * per; gi += 8) {
                    float4 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = __ldg(p4 + (size_t)(gi + u) * c4 + i);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        s.x += v[u].x;
                        s.y += v[u].y;
                        s.z += v[u].z;
                        s.w += v[u].w;
                    }
                }
            }
            float4 o;  // (q0 + q1) + (q2 + q3) on lane q0 of the quad
            o.x = s.x + __shfl_down_sync(0xffffffffu, s.x, 1);
            o.y = s.y + __shfl_down_sync(0xffffffffu, s.y, 1);
            o.z = s.z + __shfl_down_sync(0xffffffffu, s.z, 1);
            o.w = s.w + __shfl_down_sync(0xffffffffu, s.w, 1);
            o.x += __shfl_down_sync(0xffffffffu, o.x, 2);
            o.y += __shfl_down_sync(0xffffffffu, o.y, 2);
            o.z += __shfl_down_sync(0xffffffffu, o.z, 2);
            o.w += __shfl_down_sync(0xffffffffu, o.w, 2);
            if (ok && qq == 0) {
                if (accumulate == 1) {
                    const float4 a = o4[i];
                    o = make_float4(a.x + o.x, a.y + o.y, a.z + o.z, a.w + o.w);
                }
                if (accumulate == 2)
                    mc_red_add4(o4 + i, o);
                else
                    o4[i] = o;
            }
        }
        return;
    }
    if (aligned) {
        const size_t c4 = count / 4;
        const float4* p4 = reinterpret_cast<const float4*>(part);
        float4* o4 = reinterpret_cast<float4*>(out);
        for (size_t i = t0; i < c4; i += stride) {
            float4 s = accumulate == 1 ? o4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
            int gi = 0;
            // 8 loads in flight, summed in plane order (16 or 32 in flight: the same
            // time at config 2 -- the reduce is not bound by its load latency)
            constexpr int NF = 8;
            for (; gi + NF <= groups; gi += NF) {
                float4 v[NF];
#pragma unroll
                for (int u = 0; u < NF; ++u) v[u] = __ldg(p4 + (size_t)(gi + u) * c4 + i);
#pragma unroll
                for (int u = 0; u < NF; ++u) {
                    s.x += v[u].x;
                    s.y += v[u].y;
                    s.z += v[u].z;
                    s.w += v[u].w;
                }
            }
            for (; gi < groups; ++gi) {
                const float4 v = __ldg(p4 + (size_t)gi * c4 + i);
                s.x += v.x;
                s.y += v.y;
                s.z += v.z;
                s.w += v.w;
            }
            if (accumulate == 2)
                mc_red_add4(o4 + i, s);
            else
                o4[i] = s;
        }
        return;
    }
    for (size_t i = t0; i < count; i += stride) {
        float s = accumulate == 1 ? out[i] : 0.0f;
        for (int gi = 0; gi < groups; ++gi) s += part[(size_t)gi * count + i];
        if (accumulate == 2)
            mc_red_add(out + i, s);
        else
            out[i] = s;
    }
}

}  // namespace cbp
