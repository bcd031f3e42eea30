// cbp_fp.cuh -- rows a2-a5: forward projection y = A c (Eq. 6) as an
// atomics-free per-(view, bin) gather over the pixel strip the fan ray covers.
//
// Thread = one detector bin j of one view v of one image.  For the ray of bin
// j everything of Eq. 11-13 that does not depend on the pixel is a constant:
// the ray frame r_j, v_j, the projected pixel directions zeta1 = h r_x,
// zeta2 = h r_y (Eq. 12) and the effective-blur gain g_j.  The
// pixel-dependent quantities are affine in (row, col):
//   s'(k)   = r_j . (p - k)       (Eq. 11 with the pixel moved to the origin, Eq. 4)
//   tau'(k) = g_j (k - p) . v_j   (Eq. 13 on the plane through k, ledger #1)
// so the thread walks the image along the axis most parallel to the ray
// ("lines" i) and, on each line, visits the K pixels q whose blurred support
// can contain the ray, |s'| < (A + B + C)/2.  The crossing of the ray's
// support edge with line i is carried in 32.32 fixed point, which keeps s'
// exact to ~1e-7 h at any image size (an FP32 absolute coordinate would lose
// log2(n) bits).
//
// Layout: the image is read from a zero-padded copy (rows-major rays) or a
// zero-padded transposed copy (column-major rays) built by cbp_pad_kernel,
// so the K candidates of a line are always K consecutive floats (coalesced
// across the warp's adjacent bins, no bounds checks).  Two lines are
// evaluated together in packed f32x2 arithmetic (FFMA2), K is warp-uniform
// and unrolled.  Each output is written once (no atomics, deterministic; the
// paper's FP used atomic adds).
#pragma once

#include "cbp_common.cuh"

namespace cbp {

struct FPParams {
    GeomDev g;
    Tables t;
    // zero-padded image copies, S slices interleaved per pixel:
    // pad [G][np][np][S], pixel (r, c) of slice g S + s at ((g np + r + P) np + c + P) S + s;
    // padT the same with r and c swapped (G = ceil(batch / S))
    const float* pad;
    const float* padT;
    int np, P;          // padded side, pad width (>= max K)
    float* sino;        // [batch][view_count][n_det]
    int view_begin, view_count, batch;
    // a second block of (base) views in the same launch: blockIdx.x >= split
    // is view view_begin2 + (blockIdx.x - split), written through sino2
    // (the dihedral shard's mirrored block; split = INT_MAX: none)
    int split, view_begin2;
    float* sino2;
    // > 0: 4-fold rotational symmetry (see cbp_pad_sym4_kernel): the S = 4
    // slices are the image rotated by 0, 90, 180, 270 degrees and slice q of
    // base view vl is view vl + q sym_stride of the single output sinogram
    int sym_stride;
    // 8: the full dihedral symmetry (S = 8, cbp_pad_sym8_kernel) over base
    // views [0, n_views/8], output the natural [n_views][n_det] sinogram
    int sym_mode;
    // 1 (with sym_stride > 0): a column-major ray of base view v is walked as
    // the row-major ray of view v + n_views/4 and its frame s written as frame
    // s + 1, so only the row-major padded copy is read (padT is not built)
    int rot_rows;
    // (the line split is the kernel's PARTS template parameter, see cbp_fp_kernel)
};

constexpr int FP_BLOCK = 128;
// threads of an FP CTA: 128, or 32 PARTS when a ray group's lines are split
// over more than 4 warps (small grids: view shards, small images)
__host__ __device__ constexpr int fp_threads(int parts) { return parts <= 4 ? FP_BLOCK : 32 * parts; }
constexpr int FP_KMAX_UNROLLED = 6;
#ifndef CBP_FP_S4_MINB  // resident 128-thread CTAs per SM of the 4-slice FP (A/B knob)
#define CBP_FP_S4_MINB 6
#endif
#ifndef CBP_FP_P8_MINB  // resident 256-thread CTAs per SM of the 8-part FP (A/B knob)
#define CBP_FP_P8_MINB 2
#endif

// ---- zero-padded (and transposed) image copies, S slices interleaved ------
constexpr int PAD_TILE = 32;
#ifndef CBP_PAD_ROWS  // threads per tile column of the pad kernels (A/B knob)
#define CBP_PAD_ROWS 8
#endif
constexpr int PAD_ROWS = CBP_PAD_ROWS;  // a CTA is PAD_TILE x PAD_ROWS threads
// the 4-rotation pad: one row of each staged block per thread, 1024-thread CTAs
// (measured at config 2: 5.6 / 6.4 / 8.5 us for 32 / 16 / 8 rows under ncu)
constexpr int PAD4_ROWS = 32;

template <int S>
__global__ void __launch_bounds__(PAD_TILE * PAD_ROWS) cbp_pad_kernel(const float* __restrict__ img,
                                                               float* __restrict__ pad,
                                                               float* __restrict__ padT, int n,
                                                               int P, int np, int batch)
{
    griddep_launch_dependents();  // the FP may launch and set up its rays meanwhile
    __shared__ float tile[PAD_TILE][PAD_TILE + 1][S];
    const int grp = blockIdx.z;
    const int r0 = blockIdx.y * PAD_TILE, c0 = blockIdx.x * PAD_TILE;
    float* dst = pad + (size_t)grp * np * np * S;
    float* dstT = padT + (size_t)grp * np * np * S;
    for (int rr = threadIdx.y; rr < PAD_TILE; rr += PAD_ROWS) {
        const int r = r0 + rr, c = c0 + threadIdx.x;
        const int sr = r - P, sc = c - P;
        const bool in = sr >= 0 && sr < n && sc >= 0 && sc < n;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const int b = grp * S + k;
            const float v = (in && b < batch) ? img[((size_t)b * n + sr) * n + sc] : 0.0f;
            tile[rr][threadIdx.x][k] = v;
            if (r < np && c < np) dst[((size_t)r * np + c) * S + k] = v;
        }
    }
    __syncthreads();
    for (int cc = threadIdx.y; cc < PAD_TILE; cc += PAD_ROWS) {
        const int c = c0 + cc, r = r0 + threadIdx.x;
        if (r < np && c < np)
#pragma unroll
            for (int k = 0; k < S; ++k) dstT[((size_t)c * np + r) * S + k] = tile[threadIdx.x][cc][k];
    }
}

// Rotation R by +90 degrees about the rotation centre maps pixel (r, c) to
// R(r, c) = (n-1-c, r) and carries view theta to theta + pi/2 with the same
// detector coordinates, so W(v + N/4, j, k) = W(v, j, R^-1 k) exactly (the
// square pixel basis is invariant).  Hence y[v + q N/4] = sum_k c[R^q k] W(v, j, k):
// slice q of the padded copy holds c o R^q, and one weight serves 4 views.
__device__ __forceinline__ void rot90_pow(int n, int q, int& r, int& c)
{
    for (int t = 0; t < q; ++t) {
        const int nr = n - 1 - c;
        c = r;
        r = nr;
    }
}

// The 4 rotated copies: output pixel (R0 + i, C0 + t) of a 32 x 32 tile (image
// coordinates, the padding offset removed) takes c o R^q, and R^q maps the
// tile onto a 32 x 32 image block whose local index is a fixed permutation:
//   q = 0: block (R0, C0),               value at [i][t]
//   q = 1: block (n-32-C0, R0),          value at [31-t][i]
//   q = 2: block (n-32-R0, n-32-C0),     value at [31-i][31-t]
//   q = 3: block (C0, n-32-R0),          value at [t][31-i]
// so the four blocks are staged with coalesced row loads (out-of-image
// pixels load 0: the zero border) and gathered from shared memory for pad
// (row-major) and padT (the transposed tile) without per-pixel rotation
// arithmetic.  (Reading the rotated pixels straight from global memory walks
// a column per warp for q = 1, 3: 17 sectors per request, L1-bound; and a
// staged variant with per-pixel rotation maths was slower still.)
template <bool TRANSPOSE>
__global__ void __launch_bounds__(PAD_TILE * PAD4_ROWS) cbp_pad_sym4_kernel(const float* __restrict__ img,
                                                                          float* __restrict__ pad,
                                                                          float* __restrict__ padT, int n,
                                                                          int P, int np)
{
    griddep_launch_dependents();  // the FP may launch and set up its rays meanwhile
    __shared__ float S[4][PAD_TILE][PAD_TILE + 1];
    const int r0 = blockIdx.y * PAD_TILE, c0 = blockIdx.x * PAD_TILE;  // padded coordinates
    const int R0 = r0 - P, C0 = c0 - P, t = threadIdx.x;
    const int ar[4] = {R0, n - PAD_TILE - C0, n - PAD_TILE - R0, C0};  // block origins (row, col)
    const int ac[4] = {C0, R0, n - PAD_TILE - C0, n - PAD_TILE - R0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int b = ac[q] + t;
        const bool bin = b >= 0 && b < n;
#pragma unroll
        for (int i = threadIdx.y; i < PAD_TILE; i += PAD4_ROWS) {
            const int a = ar[q] + i;
            S[q][i][t] = (bin && a >= 0 && a < n) ? __ldg(img + (size_t)a * n + b) : 0.0f;
        }
    }
    __syncthreads();
    constexpr int L = PAD_TILE - 1;
    for (int i = threadIdx.y; i < PAD_TILE; i += PAD4_ROWS) {
        const int r = r0 + i, c = c0 + t;
        if (r < np && c < np)
            *reinterpret_cast<float4*>(pad + ((size_t)r * np + c) * 4) =
                make_float4(S[0][i][t], S[1][L - t][i], S[2][L - i][L - t], S[3][t][L - i]);
    }
    if constexpr (!TRANSPOSE) return;  // the rot_rows FP reads pad only
    for (int i = threadIdx.y; i < PAD_TILE; i += PAD4_ROWS) {
        const int r = r0 + t, c = c0 + i;  // pixel (r, c) of the tile, stored at padT[c][r]
        if (r < np && c < np)
            *reinterpret_cast<float4*>(padT + ((size_t)c * np + r) * 4) =
                make_float4(S[0][t][i], S[1][L - i][t], S[2][L - t][L - i], S[3][i][L - t]);
    }
}

// The mirror M: (x, y) -> (x, -y) maps view theta to -theta and detector
// coordinate s to -s (bin j to N_s-1-j), and pixel (r, c) to (n-1-r, c).  With
// the rotations it gives 8 frames g = R^q M^m:  W(view_g(v), bin_m(j), g k) =
// W(v, j, k), view_g(v) = (m ? n_views - v : v) + q n_views/4 (mod n_views),
// so y[view_g(v)][bin_m(j)] = sum_k c[g k] W(v, j, k): slice 4m + q of the
// padded copy holds c o (R^q M^m).  Base views v in [0, n_views/8]; for v = 0
// and v = n_views/8 the mirrored frames repeat the rotated ones.
__global__ void __launch_bounds__(PAD_TILE * PAD_ROWS) cbp_pad_sym8_kernel(const float* __restrict__ img,
                                                                    float* __restrict__ pad,
                                                                    float* __restrict__ padT, int n,
                                                                    int P, int np)
{
    griddep_launch_dependents();  // the FP may launch and set up its rays meanwhile
    __shared__ float tile[PAD_TILE][PAD_TILE + 1][8];
    const int r0 = blockIdx.y * PAD_TILE, c0 = blockIdx.x * PAD_TILE;
    for (int rr = threadIdx.y; rr < PAD_TILE; rr += PAD_ROWS) {
        const int r = r0 + rr, c = c0 + threadIdx.x;
        const int sr = r - P, sc = c - P;
        const bool in = sr >= 0 && sr < n && sc >= 0 && sc < n;
        float v[8];
#pragma unroll
        for (int f = 0; f < 8; ++f) {
            int a = f >= 4 ? n - 1 - sr : sr, b = sc;  // M first, then R^q
            rot90_pow(n, f & 3, a, b);
            v[f] = in ? img[(size_t)a * n + b] : 0.0f;
            tile[rr][threadIdx.x][f] = v[f];
        }
        if (r < np && c < np) {
            float4* d = reinterpret_cast<float4*>(pad + ((size_t)r * np + c) * 8);
            d[0] = make_float4(v[0], v[1], v[2], v[3]);
            d[1] = make_float4(v[4], v[5], v[6], v[7]);
        }
    }
    __syncthreads();
    for (int cc = threadIdx.y; cc < PAD_TILE; cc += PAD_ROWS) {
        const int c = c0 + cc, r = r0 + threadIdx.x;
        if (r < np && c < np) {
            const float* t = tile[threadIdx.x][cc];
            float4* d = reinterpret_cast<float4*>(padT + ((size_t)c * np + r) * 8);
            d[0] = make_float4(t[0], t[1], t[2], t[3]);
            d[1] = make_float4(t[4], t[5], t[6], t[7]);
        }
    }
}

// S consecutive floats of one padded pixel
template <int S>
__device__ __forceinline__ void ld_pix(const float* p, float (&v)[S])
{
    if constexpr (S == 1) {
        v[0] = __ldg(p);
    } else if constexpr (S == 2) {
        const float2 a = __ldg(reinterpret_cast<const float2*>(p));
        v[0] = a.x;
        v[1] = a.y;
    } else {
#pragma unroll
        for (int q = 0; q < S; q += 4) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(p) + q / 4);
            v[q] = a.x;
            v[q + 1] = a.y;
            v[q + 2] = a.z;
            v[q + 3] = a.w;
        }
    }
}

// ---- per-ray constants -----------------------------------------------------
// On line i the first candidate is q_lo = floor(e(i)) + 1, where e(i) is the
// lower support edge in 32.32 fixed point; with f = frac(e(i)):
//   s'(q_lo)   = b_q (1 - sigma_q - f)
//   tau'(q_lo) = Be0 + i dB - tq f           (affine in i and f)
//   z11(q_lo)  = z0c + bqs f + tau'/2
// and the k-th candidate adds k dz to z11 (and z21), k tq to tau', k mtqc to w1.
struct FPRay {
    float z0c, bqs;       // z11 = z0c + bqs f_u + tau'/2   (f_u = f 2^32)
    float Be0, dB, btq;   // tau' = Be0 + i dB + btq f_u
    float dz, tq, mtqc;   // per-candidate increments of z11 (and z21), tau', w1
    float A, invC, hC;
    uint32_t flo, mlo;    // 32.32 fixed point: support lower edge on the first line, step
    int32_t fhi, mhi;
    const float* base;    // padded image of this ray's orientation (row / column major)
};

// MAB: how min(A, tau') is known along the ray (warp-uniform): 0 = evaluate
// per candidate, 1 = tau' <= A everywhere (min = tau'), 2 = tau' >= A (min = A).
//
// Along a line every knot argument is affine in the candidate index k, so the
// four sat() arguments t.. = sat(z/C + ...) are formed directly from k
// (u11 = z11/C + 1, u12 = u11 - tau'/C, u21 = u11 - A/C, u22 = u12 - A/C),
// and the trapezoid bound r = A + tau' - z11 is affine in k too.
// `out` holds the thread's S FP64 totals at stride NT (shared memory)
// CLAMP = 1: keep 1 / tau' finite for candidates in the zero border behind a
// close source (tau' <= 0 there); 0: the host proved tau' > 0 at every padded
// pixel of every ray (fp_tau_positive); 2: parallel beam, tau' = tau for every
// candidate (Eq. 9-10), so its update and reciprocal leave the loops
template <int K, int MAB, int S, bool PRE, int NT, int CLAMP = 1>
__device__ __forceinline__ void fp_walk(const FPRay& R, int i0, int i1, int n, int np, int P,
                                        double* out)
{
    uint32_t flo = R.flo;
    int32_t fhi = R.fhi;
    const int qmax = n + P - K;
    const float* row = R.base + ((size_t)(i0 + P) * np + P) * S;  // line i0, column 0
    float2 fi = make_float2((float)i0, (float)i0 + 1.0f);
    const float2 AC = make_float2(-R.A * R.invC, -R.A * R.invC);
    const float iBpar = CLAMP == 2 ? rcp_approx(R.Be0) : 0.0f;  // parallel beam: 1 / tau, once per ray
    const float dzC = R.dz * R.invC, dzC2 = dzC - R.tq * R.invC, dr = R.tq - R.dz;
    for (int i = i0; i <= i1;) {
        // S == 1: acc[0] = (line a, line b).  S >= 2: acc[q2] = slices (2 q2, 2 q2 + 1) of
        // line a, acc[S/2 + q2] the same of line b -- the packed operands are then the
        // register pairs of the pixel loads (no moves to pair up the two lines)
        float2 acc[S];
#pragma unroll
        for (int q = 0; q < S; ++q) acc[q] = make_float2(0.0f, 0.0f);
        const int iend = min(i1, i + 31);  // FP32 partial sums over <= 16 line pairs
        for (; i <= iend; i += 2) {
            // line a = i, line b = i + 1
            const uint32_t fla = flo;
            const int32_t ha = fhi;
            uint32_t flb;
            int32_t hb;
            asm("add.cc.u32 %0, %2, %3;\n\taddc.s32 %1, %4, %5;"
                : "=r"(flb), "=r"(hb) : "r"(flo), "r"(R.mlo), "r"(fhi), "r"(R.mhi));
            asm("add.cc.u32 %0, %2, %3;\n\taddc.s32 %1, %4, %5;"
                : "=r"(flo), "=r"(fhi) : "r"(flb), "r"(R.mlo), "r"(hb), "r"(R.mhi));
            // first candidate (clamped into the zero border when the ray misses the line)
            const int qa = min(max(ha + 1, -P), qmax), qb = min(max(hb + 1, -P), qmax);
            const float* pa = row + qa * S;
            const float* pb = row + ((size_t)np + qb) * S;
            row += 2 * (size_t)np * S;
            const float2 f = make_float2((float)fla, (float)flb);
            float2 B0 = CLAMP == 2 ? make_float2(R.Be0, R.Be0)  // parallel beam: tau' = tau
                                   : __ffma2_rn(f, make_float2(R.btq, R.btq),
                                                __ffma2_rn(fi, make_float2(R.dB, R.dB), make_float2(R.Be0, R.Be0)));
            // (no clamp here: tau' is affine along the line, and the first candidate
            // may lie in the zero border behind a close source with tau' < 0 --
            // clamping it shifted every later candidate's tau'; only the
            // reciprocal below is kept finite)
            fi = __fadd2_rn(fi, make_float2(2.0f, 2.0f));
            float2 z0 = __ffma2_rn(f, make_float2(R.bqs, R.bqs), make_float2(R.z0c, R.z0c));
            z0 = __ffma2_rn(make_float2(0.5f, 0.5f), B0, z0);                       // z11
            const float2 r0 = __fadd2_rn(__fadd2_rn(B0, make_float2(R.A, R.A)), neg2(z0));  // A + B - z11
            const float2 u11 = __ffma2_rn(z0, make_float2(R.invC, R.invC), make_float2(1.0f, 1.0f));
            const float2 u12 = __ffma2_rn(neg2(B0), make_float2(R.invC, R.invC), u11);
            const float2 u21 = __fadd2_rn(u11, AC), u22 = __fadd2_rn(u12, AC);
            // PRE: issue all of the line pair's loads first (more loads in flight;
            // measured: +1 % at S = 4 on the line-part grids, -1 % on a batch grid)
            float cpa[PRE ? K : 1][S], cpb[PRE ? K : 1][S];
            if constexpr (PRE) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    ld_pix<S>(pa + k * S, cpa[k]);
                    ld_pix<S>(pb + k * S, cpb[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                float ca[S], cb[S];
                if constexpr (PRE) {
#pragma unroll
                    for (int q = 0; q < S; ++q) {
                        ca[q] = cpa[k][q];
                        cb[q] = cpb[k][q];
                    }
                } else {
                    ld_pix<S>(pa + k * S, ca);
                    ld_pix<S>(pb + k * S, cb);
                }
                const float kf = (float)k;
                const float2 kk = make_float2(kf, kf);
                const float2 z11 = k ? __ffma2_rn(kk, make_float2(R.dz, R.dz), z0) : z0;
                const float2 r = k ? __ffma2_rn(kk, make_float2(dr, dr), r0) : r0;
                const float2 B = (k && CLAMP != 2) ? __ffma2_rn(kk, make_float2(R.tq, R.tq), B0) : B0;
                const float2 t11 = make_float2(sat_fma(kf, dzC, u11.x), sat_fma(kf, dzC, u11.y));
                const float2 t12 = make_float2(sat_fma(kf, dzC2, u12.x), sat_fma(kf, dzC2, u12.y));
                const float2 t21 = make_float2(sat_fma(kf, dzC, u21.x), sat_fma(kf, dzC, u21.y));
                const float2 t22 = make_float2(sat_fma(kf, dzC2, u22.x), sat_fma(kf, dzC2, u22.y));
                float2 T = __fmul2_rn(t11, t11);
                T = __ffma2_rn(neg2(t12), t12, T);
                T = __ffma2_rn(neg2(t21), t21, T);
                T = __ffma2_rn(t22, t22, T);
                const float ma = MAB == 1 ? B.x : (MAB == 2 ? R.A : fminf(R.A, B.x));
                const float mb = MAB == 1 ? B.y : (MAB == 2 ? R.A : fminf(R.A, B.y));
                const float2 M2 = make_float2(fmaxf(fmin3(z11.x, ma, r.x), 0.0f),
                                              fmaxf(fmin3(z11.y, mb, r.y), 0.0f));
                const float2 num = __ffma2_rn(make_float2(R.hC, R.hC), T, M2);
                // tau' > 0 at every pixel a ray's support reaches; candidates in the zero
                // border behind a close source can have tau' <= 0: keep 1/tau' finite
                // (their image values are 0)
                const float2 iB = CLAMP == 1   ? rcp2(make_float2(fmaxf(B.x, 1e-30f), fmaxf(B.y, 1e-30f)))
                                  : CLAMP == 2 ? make_float2(iBpar, iBpar)
                                               : rcp2(B);
                if constexpr (S == 1) {
                    const float2 cw = __fmul2_rn(make_float2(ca[0], cb[0]), iB);
                    acc[0] = __ffma2_rn(cw, num, acc[0]);
                } else {  // one weight, S slices
                    const float2 w = __fmul2_rn(num, iB);
#pragma unroll
                    for (int q = 0; q < S; q += 2) {
                        acc[q / 2] = __ffma2_rn(make_float2(ca[q], ca[q + 1]), make_float2(w.x, w.x), acc[q / 2]);
                        acc[S / 2 + q / 2] = __ffma2_rn(make_float2(cb[q], cb[q + 1]), make_float2(w.y, w.y),
                                                        acc[S / 2 + q / 2]);
                    }
                }
            }
        }
        if constexpr (S == 1) {
            out[0] += (double)acc[0].x + (double)acc[0].y;  // two-level sum
        } else {
#pragma unroll
            for (int q = 0; q < S; q += 2) {
                out[q * NT] += (double)acc[q / 2].x + (double)acc[S / 2 + q / 2].x;
                out[(q + 1) * NT] += (double)acc[q / 2].y + (double)acc[S / 2 + q / 2].y;
            }
        }
    }
}

template <int K, int S, bool PRE, int NT, int CLAMP = 1>
__device__ __forceinline__ void fp_walk_k(const FPRay& R, int mab, int i0, int i1, int n, int np,
                                          int P, double* out)
{
    if (mab == 1) fp_walk<K, 1, S, PRE, NT, CLAMP>(R, i0, i1, n, np, P, out);
    else if (mab == 2) fp_walk<K, 2, S, PRE, NT, CLAMP>(R, i0, i1, n, np, P, out);
    else fp_walk<K, 0, S, PRE, NT, CLAMP>(R, i0, i1, n, np, P, out);
}

// generic K (wide bins relative to pixels): same arithmetic, runtime trip count
template <int S, int NT>
__device__ void fp_walk_generic(const FPRay& R, int K, int i0, int i1, int n, int np, int P,
                                double* out)
{
    uint32_t flo = R.flo;
    int32_t fhi = R.fhi;
    const int qmax = n + P - K;
    for (int i = i0; i <= i1; ++i) {
        const uint32_t fl = flo;
        const int qc = min(max(fhi + 1, -P), qmax);
        asm("add.cc.u32 %0, %0, %2;\n\taddc.s32 %1, %1, %3;"
            : "+r"(flo), "+r"(fhi) : "r"(R.mlo), "r"(R.mhi));
        const float* p = R.base + ((size_t)(i + P) * np + (qc + P)) * S;
        const float ff = (float)fl;
        const float B0 = fmaf(ff, R.btq, fmaf((float)i, R.dB, R.Be0));  // affine: no clamp (see fp_walk)
        const float z0 = fmaf(0.5f, B0, fmaf(ff, R.bqs, R.z0c));
        float part[S];
#pragma unroll
        for (int q = 0; q < S; ++q) part[q] = 0.0f;
        for (int k = 0; k < K; ++k) {
            const float kf = (float)k;
            const float z11 = fmaf(kf, R.dz, z0);
            const float z21 = z11 - R.A;
            const float B = fmaf(kf, R.tq, B0);
            const float w1 = fmaf(-B, R.invC, 1.0f);
            const float2 num = cnsf_num2(make_float2(z11, z11), make_float2(z21, z21),
                                         make_float2(B, B), make_float2(w1, w1), R.A, R.invC, R.hC);
            const float w = num.x * rcp_approx(fmaxf(B, 1e-30f));
            float c[S];
            ld_pix<S>(p + k * S, c);
#pragma unroll
            for (int q = 0; q < S; ++q) part[q] = fmaf(c[q], w, part[q]);
        }
#pragma unroll
        for (int q = 0; q < S; ++q) out[q * NT] += (double)part[q];
    }
}

// The precise mode (narrow bins, cbp_common.cuh cnsf_prec): s' and tau' of a
// candidate come straight from their FP64 affine forms in (line, candidate)
// instead of FP32 increments; the 32.32 crossing still picks the candidates.
struct FPRayD {
    double X00, a_i, b_q;  // s'(line i, candidate q) = X00 + i a_i + q b_q
    double T00, t_i, t_q;  // tau'(i, q) = T00 + i t_i + q t_q
    double A;              // max |zeta|
    float Cz;              // min |zeta|
};

template <int NT>
__device__ void fp_walk_prec(const FPRay& R, const FPRayD& D, int K, int i0, int i1, int n, int np, int P,
                             double* out)
{
    uint32_t flo = R.flo;
    int32_t fhi = R.fhi;
    const int qmax = n + P - K;
    for (int i = i0; i <= i1; ++i) {
        const int qc = min(max(fhi + 1, -P), qmax);
        asm("add.cc.u32 %0, %0, %2;\n\taddc.s32 %1, %1, %3;"
            : "+r"(flo), "+r"(fhi) : "r"(R.mlo), "r"(R.mhi));
        const float* p = R.base + ((size_t)(i + P) * np + (qc + P));
        const double Xi = fma((double)i, D.a_i, D.X00), Ti = fma((double)i, D.t_i, D.T00);
        float part = 0.0f;
        for (int k = 0; k < K; ++k) {
            const double q = (double)(qc + k);
            const float w = cnsf_prec(fma(q, D.b_q, Xi), D.A, (float)fma(q, D.t_q, Ti), D.Cz);
            part = fmaf(__ldg(p + k), w, part);
        }
        out[0] += (double)part;
    }
}

// PARTS (1, 2, 4) warps of a CTA share the same 32 rays and walk disjoint
// parts of their lines; the parts' FP64 totals are summed in part order in
// shared memory (deterministic).  A CTA covers 128 / PARTS bins.  PARTS > 1
// when the grid would otherwise be short of ~16 waves: the ragged last wave
// of a 1.6-wave grid cost ~25 %.
template <int S, int PARTS, bool PREC = false, int CLAMP = 1>
__global__ void __launch_bounds__(fp_threads(PARTS), PARTS > 4 ? CBP_FP_P8_MINB : (S == 1 ? 7 : (S == 4 ? CBP_FP_S4_MINB : 4)))
    cbp_fp_kernel(const FPParams P)
{
    static_assert(!PREC || S == 1, "the precise mode runs one slice per weight");
    const GeomDev& g = P.g;
    constexpr int NT = fp_threads(PARTS);
    // PDL: with one part per ray (long walks, large grids) the wait comes first
    // -- placed after the set-up it cost the walk 2.4 % at config 5 (code
    // generation); with line parts (short walks) the set-up overlaps the pad's
    // tail (config 2: 1.5 % faster)
    if constexpr (PARTS == 1) {
        griddep_wait();
        griddep_launch_dependents();
    }
    constexpr int BINS = NT / PARTS;  // bins per CTA
    const int warp = threadIdx.x >> 5, part = warp % PARTS;
    // view-major CTA order (grid.x = view slot, grid.y = detector tile): the
    // CTAs in flight read the image strips of a few detector tiles over many
    // views, not the whole image for a few views -- config 5 (64 MB of padded
    // frames) reads 136 MB from DRAM per FP instead of 1.19 GB
    const int jr = blockIdx.y * BINS + (warp / PARTS) * 32 + (threadIdx.x & 31);
    const bool valid = jr < g.n_det;
    const int j = valid ? jr : g.n_det - 1;
    const bool second = (int)blockIdx.x >= P.split;
    const int vl = second ? (int)blockIdx.x - P.split : (int)blockIdx.x;
    const int grp = blockIdx.z;  // slices grp S .. grp S + S - 1
    const int v = (second ? P.view_begin2 : P.view_begin) + vl;
    float* const sino_out = second ? P.sino2 : P.sino;
    const int n = g.n;

    // ---- per-ray constants (FP64): Eq. 11 frame, Eq. 12 directions, Eq. 13 gain
    const double2 cs = P.t.view_cs[v];
    const double2 bd = P.t.bin_d[j];
    const double s = bd.x, invL = bd.y;
    const double sphi = g.parallel ? 0.0 : s * invL, cphi = g.parallel ? 1.0 : g.sdd * invL;
    double cth = cs.x, sth = cs.y;
    // rot_rows: rotating the scanner by +90 degrees (u -> (-sin, cos)) maps this
    // ray onto the same bin of view v + N/4, where it runs along the rows
    // (r' = (-r_y, r_x)), and W(v + N/4, j, R k) = W(v, j, k):
    // frame s of the rotated walk is output frame s + 1
    int rq = 0;
    if (P.rot_rows && fabs(sphi * cth - cphi * sth) < fabs(cphi * cth + sphi * sth)) {
        const double t = cth;
        cth = -sth;
        sth = t;
        rq = 1;
    }
    const double rx = sphi * cth - cphi * sth;  // r_j = (D_ps e + s_j u) / L_j  (parallel: e)
    const double ry = cphi * cth + sphi * sth;
    const double vx = -ry, vy = rx;             // v_j = (-D_ps u + s_j e) / L_j
    const double h = g.h, c0 = g.c0;
    // s'(row, col) = X00 + col * bcol + row * brow   (r.p = s_j D_po / L_j; parallel: s' = s_j - k.e)
    const double X00 = (g.parallel ? s : s * g.sid * invL) + h * c0 * (rx - ry);
    const double bcol = -rx * h, brow = ry * h;
    // d(row, col) = (k - p).v = D00 + col * dcol + row * drow  (p.v = -D_po D_ps / L_j);
    // parallel: tau' = tau everywhere (g_j d = 1 * tau)
    const double D00 = g.parallel ? g.tau : g.sid * g.sdd * invL + h * c0 * (vy - vx);
    const double dcol = g.parallel ? 0.0 : vx * h, drow = g.parallel ? 0.0 : -vy * h;
    const double gj = g.parallel ? 1.0 : (double)P.t.bin_f[j].z;

    const bool rows_major = fabs(rx) >= fabs(ry);
    const double a_i = rows_major ? brow : bcol;  // step of s' along the line index
    const double b_q = rows_major ? bcol : brow;  // step of s' along the line (|b_q| = A)
    const double t_i = gj * (rows_major ? drow : dcol);
    const double t_q = gj * (rows_major ? dcol : drow);
    const double A = fabs(b_q), C = fabs(a_i);
    double dmax = D00;
    dmax = fmax(dmax, D00 + (n - 1) * dcol);
    dmax = fmax(dmax, D00 + (n - 1) * drow);
    dmax = fmax(dmax, D00 + (n - 1) * (dcol + drow));
    const double inv_bq = 1.0 / b_q, inv_A = fabs(inv_bq);  // one FP64 division for both
    const double sig_q = 0.5 * (A + C + gj * dmax) * inv_A;  // support half-width in pixels
    int K = (int)floor(2.0 * sig_q) + 1;                // candidates per line

    // ray crossing of line i: q*(i) = Q0 + i m; lines whose window meets [0, n)
    const double Q0 = -X00 * inv_bq, m = -a_i * inv_bq;
    int ilo, ihi;
    if (fabs(m) < 1e-15) {
        const bool hit = Q0 > -sig_q && Q0 < (n - 1) + sig_q;
        ilo = hit ? 0 : n;
        ihi = hit ? n - 1 : -1;
    } else {
        const double inv_m = 1.0 / m;
        double a = (-sig_q - Q0) * inv_m, c = ((n - 1) + sig_q - Q0) * inv_m;
        if (a > c) {
            const double tmp = a;
            a = c;
            c = tmp;
        }
        a = fmax(-1.0, fmin((double)n, floor(a)));
        c = fmax(-1.0, fmin((double)n, ceil(c)));
        ilo = max(0, (int)a);
        ihi = min(n - 1, (int)c);
    }
    if (!valid) {
        ilo = n;
        ihi = -1;
        K = 1;
    }
    const int wlo = __reduce_min_sync(0xffffffffu, ilo);
    const int whi = __reduce_max_sync(0xffffffffu, ihi);
    const int Kw = __reduce_max_sync(0xffffffffu, K);

    __shared__ double sacc[S * NT];  // FP64 totals, [q][thread]
    double* acc = sacc + threadIdx.x;
#pragma unroll
    for (int q = 0; q < S; ++q)
        acc[q * NT] = Kw > P.P ? __longlong_as_double(0x7ff8000000000000ll) : 0.0;  // pad too thin: NaN
    int i0 = wlo, i1 = whi;
    if (PARTS > 1) {  // this warp's part of the lines: even lengths, because the walk takes
                      // lines in pairs (an odd range reads one line past its end -- harmless
                      // past whi, not inside the next part)
        const int L = 2 * ((whi - wlo + 2 * PARTS) / (2 * PARTS));
        i0 = wlo + part * L;
        i1 = part == PARTS - 1 ? whi : min(whi, i0 + L - 1);
    }
    if constexpr (PARTS > 1) {
        griddep_launch_dependents();  // the BP may launch into this grid's tail
        griddep_wait();               // the padded image (and its pool memory) is ready
    }
    if (i0 <= i1 && Kw <= P.P) {
        FPRay R;
        // lower support edge on line i: q*(i) - sig_q, as 32.32 fixed point from line i0
        const int64_t E0 = (int64_t)llrint((Q0 + (double)i0 * m - sig_q) * 0x1p32);
        const int64_t Mfx = (int64_t)llrint(m * 0x1p32);
        R.flo = (uint32_t)(uint64_t)E0;
        R.fhi = (int32_t)(E0 >> 32);
        R.mlo = (uint32_t)(uint64_t)Mfx;
        R.mhi = (int32_t)(Mfx >> 32);
        // candidate q_lo = floor(e) + 1 has s' = b_q (q_lo - q*) = b_q (1 - sig_q - frac(e));
        // z11 = s' + (A - C)/2 + B/2
        R.z0c = (float)(b_q * (1.0 - sig_q) + 0.5 * (A - C));
        R.bqs = (float)(-b_q * 0x1p-32);
        R.Be0 = (float)(gj * D00 + (Q0 - sig_q + 1.0) * t_q);
        R.dB = (float)(t_i + m * t_q);
        R.btq = (float)(-t_q * 0x1p-32);
        R.dz = (float)(b_q + 0.5 * t_q);
        R.tq = (float)t_q;
        R.A = (float)A;
        const float Cf = (float)C;
        R.invC = 1.0f / Cf;  // +inf for C == 0: handled by sat()
        R.hC = 0.5f * Cf;
        R.mtqc = -R.tq * R.invC;
        R.base = (rows_major ? P.pad : P.padT) + (size_t)grp * P.np * P.np * S;
        // is min(A, tau') decided along the whole ray?  tau' = g d with d affine
        // over the image: its extremes are at the image corners
        double dmin = D00;
        dmin = fmin(dmin, D00 + (n - 1) * dcol);
        dmin = fmin(dmin, D00 + (n - 1) * drow);
        dmin = fmin(dmin, D00 + (n - 1) * (dcol + drow));
        const int mab_t = gj * dmax * (1.0 + 1e-6) < A ? 1 : (gj * dmin * (1.0 - 1e-6) > A ? 2 : 0);
        const int mab = __all_sync(0xffffffffu, mab_t == 1) ? 1 : (__all_sync(0xffffffffu, mab_t == 2) ? 2 : 0);
        if constexpr (PREC) {
            FPRayD Dr;
            Dr.X00 = X00;
            Dr.a_i = a_i;
            Dr.b_q = b_q;
            Dr.T00 = gj * D00;
            Dr.t_i = t_i;
            Dr.t_q = t_q;
            Dr.A = A;
            Dr.Cz = (float)C;
            fp_walk_prec<NT>(R, Dr, Kw, i0, i1, n, P.np, P.P, acc);
        } else {
          switch (Kw) {
            case 1: fp_walk_k<1, S, (S <= 2 || (S == 4 && PARTS > 1)), NT, CLAMP>(R, mab, i0, i1, n, P.np, P.P, acc); break;
            case 2: fp_walk_k<2, S, (S <= 2 || (S == 4 && PARTS > 1)), NT, CLAMP>(R, mab, i0, i1, n, P.np, P.P, acc); break;
            case 3: fp_walk_k<3, S, (S <= 2 || (S == 4 && PARTS > 1)), NT, CLAMP>(R, mab, i0, i1, n, P.np, P.P, acc); break;
            case 4: fp_walk_k<4, S, (S <= 2 || (S == 4 && PARTS > 1)), NT, CLAMP>(R, mab, i0, i1, n, P.np, P.P, acc); break;
            case 5: fp_walk_k<5, S, (S <= 2 || (S == 4 && PARTS > 1)), NT, CLAMP>(R, mab, i0, i1, n, P.np, P.P, acc); break;
            case 6: fp_walk_k<6, S, (S <= 2 || (S == 4 && PARTS > 1)), NT, CLAMP>(R, mab, i0, i1, n, P.np, P.P, acc); break;
            default: fp_walk_generic<S, NT>(R, Kw, i0, i1, n, P.np, P.P, acc); break;
          }
        }
        // (an `else switch` followed by a `#pragma unroll` loop lost that loop in the
        // PREC instantiation -- nvcc 12.9; keep the braces)
        for (int q = 0; q < S; ++q) acc[q * NT] *= h * h * inv_A;  // W = (h^2 / A) num / B
    }
    if (PARTS > 1) {  // sum the parts in part order; the first part's warp writes
        __syncthreads();
        if (part != 0) return;
#pragma unroll
        for (int q = 0; q < S; ++q) {
            double t = acc[q * NT];
#pragma unroll
            for (int pp = 1; pp < PARTS; ++pp) t += acc[q * NT + pp * 32];
            acc[q * NT] = t;
        }
    }
    if (valid)
#pragma unroll
        for (int q = 0; q < S; ++q) {
            const int b = grp * S + q;
            float* dst = nullptr;
            if (P.sym_mode == 8) {
                const int N = g.n_views, m = q >> 2, qq = q & 3;
                if (m && (v == 0 || 8 * v == N)) continue;  // mirrored frame repeats a rotation
                const int view = ((m ? N - v : v) + qq * (N / 4)) % N;
                const int bin = m ? g.n_det - 1 - j : j;
                dst = sino_out + (size_t)view * g.n_det + bin;
            } else if (P.sym_stride > 0) {
                dst = sino_out + ((size_t)vl + (size_t)((q + rq) & 3) * P.sym_stride) * g.n_det + j;
            } else if (b < P.batch) {
                dst = sino_out + ((size_t)b * P.view_count + vl) * g.n_det + j;
            }
            if (dst) *dst = (float)acc[q * NT];
        }
}

}  // namespace cbp
