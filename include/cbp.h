/*
 * cbp.h -- C ABI of the B200-native CNSF fan-beam projector
 * (Zhang & Entezari, "A Convolutional Forward and Back-Projection Model for
 * Fan-Beam Geometry", arXiv 1907.10526).
 *
 * Citations: "P:n" is line n of the paper text, "S:n" line n of
 * SPEC.md, "ledger #k" reading k of DESIGN.md section 3.
 *
 * The library computes, matrix-free and on the fly,
 *   forward   y = A c       (Eq. 6)
 *   back      c = A^T y     (the exact adjoint with the same weights)
 * where A[(v, j), k] = W(v, j, k) = h^2 M_{zeta1, zeta2, tau'}(s'), the
 * blurred fan-beam footprint of Eq. 14 of the indicator pixel k
 * on detector bin j of view v: zeta1, zeta2 from Eq. 12, the
 * effective blur tau' from Eq. 13 on the plane through the pixel centre
 * (ledger #1), s' = R_{v(s_j)^perp}(p - k) (Eq. 11).
 *
 * Conventions:
 *   views   theta_v = 2 pi v / n_views, counter-clockwise from +x (ledger #9)
 *   source  p = sid * (cos theta, sin theta); detector line through
 *           -(sdd - sid) * (cos theta, sin theta) along e = (-sin, cos) (ledger #6)
 *   bins    s_j = (j - (n_det - 1)/2) * det_pitch (ledger #10)
 *   pixels  k(row, col) = ((col - (n-1)/2) h, ((n-1)/2 - row) h) (ledger #13)
 *   blur    unit-mass average over [s_j - tau/2, s_j + tau/2] (ledger #3)
 *
 * Data layout (FP32, contiguous, row-major):
 *   image  [batch][n][n]
 *   sino   [batch][view_count][n_det]   (views view_begin .. view_begin+view_count-1)
 *
 * Memory: every data pointer may be device memory (cudaMalloc / torch CUDA
 * tensors) or host memory (pageable or pinned).  Device pointers must be on
 * the current device.  Host pointers are staged through an internal device
 * workspace with cudaMemcpyAsync on `stream`, and the call then synchronises
 * `stream` before returning so the host result is ready.  The caller owns
 * every buffer; the library never retains a data pointer.  Per-geometry
 * tables (a few KB) and the BP's per-(tile, view) headers (96 B each: up to
 * 256 MB per geometry and view range, 1 GB in all; beyond that they are
 * rebuilt per call in stream-ordered scratch) are cached per device until the
 * process exits, guarded by a mutex.
 *
 * Streams: `stream` is a cudaStream_t (0 = legacy default stream).  With
 * device pointers all work is stream-ordered and asynchronous: execution
 * errors surface at the caller's next synchronisation, not in the return
 * value.  No call except cbp_adjoint_check synchronises the device.
 *
 * Errors: functions return CBP_OK (0) or a negative code; arguments are
 * validated before any CUDA call ("geometry violation -> error before
 * computation").
 */
#ifndef CBP_H
#define CBP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBP_OK      0
#define CBP_EINVAL -1  /* invalid geometry or argument (see cbp_validate)         */
#define CBP_ECUDA  -2  /* CUDA error at launch / copy / allocation of workspace   */
#define CBP_ENOMEM -3  /* host allocation failure                                 */

/* Scanner kinds (cbp_geometry_t.kind) */
#define CBP_FAN_FLAT  0  /* fan beam, flat detector: the paper's geometry          */
#define CBP_PARALLEL  1  /* parallel beam (Eq. 9-10, row f3): the rays of view v run along
                            -u_v through s e_v; sid and sdd are unused (must be finite)      */
#define CBP_FAN_ARC   2  /* fan beam, arc (equiangular) detector (row f3): the detector
                            is the circle of radius sdd about the source, s is arc length
                            (angle s/sdd from the central ray); det_pitch and det_width are
                            arc lengths; every bin must lie within +-90 degrees            */

/* Weight models (cbp_geometry_t.model) */
#define CBP_MODEL_CNSF 0  /* the paper's CNSF weight: per bin ray, Eq. 11-14 with the effective
                             blur tau' of Eq. 13                               */
#define CBP_MODEL_MAG  1  /* row f3, the magnified-footprint variant: the pixel's box-spline
                             footprint mapped onto the detector by the perspective map (Eq. 4,
                             P:144-152) linearised at the pixel centre -- zeta_i = h dP/dx_i(k)
                             -- convolved with the detector cell: W = h^2 m(k)
                             M_{|zeta1|,|zeta2|,tau}(s_j - P(k)), m(k) the pixel's
                             detector-integrated chord length per unit area at its centre
                             ((D_ps^2 + P^2)/(D_ps |k - p|) flat, D_ps/|k - p| arc, 1 parallel).
                             One footprint per (view, pixel) shared by its bins; no view
                             symmetry is used (cbp_symmetry_fold returns 1); the FP64
                             reference projector is the same for both models.            */

/* Scanner and grid (P:96-106 geometry; P:157-159 image; P:124 and P:416
 * detector).  All lengths in mm.                                            */
typedef struct cbp_geometry {
    int32_t n;          /* image is n x n pixels, n >= 1                               */
    double  pixel;      /* pixel side h > 0                                            */
    int32_t n_views;    /* views over [0, 2 pi): theta_v = 2 pi v / n_views, >= 1      */
    int32_t n_det;      /* detector bins N_s >= 1                                      */
    double  det_pitch;  /* bin spacing Delta_s > 0                                     */
    double  det_width;  /* bin width tau > 0 (the detector blur, Eq. 2)                */
    double  sid;        /* D_po, source to rotation centre; n h / sqrt(2) < sid        */
    double  sdd;        /* D_ps, source to detector; sdd >= sid (D_so = sdd - sid)     */
    int32_t kind;       /* CBP_FAN_FLAT (0), CBP_PARALLEL (1) or CBP_FAN_ARC (2)        */
    int32_t model;      /* weight model: CBP_MODEL_CNSF (0, the paper's) or CBP_MODEL_MAG (1) */
} cbp_geometry_t;

/* Validate a geometry (no CUDA call).  CBP_EINVAL if n < 1, pixel <= 0,
 * n_views < 1, n_det < 1, det_pitch <= 0, det_width <= 0, any value
 * non-finite, kind or model unknown, or (fan beam) sid <= 0, sdd < sid,
 * det_width >= 2 sdd, or the field of view's circumscribed circle
 * n h / sqrt(2) is not strictly inside the source orbit (every pixel
 * must lie strictly in front of the source).  In parallel beam W is the
 * 3-direction box spline M_{[h|sin|, h|cos|, tau]}(s_j - k.e) -- exact
 * (Theorem 1).  On the arc the bin of ray angle gamma subtends
 * tau/sdd at the source, tau'(k) = 2 d tan(tau / (2 sdd)).  The reference
 * projector (cbp_ref_*) takes every kind. */
int cbp_validate(const cbp_geometry_t* g);
/* (cbp_validate also rejects bins so narrow that no FP32 projector meets the
 * parity bar: tau'_min / h < 1e-4, with tau'_min / h the lower bound of
 * cbp_narrow_ratio below.) */

/* Narrow bins and the precise mode.  Eq. 14's weight has
 * ramps of width tau' + min|zeta|, and on views where a pixel edge
 * is parallel to the ray min|zeta| -> 0, so an absolute error e in the FP32
 * position s' becomes a relative weight error ~e / tau'.  When
 * cbp_narrow_ratio(g) -- a lower bound on tau' / h over the field of view
 * (tau / h in parallel beam; (sid - n h / sqrt 2) tau sdd / (sdd^2 + s_max^2) / h
 * flat, with the arc's tau / sdd gain) -- is below 0.02, every call runs the
 * precise mode: s', A = max|zeta| and the four knot arguments of the nested
 * form in FP64, rounded once to FP32, with the smallest width nested
 * innermost (cbp_common.cuh cnsf_prec); FP32 elsewhere.  It is slower (no
 * view symmetry or batch sharing, FP64 arithmetic per weight: 3-10x) and
 * holds the parity bar down to tau'/h = 1e-4.  The environment variable CBP_PRECISE=1
 * (or 0) forces the mode on (off) for every geometry.
 * cbp_precise_mode returns 1 if calls with g run the precise mode, 0 if not,
 * CBP_EINVAL for an invalid geometry; cbp_narrow_ratio returns the bound
 * (negative for an invalid geometry). */
int cbp_precise_mode(const cbp_geometry_t* g);
double cbp_narrow_ratio(const cbp_geometry_t* g);

/* Forward projection y = A c (Eq. 6) for views [view_begin,
 * view_begin + view_count) of `batch` images.  Overwrites sino.
 * CBP_EINVAL: invalid geometry, null pointer, batch < 1, view range outside
 * [0, n_views), view_count < 1, device pointer not 4-byte aligned. */
int cbp_forward(const cbp_geometry_t* g, const float* image, float* sino, int32_t batch,
                int32_t view_begin, int32_t view_count, void* stream);

/* Accumulate modes of the back-projections (the `accumulate` argument) */
#define CBP_ACC_OVERWRITE 0  /* image = A^T y                                               */
#define CBP_ACC_ADD       1  /* image += A^T y                                              */
#define CBP_ACC_MULTIMEM  2  /* row a7 fused into the BP: `image` is a MULTICAST address (an
                                NVLink/NVSwitch multicast object, e.g. torch symmetric memory's
                                multicast_ptr, bound to one n x n buffer per rank); the BP's last
                                kernel adds this rank's partial A_g^T y_g to EVERY rank's copy with
                                multimem.red.add.f32 (the switch performs the sum), so after all
                                ranks' calls complete and a barrier, each copy holds sum_g A_g^T y_g
                                -- the view-sharded all-reduce with no separate collective.  The
                                caller zeroes the copies and fences (barrier) before the first
                                rank's call.  Device sinogram only; the image pointer is not
                                checked (a multicast address is not an ordinary allocation);
                                the order of the cross-rank sum is the switch's (not bitwise
                                deterministic).                                            */

/* Back-projection c = A^T y over views [view_begin, view_begin + view_count)
 * (the partial adjoint when the range is a shard of the views).  Overwrites
 * image, adds to it (CBP_ACC_ADD) or adds through a multicast address
 * (CBP_ACC_MULTIMEM).  Errors as cbp_forward, or accumulate outside 0..2. */
int cbp_back(const cbp_geometry_t* g, const float* sino, float* image, int32_t batch,
             int32_t view_begin, int32_t view_count, int32_t accumulate, void* stream);

/* The normal operator out = A^T A image over all views (one FP+BP pair, the
 * benchmark's unit): the sinogram A c lives in an internal device buffer
 * and never crosses to the host.  Host or device pointers as cbp_forward
 * (host pointers: the call synchronises `stream`).  Overwrites out.  Errors
 * as cbp_forward. */
int cbp_normal(const cbp_geometry_t* g, const float* image, float* out, int32_t batch, void* stream);

/* The normal operator over a sequence of `count` inputs, pipelined: input i
 * is images + i batch n n, its result out + i batch n n (both [count][batch][n][n]).
 * With HOST buffers (pinned for overlap; pageable memory works but its
 * copies serialise) the library runs a three-stage pipeline on the device:
 * the host->device copy of input i+1 and the device->host copy of result
 * i-1 (two internal streams, double-buffered device images) overlap the
 * FP+BP pair of input i on `stream`; the call returns when every result is
 * in host memory (one host-buffer call at a time per device: a mutex
 * serialises them).  With DEVICE buffers the pairs run back to back on
 * `stream` (asynchronous; the sinogram is stream-ordered scratch of the
 * call, so calls on different streams do not share it).  The sinogram never
 * leaves the device.  CBP_EINVAL as
 * cbp_normal, count < 1, or one host and one device pointer. */
int cbp_normal_stream(const cbp_geometry_t* g, const float* images, float* out, int32_t count, int32_t batch,
                      void* stream);

/* Rotational symmetry.  Rotating the whole scanner by 90
 * degrees maps view v to view v + n_views/4, keeps every detector coordinate
 * and permutes the square pixel grid, so W(v + n_views/4, j, k) = W(v, j, R^-1 k)
 * exactly, R(row, col) = (n-1-col, row).  When n_views % 4 == 0 one weight
 * therefore serves 4 views.  With the mirror (x, y) -> (x, -y), which maps
 * view v to n_views - v, bin j to n_det-1-j and (row, col) to (n-1-row, col),
 * one weight serves 8 views when n_views % 8 == 0.  cbp_forward / cbp_back
 * use this automatically over the full view range: the FP for a single image
 * (the 4 rotations; a batch shares each weight across 4 images instead), the
 * BP for a single image and, image by image, for a batch.
 * cbp_symmetry_fold returns the BP's views per weight evaluation (8, 4 or 1;
 * CBP_EINVAL for an invalid geometry).  The environment variables
 * CBP_NO_SYMMETRY (all) and CBP_NO_MIRROR (the mirror) disable it. */
int cbp_symmetry_fold(const cbp_geometry_t* g, int32_t batch, int32_t view_begin,
                      int32_t view_count);

/* The orbit form, for sharding views over GPUs without losing the symmetry:
 * one image, the 4 n_b views {b + q n_views/4 : b in [base_begin,
 * base_begin + base_count), q = 0..3} (0 <= base_begin, base_begin + base_count
 * <= n_views/4; requires n_views % 4 == 0).  sino is [4][base_count][n_det]:
 * row q base_count + i is view base_begin + i + q n_views/4.  Device pointers
 * only, 4-byte aligned.  cbp_back_orbit overwrites image, or adds to
 * it when accumulate != 0.  CBP_EINVAL otherwise. */
int cbp_forward_orbit(const cbp_geometry_t* g, const float* image, float* sino,
                      int32_t base_begin, int32_t base_count, void* stream);
int cbp_back_orbit(const cbp_geometry_t* g, const float* sino, float* image,
                   int32_t base_begin, int32_t base_count, int32_t accumulate, void* stream);

/* Dihedral shards (n_views % 8 == 0): base views b in [base_begin,
 * base_begin + base_count) within [0, n_views/8]; the shard's views are
 * their orbits {view_g(b) : g = R^q M^m} (8 views per base view, 4 for
 * b = 0 and b = n_views/8), so shards of a partition of [0, n_views/8] cover
 * every view once and each keeps one weight per 8 views.  sino is the
 * NATURAL [n_views][n_det] layout: cbp_forward_dihedral writes the shard's
 * rows only, cbp_back_dihedral reads them only (overwrites image, or adds
 * to it when accumulate != 0).  Device pointers only, 4-byte aligned;
 * CBP_EINVAL otherwise. */
int cbp_forward_dihedral(const cbp_geometry_t* g, const float* image, float* sino,
                         int32_t base_begin, int32_t base_count, void* stream);
int cbp_back_dihedral(const cbp_geometry_t* g, const float* sino, float* image,
                      int32_t base_begin, int32_t base_count, int32_t accumulate, void* stream);

/* ---- Row f1: building blocks of the iterative loops (SART, CGLS) around
 * the projector.  Device pointers, FP32 vectors of `count` elements,
 * stream-ordered; CBP_EINVAL for null pointers or negative counts.
 *
 * SART (the simultaneous ART step used inside ASD-POCS):
 *   c <- c + beta A^T((y - A c) ./ A1) ./ A^T 1, zero where a weight sum <= 1e-12,
 *   optionally clamped to c >= 0.                                            */
int cbp_sart_residual(const float* y, const float* ay, const float* rowsum, float* r,
                      int64_t count, void* stream);   /* r = (y - ay) ./ rowsum       */
int cbp_sart_update(float* c, const float* bp, const float* colsum, float beta,
                    int32_t nonneg, int64_t count, void* stream);  /* c += beta bp ./ colsum */
int cbp_fill(float* x, float value, int64_t count, void* stream);
/* <a, b> into the DEVICE double *out: deterministic two-stage FP64 sum.    */
int cbp_dot(const float* a, const float* b, int64_t count, double* out, void* stream);
/* CGLS (conjugate gradients on A^T A x = A^T y) with device-resident FP64
 * scalars, so an iteration never waits for the host:
 *   cbp_cgls_step:       x += (num/den) p (nx elements), r -= (num/den) q (nr)
 *   cbp_cgls_direction:  p = s + (num/den) p
 * (den == 0 leaves the vectors unchanged).                                  */
int cbp_cgls_step(float* x, const float* p, float* r, const float* q, const double* num,
                  const double* den, int64_t nx, int64_t nr, void* stream);
int cbp_cgls_direction(float* p, const float* s, const double* num, const double* den,
                       int64_t count, void* stream);

/* ---- Row f2: the paper's reference projector "Ref", FP64.
 *   sino[b][v][j] = sum_k image[b][k] (1/tau) int_{s_j - tau/2}^{s_j + tau/2} chord_k(s) ds
 * with chord_k(s) the length the ray from the source to detector coordinate s
 * cuts through the indicator pixel k (Eq. 10: the exact fan-beam transform of
 * the pixel basis, no blur), integrated by 8-point Gauss-Legendre between the
 * perspective images of the pixel corners (the integrand is smooth there).
 * An accuracy reference for the CNSF weights (Eq. 15 errors, Fig. 6-7), not
 * a hot path: ~100x the cost of cbp_forward.  image FP32 [batch][n][n],
 * sino FP64 [batch][view_count][n_det] (8-byte aligned); DEVICE pointers
 * only; stream-ordered.  CBP_EINVAL as cbp_forward, or for host pointers. */
int cbp_ref_forward(const cbp_geometry_t* g, const float* image, double* sino, int32_t batch,
                    int32_t view_begin, int32_t view_count, void* stream);

/* Its exact transpose, FP64 both sides: image[b][k] = sum_{v,j} sino[b][v][j]
 * W_ref(v, j, k) (overwrites image).  Device pointers only, 8-byte aligned. */
int cbp_ref_back(const cbp_geometry_t* g, const double* sino, double* image, int32_t batch,
                 int32_t view_begin, int32_t view_count, void* stream);

/* ---- Row f4: total variation and the steps of ASD-POCS (the
 * schedule is DESIGN.md ledger #21).  Device pointers; FP32 images
 * [batch][n][n]; scalars are DEVICE doubles (no host round trip).
 *   TV(x) = sum sqrt(dx^2 + dy^2 + eps^2), dx, dy forward differences with a
 *   reflective boundary (ledger #20); differences in FP64.
 * cbp_tv_value:    *out = TV(x) summed over the batch (deterministic FP64 sum)
 * cbp_tv_gradient: grad = d TV / d x (its exact analytic gradient)
 * cbp_diff_norm2:  *out = |a - b|^2 over count elements (FP64)
 * cbp_tv_step:     x -= (*alpha) sqrt(*dp2) g / sqrt(*gg)  (unchanged if *gg == 0):
 *                  a normalised descent step of length alpha |data step|
 * cbp_asd_adapt:   *alpha *= alpha_red if sqrt(*dg2) > r_max sqrt(*dp2)
 * CBP_EINVAL for null pointers, n < 1, batch < 1, count < 0 or eps < 0.    */
int cbp_tv_value(const float* x, int32_t n, int32_t batch, double eps, double* out, void* stream);
int cbp_tv_gradient(const float* x, float* grad, int32_t n, int32_t batch, double eps, void* stream);
int cbp_diff_norm2(const float* a, const float* b, int64_t count, double* out, void* stream);
int cbp_tv_step(float* x, const float* g, int64_t count, const double* gg, const double* alpha,
                const double* dp2, void* stream);
int cbp_asd_adapt(double* alpha, const double* dp2, const double* dg2, double r_max, double alpha_red,
                  void* stream);

/* Adjoint identity check on the current device (synchronous): draws seeded
 * c, y ~ U[0,1) (splitmix64), runs cbp_forward and cbp_back over all views,
 * and returns |<Ac,y> - <c,A^T y>| / |<Ac,y>| with FP64 inner products in
 * *rel_defect.  CBP_EINVAL for an invalid geometry or null rel_defect. */
int cbp_adjoint_check(const cbp_geometry_t* g, uint64_t seed, double* rel_defect);

/* Static description of an error code (never NULL). */
const char* cbp_strerror(int code);

/* ABI version (major * 10000 + minor * 100 + patch). */
int cbp_version(void);

/* Number of CUDA kernels this library has launched in this process (all
 * devices, all threads); instrumentation for the benchmark's launch count. */
uint64_t cbp_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CBP_H */
