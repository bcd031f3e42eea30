/*
 * cnsf_oracle.h -- plain FP64 CPU oracle for the CNSF fan-beam projector of
 * Zhang & Entezari, "A Convolutional Forward and Back-Projection Model for
 * Fan-Beam Geometry" (arXiv 1907.10526).  Citations "P:n" are lines of the
 * paper text, "S:n" lines of SPEC.md, "ledger #k" the readings
 * listed in DESIGN.md section 3.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (include/, the
 * paper_1907_10526_b200 package, libcbp.so) may include, link or call this
 * code; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs use it.  It shares no header, helper, table or
 * constant with the CUDA path.
 */
#ifndef CNSF_ORACLE_H
#define CNSF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The oracle's own description of the scanner.  All
 * lengths in mm.  Deliberately its own type: the CUDA path defines its own. */
typedef struct orc_geometry {
    int32_t n;          /* image is n x n pixels                                  */
    double  pixel;      /* pixel side h                                           */
    int32_t n_views;    /* theta_v = 2 pi v / n_views (ledger #9)                 */
    int32_t n_det;      /* N_s bins, centres s_j = (j - (N_s-1)/2) * det_pitch    */
    double  det_pitch;  /* Delta_s                                                */
    double  det_width;  /* tau, bin width used by the blur (Eq. 2)                */
    double  sid;        /* D_po, source to rotation centre                        */
    double  sdd;        /* D_ps, source to detector; D_so = D_ps - D_po           */
    int32_t kind;       /* 0 = fan beam, flat detector (the paper's case);
                           1 = parallel beam (Eq. 9-10, row f3): rays along -u through
                               s e, sid and sdd unused;
                           2 = fan beam, arc detector (row f3): the detector is
                               the circle of radius D_ps about the source, s is the arc
                               length (angle s / D_ps from the central ray), det_pitch
                               and det_width are arc lengths                        */
    int32_t model;      /* 0 = the paper's CNSF weight (Eq. 14, per bin ray, effective
                               blur in the object plane);
                           1 = the magnified-footprint variant (row f3, BASELINE.json's
                               prose): the pixel's box-spline footprint mapped onto the
                               detector by the perspective map linearised at the pixel
                               centre, convolved with the detector cell            */
} orc_geometry;

/* --- geometry steps (Eq. 4, Eq. 11, Eq. 13) ---------------------- */
void   orc_view_frame(const orc_geometry* g, double theta,
                      double u[2], double e[2], double p[2]);
void   orc_detector_point(const orc_geometry* g, double theta, double s, double q[2]);
void   orc_ray_frame(const orc_geometry* g, double theta, double s,
                     double v[2], double r[2]);
double orc_perspective_project(const orc_geometry* g, double theta, const double x[2]);
double orc_effective_blur(const orc_geometry* g, double theta, double s, const double k[2]);
void   orc_pixel_center(const orc_geometry* g, int32_t row, int32_t col, double k[2]);
double orc_bin_center(const orc_geometry* g, int32_t j);
double orc_view_angle(const orc_geometry* g, int32_t v);

/* --- box splines (Eq. 14) ---------------------------- */
int    orc_canonicalize(int32_t m, const double* raw, double eps, double* out);
double orc_box_spline(int32_t m, const double* a, double x);

/* --- footprints: Eq. 12 (no blur) and Eq. 14 (blurred) for one pixel --------
 * Both return the projection of the INDICATOR pixel of side h centred at k
 * (ledger #4: factor h^2), evaluated on the ray of detector coordinate s. */
double orc_footprint(const orc_geometry* g, double theta, double s, const double k[2]);
double orc_weight(const orc_geometry* g, double theta, double s, const double k[2]);

/* --- projectors: Eq. 6 and its adjoint -------------------------------------
 * image: [batch][n][n] row-major, row 0 at +y (ledger #13)
 * sino : [batch][nv][n_det], view index local to [v0, v0+nv)
 * threads <= 0 means all hardware threads.  Deterministic for any thread
 * count (each output element has one owner and a fixed summation order).
 * Returns 0, or -1 on invalid arguments.                                      */
int orc_forward(const orc_geometry* g, const double* image, double* sino,
                int32_t batch, int32_t v0, int32_t nv, int32_t threads);
int orc_back(const orc_geometry* g, const double* sino, double* image,
             int32_t batch, int32_t v0, int32_t nv, int32_t threads);
/* back-projection restricted to a list of pixels (for sampled parity at full
 * size): out[b*npix + i] = sum_{v,j} sino[b][v][j] W(v, j, pix[i]) */
int orc_back_pixels(const orc_geometry* g, const double* sino, int32_t batch,
                    int32_t v0, int32_t nv, const int32_t* rows, const int32_t* cols,
                    int32_t npix, double* out, int32_t threads);
/* widen the candidate-bin margin by a factor (test hook: any superset of the
 * support must give identical results) */
void orc_set_candidate_margin_scale(double s);
/* number of nonzero weights (support test of Eq. 14) over views [v0, v0+nv) */
int64_t orc_count_weights(const orc_geometry* g, int32_t v0, int32_t nv, int32_t threads);
int orc_count_weights_per_view(const orc_geometry* g, int32_t v0, int32_t nv, int64_t* out,
                               int32_t threads);

/* --- row f2: the paper's reference projector "Ref" ------------
 * orc_ref_chord: exact chord of the ray of detector coordinate s through the
 *   indicator pixel of side h centred at k (Eq. 10, no blur).
 * orc_ref_weight: that chord averaged over [s - tau/2, s + tau/2] (adaptive
 *   Simpson between the projected corners, absolute tolerance 1e-14).
 * orc_ref_forward: y = A_ref c with these weights (layout as orc_forward;
 *   zero pixels are skipped, which is exact).                                 */
double orc_ref_chord(const orc_geometry* g, double theta, double s, const double k[2]);
double orc_ref_weight(const orc_geometry* g, double theta, double s, const double k[2]);
int orc_ref_forward(const orc_geometry* g, const double* image, double* sino,
                    int32_t batch, int32_t v0, int32_t nv, int32_t threads);
/* its transpose: image = A_ref^T sino (same weights)                          */
int orc_ref_back(const orc_geometry* g, const double* sino, double* image,
                 int32_t batch, int32_t v0, int32_t nv, int32_t threads);

#ifdef __cplusplus
}
#endif
#endif
