// cbp_vec.cuh -- row f1: the elementwise and reduction steps of the SART and
// CGLS loops around the projector.  All
// HBM-bound: grid-stride, float4 where aligned, one pass each.  Reductions
// are deterministic (fixed per-block partial order, FP64 partials, one final
// block).
#pragma once

#include "cbp_common.cuh"

namespace cbp {

constexpr int VEC_BLOCK = 256;
constexpr int DOT_BLOCKS = 592;  // 148 SMs x 4

// SART residual: r = (y - Ac) / rowsum, 0 where rowsum <= 1e-12
__global__ void cbp_sart_residual_kernel(const float* __restrict__ y, const float* __restrict__ ay,
                                         const float* __restrict__ rowsum, float* __restrict__ r,
                                         int64_t count)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float w = rowsum[i];
        r[i] = w > 1e-12f ? (y[i] - ay[i]) / w : 0.0f;
    }
}

// SART update: c += beta * bp / colsum (0 where colsum <= 1e-12),
// then optionally c = max(c, 0)
__global__ void cbp_sart_update_kernel(float* __restrict__ c, const float* __restrict__ bp,
                                       const float* __restrict__ colsum, float beta, int nonneg,
                                       int64_t count)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float w = colsum[i];
        float v = c[i] + (w > 1e-12f ? beta * bp[i] / w : 0.0f);
        if (nonneg) v = fmaxf(v, 0.0f);
        c[i] = v;
    }
}

__global__ void cbp_fill_kernel(float* __restrict__ x, float v, int64_t count)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

// stage 1 of <a, b>: DOT_BLOCKS FP64 partials, each over a fixed index set
__global__ void __launch_bounds__(VEC_BLOCK) cbp_dot_partial_kernel(const float* __restrict__ a,
                                                                    const float* __restrict__ b,
                                                                    int64_t count,
                                                                    double* __restrict__ part)
{
    __shared__ double red[VEC_BLOCK];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        s += (double)a[i] * (double)b[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = VEC_BLOCK / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// stage 2: out = sum of the partials (one block, fixed order)
__global__ void __launch_bounds__(VEC_BLOCK) cbp_dot_final_kernel(const double* __restrict__ part,
                                                                  int nparts, double* __restrict__ out)
{
    __shared__ double red[VEC_BLOCK];
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += VEC_BLOCK) s += part[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = VEC_BLOCK / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// CGLS vector updates with device-resident FP64 scalars (no host round trip):
//   mode 0:  x += (num/den) p,  r -= (num/den) q        (alpha = gamma / |q|^2)
//   mode 1:  p = s + (num/den) p                         (beta = gamma_new / gamma)
// den == 0 (converged) leaves the vectors unchanged.
__global__ void cbp_cgls_step_kernel(float* __restrict__ x, const float* __restrict__ p,
                                     float* __restrict__ r, const float* __restrict__ q,
                                     const double* __restrict__ num, const double* __restrict__ den,
                                     int64_t nx, int64_t nr)
{
    const double d = *den;
    const float a = d > 0.0 ? (float)(*num / d) : 0.0f;
    const int64_t n = nx > nr ? nx : nr;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < nx) x[i] = fmaf(a, p[i], x[i]);
        if (i < nr) r[i] = fmaf(-a, q[i], r[i]);
    }
}

__global__ void cbp_cgls_dir_kernel(float* __restrict__ p, const float* __restrict__ s,
                                    const double* __restrict__ num, const double* __restrict__ den,
                                    int64_t count)
{
    const double d = *den;
    const float b = d > 0.0 ? (float)(*num / d) : 0.0f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = fmaf(b, p[i], s[i]);
}

// ---- row f4: total variation and the ASD-POCS steps ------------------------
// TV(x) = sum sqrt(dx^2 + dy^2 + eps^2), forward differences, reflective
// boundary (DESIGN.md ledger #20); differences and roots in FP64 (the inputs
// are FP32, so each difference is exact).
__device__ __forceinline__ double tv_term_at(const float* x, int n, int r, int c, double eps2, double& dx,
                                             double& dy)
{
    const size_t i = (size_t)r * n + c;
    const double v = x[i];
    dx = c + 1 < n ? (double)x[i + 1] - v : 0.0;
    dy = r + 1 < n ? (double)x[i + n] - v : 0.0;
    return sqrt(dx * dx + dy * dy + eps2);
}

// grad[b][r][c] = d TV / d x[b][r][c]
__global__ void cbp_tv_gradient_kernel(const float* __restrict__ x, float* __restrict__ grad, int n,
                                       int64_t count, double eps)
{
    const double eps2 = eps * eps;
    const int64_t plane = (int64_t)n * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float* xb = x + (i / plane) * plane;
        const int r = (int)((i % plane) / n), c = (int)(i % n);
        double dx, dy;
        const double m = tv_term_at(xb, n, r, c, eps2, dx, dy);
        double gsum = -(dx + dy) / m;
        if (c > 0) {  // left neighbour's term, through its dx
            const double ml = tv_term_at(xb, n, r, c - 1, eps2, dx, dy);
            gsum += dx / ml;
        }
        if (r > 0) {  // upper neighbour's term, through its dy
            const double mu = tv_term_at(xb, n, r - 1, c, eps2, dx, dy);
            gsum += dy / mu;
        }
        grad[i] = (float)gsum;
    }
}

// FP64 partial sums over a fixed index set per block: mode 0 = TV terms,
// mode 1 = (a - b)^2
__global__ void __launch_bounds__(VEC_BLOCK) cbp_sum_partial_kernel(const float* __restrict__ a,
                                                                    const float* __restrict__ b, int n,
                                                                    int64_t count, double eps, int mode,
                                                                    double* __restrict__ part)
{
    __shared__ double red[VEC_BLOCK];
    double s = 0.0;
    const int64_t plane = (int64_t)n * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (mode == 0) {
            double dx, dy;
            s += tv_term_at(a + (i / plane) * plane, n, (int)((i % plane) / n), (int)(i % n), eps * eps, dx, dy);
        } else {
            const double d = (double)a[i] - (double)b[i];
            s += d * d;
        }
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = VEC_BLOCK / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// x -= alpha sqrt(dp2) g / sqrt(gg)  (a normalised TV descent step of length
// alpha |data step|); gg == 0 leaves x unchanged
__global__ void cbp_tv_step_kernel(float* __restrict__ x, const float* __restrict__ g, int64_t count,
                                   const double* __restrict__ gg, const double* __restrict__ alpha,
                                   const double* __restrict__ dp2)
{
    const double n2 = *gg;
    const float a = n2 > 0.0 ? (float)(*alpha * sqrt(*dp2) / sqrt(n2)) : 0.0f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = fmaf(-a, g[i], x[i]);
}

// alpha *= alpha_red when |TV steps| > r_max |data step|
__global__ void cbp_asd_adapt_kernel(double* alpha, const double* dp2, const double* dg2, double r_max,
                                     double alpha_red)
{
    if (threadIdx.x == 0 && blockIdx.x == 0 && sqrt(*dg2) > r_max * sqrt(*dp2)) *alpha *= alpha_red;
}

}  // namespace cbp
