// cbp.cu -- the C ABI of include/cbp.h: argument validation, per-geometry
// table cache (row a1), host-buffer staging, kernel launches.
//
// Built with: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3
//             -Xcompiler -fPIC -shared  (see paper_1907_10526_b200/build.py)
#include "cbp.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "cbp_bp.cuh"
#include "cbp_common.cuh"
#include "cbp_fp.cuh"
#include "cbp_mag.cuh"
#include "cbp_ref.cuh"
#include "cbp_tables.cuh"
#include "cbp_vec.cuh"

namespace {

std::atomic<uint64_t> g_launches{0};

// launch with programmatic dependent launch allowed (cbp_common.cuh): the
// kernel may start during its stream predecessor's tail; CBP_NO_PDL turns it off
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args)
{
    static const bool off = getenv("CBP_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = off ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

bool finite_pos(double x) { return std::isfinite(x) && x > 0.0; }

cbp::GeomDev to_dev(const cbp_geometry_t& g)
{
    cbp::GeomDev d;
    d.n = g.n;
    d.n_views = g.n_views;
    d.n_det = g.n_det;
    d.h = g.pixel;
    d.pitch = g.det_pitch;
    d.tau = g.det_width;
    d.sid = g.sid;
    d.sdd = g.sdd;
    d.parallel = g.kind == CBP_PARALLEL ? 1 : 0;
    d.arc = g.kind == CBP_FAN_ARC ? 1 : 0;
    d.c0 = 0.5 * (double)(g.n - 1);
    d.cs = 0.5 * (double)(g.n_det - 1);
    return d;
}

// the accumulate mode of the second and later launches into one output
int acc_next(int32_t accumulate) { return accumulate == CBP_ACC_MULTIMEM ? CBP_ACC_MULTIMEM : 1; }

// ---- per-(geometry, device) tables --------------------------------------
struct TableKey {
    int device;
    int32_t kind;
    int32_t n_views, n_det;
    double pitch, tau, sdd;
    bool operator<(const TableKey& o) const
    {
        return std::memcmp(this, &o, sizeof(TableKey)) < 0;
    }
};

struct TableSet {
    double2* view_cs = nullptr;
    double2* bin_d = nullptr;
    float4* bin_f = nullptr;
};

std::mutex g_table_mu;
std::map<TableKey, TableSet> g_tables;

int get_tables(const cbp_geometry_t& g, cudaStream_t stream, cbp::Tables& out)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return CBP_ECUDA;
    TableKey key;
    std::memset(&key, 0, sizeof(key));
    key.device = dev;
    key.kind = g.kind;
    key.n_views = g.n_views;
    key.n_det = g.n_det;
    key.pitch = g.det_pitch;
    key.tau = g.det_width;
    key.sdd = g.sdd;
    std::lock_guard<std::mutex> lock(g_table_mu);
    auto it = g_tables.find(key);
    if (it == g_tables.end()) {
        TableSet ts;
        if (cudaMalloc(&ts.view_cs, sizeof(double2) * g.n_views) != cudaSuccess ||
            cudaMalloc(&ts.bin_d, sizeof(double2) * g.n_det) != cudaSuccess ||
            cudaMalloc(&ts.bin_f, sizeof(float4) * g.n_det) != cudaSuccess) {
            cudaFree(ts.view_cs);
            cudaFree(ts.bin_d);
            cudaFree(ts.bin_f);
            cudaGetLastError();
            return CBP_ECUDA;
        }
        const int m = g.n_views > g.n_det ? g.n_views : g.n_det;
        cbp::cbp_tables_kernel<<<(m + 127) / 128, 128, 0, stream>>>(to_dev(g), ts.view_cs,
                                                                    ts.bin_d, ts.bin_f);
        ++g_launches;
#ifdef CBP_DEBUG_CHECKS
        fprintf(stderr, "tables kernel: %s\n", cudaGetErrorString(cudaStreamSynchronize(stream)));
#endif
        if (cudaGetLastError() != cudaSuccess) return CBP_ECUDA;
        // tables are shared across streams: finish building before publishing
        if (cudaStreamSynchronize(stream) != cudaSuccess) return CBP_ECUDA;
        it = g_tables.emplace(key, ts).first;
    }
    out.view_cs = it->second.view_cs;
    out.bin_d = it->second.bin_d;
    out.bin_f = it->second.bin_f;
    return CBP_OK;
}

// ---- BP pair order per ray-direction bucket (device-resident, per device) --
// For bucket b (ray direction phi_b = (b + 1/2) pi / BP_BUCKETS, physical
// angle) the 512 pixel pairs of a 32 x 32 tile -- horizontal pairs when the
// rays are within 45 degrees of the x axis, else vertical -- sorted by the
// lateral coordinate of their centre, col sin(phi) + row cos(phi) (row axis
// pointing down = -y).  Entry = r * 32 + c of the pair's first pixel.
std::mutex g_pairs_mu;
std::map<int, uint16_t*> g_pairs;

int get_pair_order(const uint16_t** out)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return CBP_ECUDA;
    std::lock_guard<std::mutex> lock(g_pairs_mu);
    auto it = g_pairs.find(dev);
    if (it == g_pairs.end()) {
        const int NP = cbp::BP_PAIRS, T = cbp::BP_TILE;
        std::vector<uint16_t> host((size_t)cbp::BP_BUCKETS * NP);
        for (int b = 0; b < cbp::BP_BUCKETS; ++b) {
            const double phi = (b + 0.5) * 3.14159265358979323846 / cbp::BP_BUCKETS;
            const bool horiz = cbp::bucket_horiz(b);
            std::vector<std::pair<double, int>> key;
            for (int a = 0; a < T; ++a)
                for (int q = 0; q < T / 2; ++q) {
                    const int r = horiz ? a : 2 * q, c = horiz ? 2 * q : a;
                    const double cc = c + (horiz ? 0.5 : 0.0), rr = r + (horiz ? 0.0 : 0.5);
                    key.emplace_back(cc * std::sin(phi) + rr * std::cos(phi), r * T + c);
                }
            std::stable_sort(key.begin(), key.end(),
                             [](const std::pair<double, int>& x, const std::pair<double, int>& y) {
                                 return x.first < y.first;
                             });
            for (int i = 0; i < NP; ++i) host[(size_t)b * NP + i] = (uint16_t)key[i].second;
        }
        uint16_t* d = nullptr;
        if (cudaMalloc(&d, host.size() * sizeof(uint16_t)) != cudaSuccess ||
            cudaMemcpy(d, host.data(), host.size() * sizeof(uint16_t), cudaMemcpyHostToDevice) !=
                cudaSuccess) {
            cudaFree(d);
            cudaGetLastError();
            return CBP_ECUDA;
        }
        it = g_pairs.emplace(dev, d).first;
    }
    *out = it->second;
    return CBP_OK;
}

// ---- host-buffer staging workspace --------------------------------------
struct Workspace {
    void* buf[2] = {nullptr, nullptr};
    size_t cap[2] = {0, 0};
};
std::mutex g_ws_mu;
std::map<int, Workspace> g_ws;

int ws_get(Workspace& w, int slot, size_t bytes, void** p)
{
    if (w.cap[slot] < bytes) {
        cudaFree(w.buf[slot]);
        w.buf[slot] = nullptr;
        w.cap[slot] = 0;
        if (cudaMalloc(&w.buf[slot], bytes) != cudaSuccess) {
            cudaGetLastError();
            return CBP_ECUDA;
        }
        w.cap[slot] = bytes;
    }
    *p = w.buf[slot];
    return CBP_OK;
}

// 1 = device (or managed) memory on the current device, 0 = host, -1 = error
int pointer_kind(const void* p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return 0;  // unknown to CUDA: plain host memory
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
        int dev = 0;
        cudaGetDevice(&dev);
        return a.device == dev ? 1 : -1;
    }
    return 0;
}

int check_common(const cbp_geometry_t* g, const void* a, const void* b, int32_t batch,
                 int32_t view_begin, int32_t view_count)
{
    if (cbp_validate(g) != CBP_OK) return CBP_EINVAL;
    if (!a || !b || batch < 1 || view_count < 1 || view_begin < 0 ||
        (int64_t)view_begin + view_count > g->n_views)
        return CBP_EINVAL;
    if (((uintptr_t)a & 3) || ((uintptr_t)b & 3)) return CBP_EINVAL;
    return CBP_OK;
}

// stream-ordered scratch from the library's own memory pool per device
// (freed blocks are kept for reuse: release threshold UINT64_MAX on this
// private pool only, so other cudaMallocAsync users of the process keep the
// default pool's behaviour); the device's default pool if creation fails
int scratch_alloc(void** p, size_t bytes, cudaStream_t stream)
{
    static std::once_flag once[64];
    static cudaMemPool_t pools[64];
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(once[dev & 63], [dev] {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            pools[dev & 63] = pool;
        } else {
            cudaGetLastError();
            pools[dev & 63] = nullptr;
        }
    });
    const cudaError_t e = pools[dev & 63] ? cudaMallocFromPoolAsync(p, bytes, pools[dev & 63], stream)
                                          : cudaMallocAsync(p, bytes, stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return CBP_ECUDA;
    }
    return CBP_OK;
}

// width of the zero border around the image for the FP kernel: the largest
// per-line candidate count K = floor(2 sigma_q) + 1 any ray can have, with
// sigma_q = (A + C + tau') / (2 A) <= 1 + tau'_max / (sqrt(2) h) and
// tau'_max <= (tau / D_ps) (D_po + n h / sqrt(2))
// tau' > 0 at every pixel of the padded grid for every ray, so the FP walk
// needs no clamp before 1 / tau' (cbp_fp_kernel's CLAMP = false): tau' =
// g_j (k - p).v_j with g_j > 0 and (k - p).v_j >= D_po D_ps / L_j - R_pad on
// the flat detector (D_po cos(gamma_j) - R_pad on the arc; parallel beam:
// tau' = tau), R_pad = sqrt(2) ((n - 1) / 2 + P) h the padded grid's corner
bool fp_tau_positive(const cbp_geometry_t& g, int P)
{
    if (g.kind == CBP_PARALLEL) return true;
    const double rpad = std::sqrt(2.0) * (0.5 * (g.n - 1) + P) * g.pixel;
    const double smax = 0.5 * (g.n_det - 1) * g.det_pitch;
    const double dmin = g.kind == CBP_FAN_ARC ? g.sid * std::cos(std::min(smax / g.sdd, 1.5))
                                              : g.sid * g.sdd / std::sqrt(g.sdd * g.sdd + smax * smax);
    static const bool always = getenv("CBP_FP_CLAMP") != nullptr;  // test knob: the clamped walk everywhere
    return !always && dmin - rpad > 1e-6 * g.sid;
}

int fp_pad_width(const cbp_geometry_t& g)
{
    const double gmax = g.kind == CBP_FAN_ARC ? 2.0 * std::tan(0.5 * g.det_width / g.sdd) : g.det_width / g.sdd;
    const double taumax = g.kind == CBP_PARALLEL ? g.det_width
                                                 : gmax * (g.sid + g.n * g.pixel / std::sqrt(2.0));
    const double sigq = 1.0 + taumax / (std::sqrt(2.0) * g.pixel);
    return (int)std::floor(2.0 * sigq) + 2;
}

// The precise mode (cbp_common.cuh cnsf_prec) for narrow
// bins: the FP32 weight carries s' and its knots with an absolute rounding of
// ~1e-7 h (several ulp after the kernels' affine steps), which a ramp of
// width tau' + C turns into a relative error ~1e-7 h / tau' on views with
// C -> 0.  narrow_ratio() is a lower bound on tau' / h over the field of view:
// tau' = g_j d with d >= D_po - R (R the circumscribed radius) and g_j >=
// tau D_ps / (D_ps^2 + s_max^2) (flat), tau / D_ps (arc), 1 (parallel, tau' = tau).
double narrow_ratio(const cbp_geometry_t& g)
{
    if (g.kind == CBP_PARALLEL) return g.det_width / g.pixel;
    const double R = 0.5 * (double)g.n * g.pixel * std::sqrt(2.0);
    const double smax = 0.5 * (double)(g.n_det - 1) * g.det_pitch + 0.5 * g.det_width;
    const double gmin = g.kind == CBP_FAN_ARC ? g.det_width / g.sdd
                                              : g.det_width * g.sdd / (g.sdd * g.sdd + smax * smax);
    return gmin * (g.sid - R) / g.pixel;
}

// below this tau'_min / h the FP32 path's weight error approaches the parity
// bar: measured (tools/narrow_sweep.py, profiles/r02_narrow_sweep.jsonl) the
// FP32 path stays <= 7e-6 relL2 / 2e-5 max down to a ratio of 0.0016 at n = 40,
// ~1e-6 at 0.02; the precise mode costs 3-10x.
// CBP_PRECISE=0/1 forces either mode
constexpr double CBP_NARROW_RATIO = 0.02;

bool precise(const cbp_geometry_t& g)
{
    const char* e = getenv("CBP_PRECISE");  // read per call: tests switch it at run time
    if (e && (e[0] == '0' || e[0] == '1')) return e[0] == '1';
    return narrow_ratio(g) < CBP_NARROW_RATIO;
}

// FP launch: PARTS warps per ray (cbp_fp_kernel) while the grid is short of
// ~8 waves of resident CTAs (config 2: 1.6 waves -> parts 4, FP -17 %;
// config 3: 6.5 waves -> parts 2; config 4 / 5: enough waves)
template <int S, bool PREC = false>
int launch_fp_kernel(cbp::FPParams& Pm, int views, int groups, cudaStream_t stream, bool noclamp = false)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static std::once_flag once[64];
    static int per_sm[64];
    std::call_once(once[dev & 63], [dev] {
        int k = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, cbp::cbp_fp_kernel<S, 1, PREC>, cbp::FP_BLOCK, 0) !=
                cudaSuccess || k < 1)
            k = 1;
        per_sm[dev & 63] = k;
    });
    static const int force = getenv("CBP_FP_PARTS") ? atoi(getenv("CBP_FP_PARTS")) : 0;  // tuning knob
    const int64_t slots = (int64_t)sms * per_sm[dev & 63];
    auto ctas = [&](int parts) {
        const int bins = cbp::fp_threads(parts) / parts;  // bins per CTA
        return (int64_t)((Pm.g.n_det + bins - 1) / bins) * views * groups;
    };
    int parts = 1;
    // fewer than 8 waves: split the lines (config 2: 4 parts, 0.181 vs 0.194 ms with 2;
    // config 3: 2 parts, 1.228 vs 1.245 ms with 4; 16 waves picked 4 there)
    while (parts < 4 && ctas(parts) < 8 * slots) parts *= 2;
    // under two waves of 4-part CTAs (a view shard, a small image): 8 warps per
    // ray group in 256-thread CTAs, each walking an eighth of the lines
    // (measured at a W = 8 dihedral shard: config 2 0.092 -> 0.085 ms, config 3
    // 0.403 -> 0.384 ms; 16 parts in 512-thread CTAs: no further gain)
    if (parts == 4 && ctas(4) < 2 * slots) parts = 8;
    if (force == 1 || force == 2 || force == 4 || force == 8) parts = force;
    // views along x (the view-major CTA order of cbp_fp_kernel), detector tiles along y
    const int64_t tiles = ctas(parts) / ((int64_t)views * groups);
    if (tiles > 65535) return CBP_EINVAL;
    const dim3 grid(views, (unsigned)tiles, groups);
    if constexpr ((S == 4 || S == 1) && !PREC) {
        if (Pm.g.parallel) {  // tau' = tau: constant over every walk (CLAMP = 2)
            if (parts == 8)
                launch_pdl(cbp::cbp_fp_kernel<S, 8, PREC, 2>, grid, dim3(cbp::fp_threads(8)), 0, stream, Pm);
            else if (parts == 4)
                launch_pdl(cbp::cbp_fp_kernel<S, 4, PREC, 2>, grid, dim3(cbp::FP_BLOCK), 0, stream, Pm);
            else if (parts == 2)
                launch_pdl(cbp::cbp_fp_kernel<S, 2, PREC, 2>, grid, dim3(cbp::FP_BLOCK), 0, stream, Pm);
            else
                launch_pdl(cbp::cbp_fp_kernel<S, 1, PREC, 2>, grid, dim3(cbp::FP_BLOCK), 0, stream, Pm);
            ++g_launches;
            return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
        }
        if (noclamp) {  // tau' > 0 over the padded grid: the walk without the clamp
            if (parts == 8)
                launch_pdl(cbp::cbp_fp_kernel<S, 8, PREC, 0>, grid, dim3(cbp::fp_threads(8)), 0, stream, Pm);
            else if (parts == 4)
                launch_pdl(cbp::cbp_fp_kernel<S, 4, PREC, 0>, grid, dim3(cbp::FP_BLOCK), 0, stream, Pm);
            else if (parts == 2)
                launch_pdl(cbp::cbp_fp_kernel<S, 2, PREC, 0>, grid, dim3(cbp::FP_BLOCK), 0, stream, Pm);
            else
                launch_pdl(cbp::cbp_fp_kernel<S, 1, PREC, 0>, grid, dim3(cbp::FP_BLOCK), 0, stream, Pm);
            ++g_launches;
            return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
        }
    }
    if (parts == 8)
        launch_pdl(cbp::cbp_fp_kernel<S, 8, PREC>, grid, dim3(cbp::fp_threads(8)), 0, stream, Pm);
    else if (parts == 4)
        launch_pdl(cbp::cbp_fp_kernel<S, 4, PREC>, grid, dim3(cbp::FP_BLOCK), 0, stream, Pm);
    else if (parts == 2)
        launch_pdl(cbp::cbp_fp_kernel<S, 2, PREC>, grid, dim3(cbp::FP_BLOCK), 0, stream, Pm);
    else
        launch_pdl(cbp::cbp_fp_kernel<S, 1, PREC>, grid, dim3(cbp::FP_BLOCK), 0, stream, Pm);
    ++g_launches;
    return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
}

template <int S, bool PREC = false>
int launch_fp_s(const cbp_geometry_t& g, const cbp::Tables& t, const float* img, float* sino,
                int32_t batch, int32_t v0, int32_t nv, cudaStream_t stream)
{
    const int P = fp_pad_width(g);
    const int np = g.n + 2 * P;
    const int G = (batch + S - 1) / S;
    const size_t plane = (size_t)np * np * S * G;
    float* pad = nullptr;
    int rc = scratch_alloc((void**)&pad, sizeof(float) * 2 * plane, stream);
    if (rc != CBP_OK) return rc;
    float* padT = pad + plane;
    dim3 pgrid((np + cbp::PAD_TILE - 1) / cbp::PAD_TILE, (np + cbp::PAD_TILE - 1) / cbp::PAD_TILE, G);
    cbp::cbp_pad_kernel<S><<<pgrid, dim3(cbp::PAD_TILE, cbp::PAD_ROWS), 0, stream>>>(img, pad, padT, g.n, P, np,
                                                                         batch);
    ++g_launches;
    cbp::FPParams Pm;
    Pm.split = 0x7fffffff;
    Pm.view_begin2 = 0;
    Pm.sino2 = nullptr;
    Pm.g = to_dev(g);
    Pm.t = t;
    Pm.pad = pad;
    Pm.padT = padT;
    Pm.np = np;
    Pm.P = P;
    Pm.sino = sino;
    Pm.view_begin = v0;
    Pm.view_count = nv;
    Pm.batch = batch;
    Pm.sym_stride = 0;
    Pm.sym_mode = 0;
    Pm.rot_rows = 0;
    rc = launch_fp_kernel<S, PREC>(Pm, nv, G, stream, fp_tau_positive(g, P));
    cudaFreeAsync(pad, stream);
    return rc;
}

// a single image over a full scan of N_v = 4 m views: one weight serves the
// 4 views v, v + m, v + 2m, v + 3m (cbp_pad_sym4_kernel)
bool use_sym4(const cbp_geometry_t& g, int32_t batch, int32_t v0, int32_t nv)
{
    static const bool off = getenv("CBP_NO_SYMMETRY") != nullptr;
    return !off && g.model == CBP_MODEL_CNSF && batch == 1 && v0 == 0 && nv == g.n_views && g.n_views % 4 == 0 &&
           !precise(g);
}

// sino holds [4][base_count][n_det]: row q base_count + b is view
// base_begin + b + q n_views / 4
// stride 0: sino is the orbit layout [4][base_count][n_det]; stride n_views/4:
// sino is the natural [n_views][n_det] layout (rows base_begin + i + q n_views/4)
int launch_fp_sym4(const cbp_geometry_t& g, const cbp::Tables& t, const float* img, float* sino,
                   int32_t base_begin, int32_t base_count, cudaStream_t stream, int32_t stride = 0,
                   int32_t begin2 = 0, int32_t count2 = 0)
{
    const int P = fp_pad_width(g);
    const int np = g.n + 2 * P;
    const size_t plane = (size_t)np * np * 4;
    // rot_rows (opt-in, CBP_ROTROWS=1): column-major rays are walked as
    // row-major rays of the view a quarter turn on, so the transposed copy is
    // not needed (half the pad kernel's writes and of the FP's image
    // footprint).  Measured slower: config 2 FP 0.187 vs 0.177 ms, config 3
    // 1.271 vs 1.231, config 5 9.50 vs 9.32 (a warp's rays near 45 degrees
    // then walk two views' geometry: split access patterns)
    static const bool rot = getenv("CBP_ROTROWS") != nullptr;
    float* pad = nullptr;
    int rc = scratch_alloc((void**)&pad, sizeof(float) * (rot ? 1 : 2) * plane, stream);
    if (rc != CBP_OK) return rc;
    float* padT = rot ? nullptr : pad + plane;
    dim3 pgrid((np + cbp::PAD_TILE - 1) / cbp::PAD_TILE, (np + cbp::PAD_TILE - 1) / cbp::PAD_TILE, 1);
    if (rot)
        cbp::cbp_pad_sym4_kernel<false><<<pgrid, dim3(cbp::PAD_TILE, cbp::PAD4_ROWS), 0, stream>>>(img, pad, padT, g.n, P, np);
    else
        cbp::cbp_pad_sym4_kernel<true><<<pgrid, dim3(cbp::PAD_TILE, cbp::PAD4_ROWS), 0, stream>>>(img, pad, padT, g.n, P, np);
    ++g_launches;
    cbp::FPParams Pm;
    Pm.split = 0x7fffffff;
    Pm.view_begin2 = 0;
    Pm.sino2 = nullptr;
    Pm.g = to_dev(g);
    Pm.t = t;
    Pm.pad = pad;
    Pm.padT = padT;
    Pm.np = np;
    Pm.P = P;
    Pm.sino = stride ? sino + (size_t)base_begin * g.n_det : sino;
    Pm.view_begin = base_begin;
    Pm.view_count = base_count;
    Pm.batch = 4;
    Pm.sym_stride = stride ? stride : base_count;
    Pm.sym_mode = 4;
    Pm.rot_rows = rot ? 1 : 0;
    if (count2 > 0) {  // a second block of base views (natural layout only), same pad, same launch
        Pm.split = base_count;
        Pm.view_begin2 = begin2;
        Pm.sino2 = sino + (size_t)begin2 * g.n_det;
    }
    rc = launch_fp_kernel<4>(Pm, base_count + (count2 > 0 ? count2 : 0), 1, stream, fp_tau_positive(g, P));
    cudaFreeAsync(pad, stream);
    return rc;
}

// the full dihedral symmetry (rotations and the mirror): one weight serves 8
// views; a single image over a full scan of N_v = 8 m views
bool use_sym8(const cbp_geometry_t& g, int32_t batch, int32_t v0, int32_t nv)
{
    static const bool off = getenv("CBP_NO_MIRROR") != nullptr;
    return !off && use_sym4(g, batch, v0, nv) && g.n_views % 8 == 0;
}

int launch_fp_sym8(const cbp_geometry_t& g, const cbp::Tables& t, const float* img, float* sino,
                   cudaStream_t stream, int32_t base_begin = 0, int32_t base_count = -1)
{
    if (base_count < 0) base_count = g.n_views / 8 + 1 - base_begin;
    const int P = fp_pad_width(g);
    const int np = g.n + 2 * P;
    const size_t plane = (size_t)np * np * 8;
    float* pad = nullptr;
    int rc = scratch_alloc((void**)&pad, sizeof(float) * 2 * plane, stream);
    if (rc != CBP_OK) return rc;
    float* padT = pad + plane;
    dim3 pgrid((np + cbp::PAD_TILE - 1) / cbp::PAD_TILE, (np + cbp::PAD_TILE - 1) / cbp::PAD_TILE, 1);
    cbp::cbp_pad_sym8_kernel<<<pgrid, dim3(cbp::PAD_TILE, cbp::PAD_ROWS), 0, stream>>>(img, pad, padT, g.n, P, np);
    ++g_launches;
    cbp::FPParams Pm;
    Pm.split = 0x7fffffff;
    Pm.view_begin2 = 0;
    Pm.sino2 = nullptr;
    Pm.g = to_dev(g);
    Pm.t = t;
    Pm.pad = pad;
    Pm.padT = padT;
    Pm.np = np;
    Pm.P = P;
    Pm.sino = sino;
    Pm.view_begin = base_begin;
    Pm.view_count = base_count;
    Pm.batch = 8;
    Pm.sym_stride = 0;
    Pm.sym_mode = 8;
    Pm.rot_rows = 0;
    rc = launch_fp_kernel<8>(Pm, base_count, 1, stream);
    cudaFreeAsync(pad, stream);
    return rc;
}

// the magnified-footprint model over a full scan of one image with N_v % 4 == 0
// and an even grid: one footprint serves 4 views (the quadrant of pixels x
// the 4 rotations)
bool use_mag_sym4(const cbp_geometry_t& g, int32_t batch, int32_t v0, int32_t nv)
{
    static const bool off = getenv("CBP_NO_SYMMETRY") != nullptr;
    return !off && g.model == CBP_MODEL_MAG && batch == 1 && v0 == 0 && nv == g.n_views && g.n_views % 4 == 0 &&
           g.n % 2 == 0 && !precise(g);
}

// frames per footprint of the symmetric magnified-footprint BP: 8 (the
// dihedral triangle) once it has enough pixels to fill the GPU, else 4 (the
// quadrant): measured config 2 (n = 512) 0.66 vs 0.73 ms for 4 vs 8,
// config 3 (n = 1024) 4.86 vs 4.30 ms
int mag_bp_fold(const cbp_geometry_t& g)
{
    static const int force = getenv("CBP_MAG_BP_FOLD") ? atoi(getenv("CBP_MAG_BP_FOLD")) : 0;  // tuning knob
    if (force == 4 || force == 8) return force;
    const int64_t half = g.n / 2;
    return half * (half + 1) / 2 >= 100000 ? 8 : 4;
}

// view groups per pixel of the magnified-footprint BP: enough threads for
// ~256 k (about 14 resident warps per SM), at most MAG_BP_VG
int mag_bp_groups(int64_t pixels)
{
    int vg = 1;
    while (vg < cbp::MAG_BP_VG && pixels * vg < (256 << 10)) vg *= 2;
    return vg;
}

// Row f3, the magnified-footprint model (cbp_mag.cuh).  sigma_max bounds
// every pixel's support half-width (A + tau + C) / 2 <= (sqrt(2) h |grad P| + tau) / 2
// over the field of view's circumscribed disk (radius R): |grad P| = D_ps |k - p| / depth^2
// <= D_ps (D_po + R) / (D_po - R)^2 on the flat detector, D_ps / |k - p| <= D_ps / (D_po - R)
// on the arc, 1 in parallel beam.  fp: img -> sino; else sino -> img (BP).
int launch_mag(const cbp_geometry_t& g, const cbp::Tables& t, const float* img, float* sino, int32_t batch,
               int32_t v0, int32_t nv, int32_t accumulate, cudaStream_t stream, bool fp)
{
    const double R = 0.5 * (double)g.n * g.pixel * std::sqrt(2.0);
    double gmax = 1.0;
    if (g.kind == CBP_FAN_FLAT) gmax = g.sdd * (g.sid + R) / ((g.sid - R) * (g.sid - R));
    if (g.kind == CBP_FAN_ARC) gmax = g.sdd / (g.sid - R);
    cbp::MagParams P;
    P.g = to_dev(g);
    P.view_cs = t.view_cs;
    P.view_begin = v0;
    P.view_count = nv;
    P.batch = batch;
    P.accumulate = accumulate;  // 0, 1 or CBP_ACC_MULTIMEM
    P.vg = 1;
    P.sigma_max = 0.5 * (std::sqrt(2.0) * g.pixel * gmax + g.det_width) * (1.0 + 1e-9);
    const bool sym4 = use_mag_sym4(g, batch, v0, nv);
    P.image = nullptr;
    P.sino = nullptr;
    P.sino_in = nullptr;
    P.image_out = nullptr;
    P.pad4 = nullptr;
    if (fp) {
        P.image = img;
        P.sino = sino;
        const int bins = (g.n_det + cbp::MAG_FP_BLOCK - 1) / cbp::MAG_FP_BLOCK;
        static const bool warp_walk = getenv("CBP_MAG_FP_BLOCKWALK") == nullptr;  // A/B knob
        if (precise(g)) {
            cbp::cbp_mag_fp_kernel<1, true><<<dim3(bins, nv, batch), cbp::MAG_FP_BLOCK, 0, stream>>>(P);
        } else if (sym4) {
            P.view_count = g.n_views / 4;
            float* pad4 = nullptr;
            if (warp_walk) {  // the 4 rotations interleaved per pixel (no border)
                const dim3 pgrid((g.n + cbp::PAD_TILE - 1) / cbp::PAD_TILE, (g.n + cbp::PAD_TILE - 1) / cbp::PAD_TILE);
                if (scratch_alloc((void**)&pad4, sizeof(float) * 4 * (size_t)g.n * g.n, stream) != CBP_OK)
                    return CBP_ENOMEM;
                cbp::cbp_pad_sym4_kernel<false><<<pgrid, dim3(cbp::PAD_TILE, cbp::PAD4_ROWS), 0, stream>>>(
                    img, pad4, nullptr, g.n, 0, g.n);
                ++g_launches;
                P.pad4 = pad4;
                cbp::cbp_mag_fpw_kernel<4><<<dim3(bins, g.n_views / 4, 1), cbp::MAG_FP_BLOCK, 0, stream>>>(P);
                ++g_launches;
                cudaFreeAsync(pad4, stream);
                return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
            }
            cbp::cbp_mag_fp_kernel<4><<<dim3(bins, g.n_views / 4, 1), cbp::MAG_FP_BLOCK, 0, stream>>>(P);
        } else {
            if (warp_walk)
                cbp::cbp_mag_fpw_kernel<1><<<dim3(bins, nv, batch), cbp::MAG_FP_BLOCK, 0, stream>>>(P);
            else
                cbp::cbp_mag_fp_kernel<1><<<dim3(bins, nv, batch), cbp::MAG_FP_BLOCK, 0, stream>>>(P);
        }
    } else {  // BP: img is the output image, sino the input sinogram
        P.sino_in = sino;
        P.image_out = const_cast<float*>(img);
        if (sym4) {  // all views; CTAs of 32 pixels x VG view groups
            const int64_t half = g.n / 2;
            const int fold = mag_bp_fold(g);
            const int64_t pix = fold == 8 ? half * (half + 1) / 2 : half * half;
            P.vg = mag_bp_groups(pix);
            const int per = cbp::MAG_BP_BLOCK / P.vg;  // pixels per CTA
            const dim3 grid((unsigned)((pix + per - 1) / per), 1);
            const size_t sm = P.vg > 1 ? sizeof(float) * fold * cbp::MAG_BP_BLOCK : 0;
            if (fold == 8)  // the dihedral fundamental triangle, 8 frames
                cbp::cbp_mag_bp_kernel<8><<<grid, cbp::MAG_BP_BLOCK, sm, stream>>>(P);
            else  // the top-left quadrant, 4 rotations
                cbp::cbp_mag_bp_kernel<4><<<grid, cbp::MAG_BP_BLOCK, sm, stream>>>(P);
        } else {
            const int64_t pix = (int64_t)g.n * g.n;
            P.vg = mag_bp_groups(pix * batch);
            const int per = cbp::MAG_BP_BLOCK / P.vg;
            const dim3 grid((unsigned)((pix + per - 1) / per), batch);
            const size_t sm = P.vg > 1 ? sizeof(float) * cbp::MAG_BP_BLOCK : 0;
            if (precise(g))
                cbp::cbp_mag_bp_kernel<1, true><<<grid, cbp::MAG_BP_BLOCK, sm, stream>>>(P);
            else
                cbp::cbp_mag_bp_kernel<1><<<grid, cbp::MAG_BP_BLOCK, sm, stream>>>(P);
        }
    }
    ++g_launches;
    return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
}

// slices per thread: the weight of a (view, bin, pixel) is computed once and
// applied to S images of the batch
int launch_fp(const cbp_geometry_t& g, const cbp::Tables& t, const float* img, float* sino,
              int32_t batch, int32_t v0, int32_t nv, cudaStream_t stream)
{
    if (g.model == CBP_MODEL_MAG) return launch_mag(g, t, img, sino, batch, v0, nv, 0, stream, true);
    if (precise(g)) return launch_fp_s<1, true>(g, t, img, sino, batch, v0, nv, stream);
    // FP: the 8-fold kernel needs 128 registers (8 slices x 2 lines); on
    // sm_100a the 4-fold one is faster, so the FP uses the mirror only when
    // CBP_FP_MIRROR is set
    static const bool fp_mirror = getenv("CBP_FP_MIRROR") != nullptr;
    if (fp_mirror && use_sym8(g, batch, v0, nv)) return launch_fp_sym8(g, t, img, sino, stream);
    if (use_sym4(g, batch, v0, nv)) return launch_fp_sym4(g, t, img, sino, 0, g.n_views / 4, stream);
    if (batch >= 4) return launch_fp_s<4>(g, t, img, sino, batch, v0, nv, stream);
    if (batch >= 2) return launch_fp_s<2>(g, t, img, sino, batch, v0, nv, stream);
    return launch_fp_s<1>(g, t, img, sino, batch, v0, nv, stream);
}

// Number of view groups the BP splits the views into (one CTA per tile,
// view group and slice group).  Each group costs a CTA's fixed overhead
// (accumulator setup, the S-plane epilogue) and a partial image set that
// cbp_reduce_kernel must read back, so the BP takes the FEWEST groups that
// still give >= 3 waves of the resident CTA slots (dynamic scheduling then
// balances the tail); small problems take as many groups as allowed.
// Measured on the B200 at config 2 (256 tiles, 91 base views, 296 slots):
// G = 3/4/5/6/8/12 -> BP 0.220/0.206/0.213/0.219/0.224/0.257 ms; the earlier
// whole-wave score picked 8.  Each group has >= 8 views (8 base views of a
// symmetric launch: a small dihedral shard of 12 base views measured 0.093 /
// 0.102 / 0.107 / 0.113 ms per pair with G = 1 / 2 / 3 / 4 -- the per-CTA
// setup and the partial planes outweigh the fuller wave) and the partial
// images are capped at 32 / slice_groups per slice.
int bp_groups(const cbp_geometry_t& g, int32_t slice_groups, int32_t nv, int slots)
{
    static const int Gforce = getenv("CBP_BP_GROUPS") ? atoi(getenv("CBP_BP_GROUPS")) : 0;  // tuning knob
    if (Gforce > 0) return std::max(1, std::min(Gforce, (int)nv));
    const int tiles = ((g.n + cbp::BP_TILE - 1) / cbp::BP_TILE) * ((g.n + cbp::BP_TILE - 1) / cbp::BP_TILE);
    const int gmax = std::max(1, std::min(std::min(nv / 8, 64), 32 / std::max(1, (int)slice_groups)));
    int G = 1;
    for (; G <= gmax; ++G) {
        const int vpg = (nv + G - 1) / G;
        const int Geff = (nv + vpg - 1) / vpg;
        if ((double)tiles * Geff * slice_groups >= 3.0 * slots) return Geff;
    }
    const int vpg = (nv + gmax - 1) / gmax;
    return (nv + vpg - 1) / vpg;
}

// ---- BP tile-view headers: they depend only on the geometry and the view
// range, so they are computed once and cached per device (up to 256 MB each,
// 1 GB in all -- config 5's 142 MB included, measured 85 us per call
// otherwise; larger sets are recomputed per call into stream scratch)
struct HdrKey {
    int device;
    int32_t n, n_views, n_det, kind, v0, nv;
    double pixel, pitch, tau, sid, sdd;
    bool operator<(const HdrKey& o) const { return std::memcmp(this, &o, sizeof(HdrKey)) < 0; }
};
std::mutex g_hdr_mu;
std::map<HdrKey, cbp::BPHeader*> g_hdrs;
size_t g_hdr_bytes = 0;

// *out: the headers of (g, [v0, v0 + nv)); *owned: the caller must free them
// (stream-ordered) after use
int get_headers(const cbp_geometry_t& g, const cbp::Tables& t, int32_t v0, int32_t nv, cudaStream_t stream,
                const cbp::BPHeader** out, cbp::BPHeader** owned)
{
    const int tiles = (g.n + cbp::BP_TILE - 1) / cbp::BP_TILE;
    const size_t bytes = sizeof(cbp::BPHeader) * tiles * tiles * nv;
    const dim3 grid(tiles * tiles, (nv + 127) / 128);
    *owned = nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return CBP_ECUDA;
    HdrKey key;
    std::memset(&key, 0, sizeof(key));
    key.device = dev;
    key.n = g.n;
    key.n_views = g.n_views;
    key.n_det = g.n_det;
    key.kind = g.kind;
    key.v0 = v0;
    key.nv = nv;
    key.pixel = g.pixel;
    key.pitch = g.det_pitch;
    key.tau = g.det_width;
    key.sid = g.sid;
    key.sdd = g.sdd;
    {
        std::lock_guard<std::mutex> lock(g_hdr_mu);
        auto it = g_hdrs.find(key);
        if (it != g_hdrs.end()) {
            *out = it->second;
            return CBP_OK;
        }
        cbp::BPHeader* d = nullptr;
        if (bytes <= (256ull << 20) && g_hdr_bytes + bytes <= (1ull << 30) && cudaMalloc(&d, bytes) != cudaSuccess) {
            cudaGetLastError();  // no room to cache them: build them per call below
            d = nullptr;
        }
        if (d) {
            cbp::cbp_bp_header_kernel<<<grid, 128, 0, stream>>>(to_dev(g), t, v0, nv, tiles, d);
            ++g_launches;
            // shared across streams: finish building before publishing
            if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(stream) != cudaSuccess) {
                cudaFree(d);
                return CBP_ECUDA;
            }
            g_hdrs.emplace(key, d);
            g_hdr_bytes += bytes;
            *out = d;
            return CBP_OK;
        }
    }
    if (scratch_alloc((void**)owned, bytes, stream) != CBP_OK) return CBP_ECUDA;
    cbp::cbp_bp_header_kernel<<<grid, 128, 0, stream>>>(to_dev(g), t, v0, nv, tiles, *owned);
    ++g_launches;
    *out = *owned;
    return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
}

// ---- the persistent BP's plan (cbp_bp_plan_kernel): the
// segments of an NB-CTA launch over (g, [v0, v0 + nv)).  Cached per device
// next to the cached headers; recomputed per call (stream scratch) when the
// headers are not cached.
std::map<std::pair<HdrKey, int>, int*> g_plans;

size_t plan_ints(int tiles, int NB) { return (size_t)(tiles + NB + 1) + (NB + 1) + (tiles + 1) + NB + (NB + 1); }

int build_plan(const cbp::BPHeader* hdrs, int tiles, int nv, int NB, int* plan, cudaStream_t stream)
{
    int* cum = nullptr;
    long long* pre = nullptr;
    if (scratch_alloc((void**)&cum, sizeof(int) * (size_t)tiles * nv, stream) != CBP_OK) return CBP_ENOMEM;
    if (scratch_alloc((void**)&pre, sizeof(long long) * (tiles + 1), stream) != CBP_OK) {
        cudaFreeAsync(cum, stream);
        return CBP_ENOMEM;
    }
    cbp::cbp_bp_plan_cost_kernel<<<tiles, 256, 0, stream>>>(hdrs, nv, cum, pre);
    cbp::cbp_bp_plan_kernel<<<1, 1024, 0, stream>>>(cum, pre, tiles, nv, NB, plan);
    g_launches += 2;
    cudaFreeAsync(cum, stream);
    cudaFreeAsync(pre, stream);
    return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
}

// *out: the plan; *owned: free it after use (stream-ordered)
int get_plan(const cbp_geometry_t& g, int32_t v0, int32_t nv, int NB, const cbp::BPHeader* hdrs, bool hdrs_cached,
             cudaStream_t stream, const int** out, int** owned)
{
    const int tiles1 = (g.n + cbp::BP_TILE - 1) / cbp::BP_TILE, tiles = tiles1 * tiles1;
    const size_t bytes = sizeof(int) * plan_ints(tiles, NB);
    *owned = nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return CBP_ECUDA;
    if (hdrs_cached) {
        HdrKey key;
        std::memset(&key, 0, sizeof(key));
        key.device = dev;
        key.n = g.n;
        key.n_views = g.n_views;
        key.n_det = g.n_det;
        key.kind = g.kind;
        key.v0 = v0;
        key.nv = nv;
        key.pixel = g.pixel;
        key.pitch = g.det_pitch;
        key.tau = g.det_width;
        key.sid = g.sid;
        key.sdd = g.sdd;
        std::lock_guard<std::mutex> lock(g_hdr_mu);
        auto it = g_plans.find({key, NB});
        if (it != g_plans.end()) {
            *out = it->second;
            return CBP_OK;
        }
        int* d = nullptr;
        if (cudaMalloc(&d, bytes) != cudaSuccess) {
            cudaGetLastError();  // no room to cache it: build it per call below
            d = nullptr;
        }
        if (d) {
            // shared across streams: finish building before publishing
            if (build_plan(hdrs, tiles, nv, NB, d, stream) != CBP_OK || cudaStreamSynchronize(stream) != cudaSuccess) {
                cudaFree(d);
                return CBP_ECUDA;
            }
            g_plans.emplace(std::make_pair(key, NB), d);
            *out = d;
            return CBP_OK;
        }
    }
    if (scratch_alloc((void**)owned, bytes, stream) != CBP_OK) return CBP_ENOMEM;
    *out = *owned;
    return build_plan(hdrs, tiles, nv, NB, *owned, stream);
}

// ---- BP orbit clusters: representative tiles of the orbits
// of the dihedral group on the T x T tile grid (n = 32 T), per device
std::mutex g_orbit_mu;
std::map<std::pair<int, int>, std::pair<int2*, int>> g_orbits;

int get_orbit_reps(int T, const int2** out, int* count)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return CBP_ECUDA;
    std::lock_guard<std::mutex> lock(g_orbit_mu);
    auto it = g_orbits.find({dev, T});
    if (it == g_orbits.end()) {
        std::vector<char> seen((size_t)T * T, 0);
        std::vector<int2> reps;
        for (int ty = 0; ty < T; ++ty)
            for (int tx = 0; tx < T; ++tx) {
                if (seen[(size_t)ty * T + tx]) continue;
                reps.push_back(make_int2(tx, ty));
                for (int q = 0; q < 8; ++q) {  // the same frames as frame_fwd on tile coordinates
                    int r = ty, c = tx;
                    if (q >> 2) r = T - 1 - r;
                    for (int k = 0; k < (q & 3); ++k) {
                        const int nr = T - 1 - c;
                        c = r;
                        r = nr;
                    }
                    seen[(size_t)r * T + c] = 1;
                }
            }
        int2* d = nullptr;
        if (cudaMalloc(&d, sizeof(int2) * reps.size()) != cudaSuccess ||
            cudaMemcpy(d, reps.data(), sizeof(int2) * reps.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(d);
            cudaGetLastError();
            return CBP_ECUDA;
        }
        it = g_orbits.emplace(std::make_pair(dev, T), std::make_pair(d, (int)reps.size())).first;
    }
    *out = it->second.first;
    *count = it->second.second;
    return CBP_OK;
}

// The dihedral BP as clusters of 8 CTAs over tile orbits: each output tile is
// summed from its orbit's frame accumulators through distributed shared
// memory, so there are no frame planes (8 per image and view group: 32 MB per
// launch at config 2, 128 MB at config 5) and, with one view group, no reduce
// kernel.  n must be a multiple of BP_TILE (frames map tiles onto tiles).
// Opt-in (CBP_ORBIT=1): measured slower than the frame planes -- config 2 BP
// 0.286-0.329 ms (G = 1..4) vs 0.192 ms, config 5 11.44 vs 9.48 ms: a
// cluster holds its 8 SM slots until its slowest member (the orbit's tiles
// see the base views from different sides) and clusters pack the GPCs less
// densely than single CTAs.
bool use_orbit(const cbp_geometry_t& g)
{
    const char* e = getenv("CBP_ORBIT");  // read per call: the tests compare both paths
    return e && e[0] == '1' && g.n % cbp::BP_TILE == 0;
}

int launch_bp_orbit(const cbp_geometry_t& g, const cbp::Tables& t, const float* sino, float* img, int32_t v0,
                    int32_t nv, int32_t accumulate, cudaStream_t stream, int images)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = cbp::bp_smem_bytes(8, false);
    static std::once_flag attr[64];
    static int per_sm[64];
    std::call_once(attr[dev & 63], [smem, dev] {
        cudaFuncSetAttribute(cbp::cbp_bp_kernel<8, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(cbp::cbp_bp_kernel<8, false, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
        int k = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, cbp::cbp_bp_kernel<8, false, true>, cbp::BP_THREADS,
                                                          smem) != cudaSuccess || k < 1)
            k = 1;
        per_sm[dev & 63] = k;
    });
    const int T = g.n / cbp::BP_TILE;
    const int2* reps = nullptr;
    int nrep = 0;
    if (get_orbit_reps(T, &reps, &nrep) != CBP_OK) return CBP_ECUDA;
    const int ctas = 8 * nrep;
    // view groups: the fewest with >= 3 waves of resident CTAs (as bp_groups)
    const char* genv = getenv("CBP_BP_GROUPS");  // tuning knob (read per call)
    const int Gforce = genv ? atoi(genv) : 0;
    const int slots = sms * per_sm[dev & 63];
    const int gmax = std::max(1, std::min(nv / 8, 16));
    int G = 1;
    while (G < gmax && (double)ctas * G * images < 3.0 * slots) ++G;
    if (Gforce > 0) G = std::max(1, std::min(Gforce, (int)nv));
    const int vpg = (nv + G - 1) / G;
    G = (nv + vpg - 1) / vpg;
    const bool mc_fused = accumulate == CBP_ACC_MULTIMEM;  // (the reduce-kernel multimem path is not needed here)
    const size_t plane = (size_t)g.n * g.n;
    float* part = nullptr;
    if (G > 1 && !mc_fused) {
        int rc = scratch_alloc((void**)&part, sizeof(float) * plane * G * images, stream);
        if (rc != CBP_OK) return rc;
    }
    cbp::BPParams P;
    std::memset(&P, 0, sizeof(P));
    const cbp::BPHeader* hdrs = nullptr;
    cbp::BPHeader* hdrs_owned = nullptr;
    if (get_pair_order(&P.pairs) != CBP_OK || get_headers(g, t, v0, nv, stream, &hdrs, &hdrs_owned) != CBP_OK) {
        if (part) cudaFreeAsync(part, stream);
        return CBP_ECUDA;
    }
    P.hdrs = hdrs;
    P.g = to_dev(g);
    P.t = t;
    P.sino = sino;
    P.out = part ? part : img;
    P.view_begin = v0;
    P.view_count = nv;
    P.groups = G;
    P.views_per_group = vpg;
    P.batch = 8;
    P.accumulate = (G == 1 && accumulate == CBP_ACC_ADD) ? 1 : 0;
    P.sym_stride = 0;
    P.sym_mode = 8;
    P.images = images;
    P.mc_fused = mc_fused ? 1 : 0;
    P.orbit_reps = reps;
    P.orbit_T = T;
    static const bool no_pdl = getenv("CBP_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas, 1, G * images);
    cfg.blockDim = dim3(cbp::BP_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 8;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, cbp::cbp_bp_kernel<8, false, true>, P);
    ++g_launches;
    if (hdrs_owned) cudaFreeAsync(hdrs_owned, stream);
    if (part) {
        const int blocks = (int)std::min<size_t>((plane / 4 + 255) / 256, (size_t)sms * 8 / images + 1);
        launch_pdl(cbp::cbp_reduce_kernel, dim3(std::max(blocks, 1), images), dim3(256), 0, stream,
                   (const float*)part, img, plane, G, accumulate == CBP_ACC_ADD ? 1 : 0);
        ++g_launches;
        cudaFreeAsync(part, stream);
    }
    return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
}

// CBP_BP_PROF=path (diagnostics, a -DCBP_BP_PROFILE build): the BP launches
// record per-CTA start / end times, SMs and header features; each launch
// appends "launch <ctas>" and one line per CTA to the file
unsigned long long* bp_prof_begin(size_t ctas)
{
#ifdef CBP_BP_PROFILE
    static const char* path = getenv("CBP_BP_PROF");
    if (!path) return nullptr;
    unsigned long long* d = nullptr;
    if (cudaMalloc(&d, 64 * ctas) != cudaSuccess) return nullptr;
    cudaMemset(d, 0, 64 * ctas);
    return d;
#else
    (void)ctas;
    return nullptr;  // the timeline is compiled in only with -DCBP_BP_PROFILE (tools/bp_cta_prof.py)
#endif
}
void bp_prof_end(unsigned long long* d, size_t ctas, cudaStream_t stream)
{
    if (!d) return;
    std::vector<unsigned long long> h(8 * ctas);
    cudaStreamSynchronize(stream);
    cudaMemcpy(h.data(), d, 64 * ctas, cudaMemcpyDeviceToHost);
    cudaFree(d);
    FILE* f = fopen(getenv("CBP_BP_PROF"), "a");
    if (!f) return;
    fprintf(f, "launch %zu\n", ctas);
    for (size_t i = 0; i < ctas; ++i)
        fprintf(f, "%llu %llu %llu %llu %llu %llu %llu\n", h[8 * i], h[8 * i + 1], h[8 * i + 2], h[8 * i + 3],
                h[8 * i + 4], h[8 * i + 5], h[8 * i + 6]);
    fclose(f);
}

// The persistent 8-frame BP: one wave of CTAs over cost-
// balanced segments of the (tile, base view) pairs, compact per-segment
// blocks, cbp_seg_reduce_kernel.  Opt-in (CBP_BP_SEG=1, read per call): it
// does ~5 % less work than the view-group grid but a static split cannot
// absorb the unequal progress of the two CTAs resident on an SM (measured:
// 1.4 % faster at config 2, 7 % slower at configs 3 and 5).
bool use_seg(const cbp_geometry_t& g, int32_t nv)
{
    const char* e = getenv("CBP_BP_SEG");
    if (!e || e[0] != '1') return false;
    const long long tiles = (g.n + cbp::BP_TILE - 1) / cbp::BP_TILE;
    return tiles * tiles * (long long)nv < (1LL << 30);
}

// (accumulate: CBP_ACC_OVERWRITE or CBP_ACC_ADD; the multicast mode keeps the grid)
int launch_bp_seg(const cbp_geometry_t& g, const cbp::Tables& t, const float* sino, float* img, int32_t v0,
                  int32_t nv, int32_t accumulate, cudaStream_t stream, int images)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = cbp::bp_smem_bytes(8, false);
    static std::once_flag attr[64];
    static int per_sm[64];
    std::call_once(attr[dev & 63], [smem, dev] {
        cudaFuncSetAttribute(cbp::cbp_bp_kernel<8, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        int k = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, cbp::cbp_bp_kernel<8, false, false, true>,
                                                          cbp::BP_THREADS, smem) != cudaSuccess || k < 1)
            k = 1;
        per_sm[dev & 63] = k;
    });
    const char* nbenv = getenv("CBP_BP_SEG_CTAS");  // tuning knob (read per call)
    const int NB = nbenv && atoi(nbenv) > 0 ? atoi(nbenv) : sms * per_sm[dev & 63];
    const int tiles1 = (g.n + cbp::BP_TILE - 1) / cbp::BP_TILE, tiles = tiles1 * tiles1;
    const cbp::BPHeader* hdrs = nullptr;
    cbp::BPHeader* hdrs_owned = nullptr;
    if (get_headers(g, t, v0, nv, stream, &hdrs, &hdrs_owned) != CBP_OK) return CBP_ECUDA;
    const int* plan = nullptr;
    int* plan_owned = nullptr;
    int rc = get_plan(g, v0, nv, NB, hdrs, hdrs_owned == nullptr, stream, &plan, &plan_owned);
    const int seg_max = tiles + NB;
    float* blocks = nullptr;
    if (rc == CBP_OK)
        rc = scratch_alloc((void**)&blocks, sizeof(float) * images * seg_max * 8 * cbp::BP_TILE * cbp::BP_TILE, stream);
    if (rc != CBP_OK) {
        if (hdrs_owned) cudaFreeAsync(hdrs_owned, stream);
        if (plan_owned) cudaFreeAsync(plan_owned, stream);
        return rc;
    }
    cbp::BPParams P;
    std::memset(&P, 0, sizeof(P));
    if (get_pair_order(&P.pairs) != CBP_OK) {
        if (hdrs_owned) cudaFreeAsync(hdrs_owned, stream);
        if (plan_owned) cudaFreeAsync(plan_owned, stream);
        cudaFreeAsync(blocks, stream);
        return CBP_ECUDA;
    }
    P.g = to_dev(g);
    P.t = t;
    P.hdrs = hdrs;
    P.sino = sino;
    P.out = blocks;
    P.sym_mode = 8;
    P.images = images;
    P.view_begin = v0;
    P.view_count = nv;
    P.groups = 1;
    P.views_per_group = nv;
    P.batch = 8;
    P.seg_idx = plan;
    P.cta_seg = plan + (tiles + NB + 1);
    P.seg_max = seg_max;
    P.prof = bp_prof_begin((size_t)NB * images);
    launch_pdl(cbp::cbp_bp_kernel<8, false, false, true>, dim3(NB, 1, images), dim3(cbp::BP_THREADS), smem, stream,
               P);
    ++g_launches;
    bp_prof_end(P.prof, (size_t)NB * images, stream);
    if (hdrs_owned) cudaFreeAsync(hdrs_owned, stream);
    {
        const size_t plane = (size_t)g.n * g.n;
        const int mode = accumulate ? 1 : 0;
        const int* seg_first = P.cta_seg + NB + 1;
        if (g.n % cbp::BP_TILE == 0) {
            launch_pdl(cbp::cbp_seg_reduce_kernel<8>, dim3(tiles, images), dim3(256), 0, stream,
                       (const float*)blocks, img, seg_first, g.n, seg_max, mode);
        } else {
            const int nblk = (int)std::min<size_t>((plane + 255) / 256, (size_t)sms * 8 / images + 1);
            launch_pdl(cbp::cbp_seg_reduce_px_kernel<8>, dim3(std::max(nblk, 1), images), dim3(256), 0, stream,
                       (const float*)blocks, img, seg_first, g.n, seg_max, mode);
        }
        ++g_launches;
        cudaFreeAsync(blocks, stream);
    }
    if (plan_owned) cudaFreeAsync(plan_owned, stream);
    return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
}

template <int S, bool PREC = false, int W = 0, bool PAR = false>
int launch_bp_s(const cbp_geometry_t& g, const cbp::Tables& t, const float* sino, float* img,
                int32_t batch, int32_t v0, int32_t nv, int32_t accumulate, cudaStream_t stream,
                int symmode = 0, int images = 1)
{
    // symmetric: 4 "slices" (the 4 rotated frames) of one image over the base
    // views [v0, v0 + nv), sinogram [4][nv][n_det]; or 8 frames (rotations
    // and mirror) over base views [0, n_views/8], natural sinogram
    const bool sym = symmode != 0;
    if constexpr (S == 8 && !PREC) {
        if (symmode == 8 && use_orbit(g)) return launch_bp_orbit(g, t, sino, img, v0, nv, accumulate, stream, images);
        if (symmode == 8 && accumulate != CBP_ACC_MULTIMEM && use_seg(g, nv))
            return launch_bp_seg(g, t, sino, img, v0, nv, accumulate, stream, images);
    }
    if (sym) batch = symmode;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int SG = sym ? images : (batch + S - 1) / S;
    const size_t smem = cbp::bp_smem_bytes(S, PREC, W);
    static std::once_flag attr[64];
    static int per_sm[64];
    std::call_once(attr[dev & 63], [smem, dev] {
        cudaFuncSetAttribute(cbp::cbp_bp_kernel<S, PREC, false, false, W, PAR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        int k = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, cbp::cbp_bp_kernel<S, PREC, false, false, W, PAR>, cbp::BP_THREADS,
                                                          smem) != cudaSuccess || k < 1)
            k = 1;
        per_sm[dev & 63] = k;
    });
    const int G = bp_groups(g, SG, nv, sms * per_sm[dev & 63]);
    const int vpg = (nv + G - 1) / G;
    const size_t plane = (size_t)g.n * g.n;
    float* part = nullptr;
    // CBP_ACC_MULTIMEM: by default the BP's epilogue adds every finished tile
    // (each frame, each view group) into the multicast image itself, so the
    // switch's reduction overlaps the tiles still computing (G x frames more
    // multicast traffic than one add of the reduced image); CBP_MC_REDUCE=1
    // sums the planes locally first and adds once from cbp_reduce_kernel
    static const bool mc_reduce = getenv("CBP_MC_REDUCE") != nullptr;
    const bool mc_fused = accumulate == CBP_ACC_MULTIMEM && !mc_reduce;
    const bool mc = accumulate == CBP_ACC_MULTIMEM && mc_reduce;  // through the reduce kernel
    if (!mc_fused && (G > 1 || sym || mc)) {
        int rc = scratch_alloc((void**)&part, sizeof(float) * plane * batch * G * (sym ? images : 1), stream);
        if (rc != CBP_OK) return rc;
    }
    cbp::BPParams P;
    std::memset(&P, 0, sizeof(P));
    if (get_pair_order(&P.pairs) != CBP_OK) {
        if (part) cudaFreeAsync(part, stream);
        return CBP_ECUDA;
    }
    const int tiles = (g.n + cbp::BP_TILE - 1) / cbp::BP_TILE;
    const cbp::BPHeader* hdrs = nullptr;
    cbp::BPHeader* hdrs_owned = nullptr;
    if (get_headers(g, t, v0, nv, stream, &hdrs, &hdrs_owned) != CBP_OK) {
        if (part) cudaFreeAsync(part, stream);
        return CBP_ECUDA;
    }
    P.hdrs = hdrs;
    P.g = to_dev(g);
    P.t = t;
    P.sino = sino;
    P.out = mc_fused ? img : ((G > 1 || sym || mc) ? part : img);
    P.mc_fused = mc_fused ? 1 : 0;
    P.orbit_reps = nullptr;
    P.orbit_T = 0;
    P.sym_stride = symmode == 4 ? nv : 0;
    P.sym_mode = symmode;
    P.images = sym ? images : 1;
    P.view_begin = v0;
    P.view_count = nv;
    P.groups = (G > 1 || sym || mc) ? G : 1;
    P.views_per_group = vpg;
    P.batch = batch;
    P.accumulate = (G == 1 && !sym && !mc && !mc_fused && accumulate) ? 1 : 0;
    P.hdr_ready = hdrs_owned == nullptr ? 1 : 0;  // cached: complete before this launch
    dim3 grid(tiles, tiles, G * SG);
#ifdef CBP_DEBUG_CHECKS
    fprintf(stderr, "launch_bp S=%d G=%d vpg=%d grid=%d,%d,%d smem=%zu\n", S, G, vpg, grid.x, grid.y,
            grid.z, smem);
#endif
    P.seg_idx = P.cta_seg = nullptr;
    P.seg_max = 0;
    P.prof = bp_prof_begin((size_t)grid.x * grid.y * grid.z);
    launch_pdl(cbp::cbp_bp_kernel<S, PREC, false, false, W, PAR>, grid, dim3(cbp::BP_THREADS), smem, stream, P);
    ++g_launches;
    bp_prof_end(P.prof, (size_t)grid.x * grid.y * grid.z, stream);
#ifdef CBP_DEBUG_CHECKS
    fprintf(stderr, "bp kernel: %s\n", cudaGetErrorString(cudaStreamSynchronize(stream)));
#endif
    if (hdrs_owned) cudaFreeAsync(hdrs_owned, stream);
    if (!mc_fused && (sym || G > 1 || mc)) {
        // symmetric: the G x S frame planes are already in output orientation
        const size_t count = sym ? plane : plane * batch;
        const int planes = sym ? G * batch : G;
        const int outs = sym ? images : 1;  // symmetric batch: one reduction per image
        const size_t lanes = planes >= 16 && planes % 32 == 0 ? count : count / 4;  // 4 lanes per float4 (quad)
        const int blocks = (int)std::min<size_t>((lanes + 255) / 256, (size_t)sms * 8 / outs + 1);
        launch_pdl(cbp::cbp_reduce_kernel, dim3(std::max(blocks, 1), outs), dim3(256), 0, stream,
                   (const float*)part, img, count, planes, mc ? 2 : (accumulate ? 1 : 0));
        ++g_launches;
        cudaFreeAsync(part, stream);
    }
    return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
}

// the wide chunk shape of the 8-frame BP (cbp::BPShape<1>: 4 views x 128
// bins) when a tile's projection is wide: its mean span in bins, 32 h m (4 /
// pi) / pitch with the magnification m = D_ps / D_po at the centre (the mean
// of |cos| + |sin| over directions is 4 / pi), above 68 -- config 2-5: 54
// (default shape), the paper's timing shapes: 81 (wide; BP 0.194 -> 0.163 ms
// at p512, 0.716 -> 0.567 at p1024; config 2 with the wide shape 0.187 ->
// 0.203).  CBP_BP_WIDE=0 / 1 forces it (read per call).
bool bp_wide(const cbp_geometry_t& g)
{
    const char* e = getenv("CBP_BP_WIDE");
    if (e && (e[0] == '0' || e[0] == '1')) return e[0] == '1';
    const double m = g.kind == CBP_PARALLEL ? 1.0 : g.sdd / g.sid;
    return cbp::BP_TILE * g.pixel * m * (4.0 / M_PI) / g.det_pitch > 68.0;
}

// the 8-frame BP over base views [v0, v0 + nv): the chunk shape (bp_wide)
// and, in parallel beam, the weight with tau' = tau (PAR)
int launch_bp_sym8(const cbp_geometry_t& g, const cbp::Tables& t, const float* sino, float* img, int32_t batch,
                   int32_t v0, int32_t nv, int32_t accumulate, cudaStream_t stream, int images)
{
    const bool wide = bp_wide(g), par = g.kind == CBP_PARALLEL;
    if (par)
        return wide ? launch_bp_s<8, false, 1, true>(g, t, sino, img, batch, v0, nv, accumulate, stream, 8, images)
                    : launch_bp_s<8, false, 0, true>(g, t, sino, img, batch, v0, nv, accumulate, stream, 8, images);
    return wide ? launch_bp_s<8, false, 1>(g, t, sino, img, batch, v0, nv, accumulate, stream, 8, images)
                : launch_bp_s<8>(g, t, sino, img, batch, v0, nv, accumulate, stream, 8, images);
}

int launch_bp(const cbp_geometry_t& g, const cbp::Tables& t, const float* sino, float* img,
              int32_t batch, int32_t v0, int32_t nv, int32_t accumulate, cudaStream_t stream)
{
    if (g.model == CBP_MODEL_MAG)
        return launch_mag(g, t, img, const_cast<float*>(sino), batch, v0, nv, accumulate, stream, false);
    if (precise(g)) return launch_bp_s<1, true>(g, t, sino, img, batch, v0, nv, accumulate, stream);
    // test knob: the one-slice-per-weight kernel for any batch (tests/test_gpu_parity.py)
    static const bool force_s1 = getenv("CBP_BP_FORCE_S1") != nullptr;
    if (force_s1) return launch_bp_s<1>(g, t, sino, img, batch, v0, nv, accumulate, stream);
    if (use_sym8(g, batch, v0, nv))
        return launch_bp_sym8(g, t, sino, img, batch, 0, g.n_views / 8 + 1, accumulate, stream, 1);
    if (batch > 1 && use_sym8(g, 1, v0, nv))  // a batch: the 8 frames of each image
        return launch_bp_sym8(g, t, sino, img, batch, 0, g.n_views / 8 + 1, accumulate, stream, batch);
    if (use_sym4(g, batch, v0, nv))
        return launch_bp_s<4>(g, t, sino, img, batch, 0, g.n_views / 4, accumulate, stream, 4);
    if (batch >= 4) return launch_bp_s<4>(g, t, sino, img, batch, v0, nv, accumulate, stream);
    if (batch >= 2) return launch_bp_s<2>(g, t, sino, img, batch, v0, nv, accumulate, stream);
    if (g.kind == CBP_PARALLEL)  // tau' = tau: the weight's tau' terms leave the loop
        return launch_bp_s<1, false, 0, true>(g, t, sino, img, batch, v0, nv, accumulate, stream);
    return launch_bp_s<1>(g, t, sino, img, batch, v0, nv, accumulate, stream);
}

}  // namespace

extern "C" {

int cbp_validate(const cbp_geometry_t* g)
{
    if (!g) return CBP_EINVAL;
    if (g->n < 1 || g->n_views < 1 || g->n_det < 1) return CBP_EINVAL;
    if (!finite_pos(g->pixel) || !finite_pos(g->det_pitch) || !finite_pos(g->det_width))
        return CBP_EINVAL;
    if (g->model != CBP_MODEL_CNSF && g->model != CBP_MODEL_MAG) return CBP_EINVAL;
    if (g->kind == CBP_PARALLEL)
        return std::isfinite(g->sid) && std::isfinite(g->sdd) && narrow_ratio(*g) >= 1e-4 ? CBP_OK : CBP_EINVAL;
    if (g->kind != CBP_FAN_FLAT && g->kind != CBP_FAN_ARC) return CBP_EINVAL;
    if (!finite_pos(g->sid) || !finite_pos(g->sdd)) return CBP_EINVAL;
    // arc: every bin (and its blur) strictly inside +-90 degrees of the central ray
    if (g->kind == CBP_FAN_ARC &&
        !((0.5 * (g->n_det - 1) * g->det_pitch + 0.5 * g->det_width) / g->sdd < 0.5 * 3.14159265358979))
        return CBP_EINVAL;
    if (g->sdd < g->sid) return CBP_EINVAL;
    if (g->det_width >= 2.0 * g->sdd) return CBP_EINVAL;
    const double radius = 0.5 * (double)g->n * g->pixel * std::sqrt(2.0);
    if (!(radius < g->sid)) return CBP_EINVAL;
    if (!(narrow_ratio(*g) >= 1e-4)) return CBP_EINVAL;  // below the precise mode's range
    return CBP_OK;
}

int cbp_precise_mode(const cbp_geometry_t* g)
{
    if (cbp_validate(g) != CBP_OK) return CBP_EINVAL;
    return precise(*g) ? 1 : 0;
}

double cbp_narrow_ratio(const cbp_geometry_t* g)
{
    if (cbp_validate(g) != CBP_OK && !(g && g->n >= 1 && finite_pos(g->pixel) && finite_pos(g->det_width)))
        return -1.0;
    return narrow_ratio(*g);
}

int cbp_forward(const cbp_geometry_t* g, const float* image, float* sino, int32_t batch,
                int32_t view_begin, int32_t view_count, void* stream_)
{
    int rc = check_common(g, image, sino, batch, view_begin, view_count);
    if (rc != CBP_OK) return rc;
    cudaStream_t stream = (cudaStream_t)stream_;
    cbp::Tables t;
    if ((rc = get_tables(*g, stream, t)) != CBP_OK) return rc;
    const int ki = pointer_kind(image), ks = pointer_kind(sino);
    if (ki < 0 || ks < 0) return CBP_EINVAL;
    if (ki == 1 && ks == 1) return launch_fp(*g, t, image, sino, batch, view_begin, view_count, stream);

    // host buffers: stage through the device workspace, then synchronise
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_ws_mu);
    Workspace& w = g_ws[dev];
    const size_t ib = sizeof(float) * (size_t)batch * g->n * g->n;
    const size_t sb = sizeof(float) * (size_t)batch * view_count * g->n_det;
    void *di = (void*)image, *ds = (void*)sino;
    if (ki == 0 && (rc = ws_get(w, 0, ib, &di)) != CBP_OK) return rc;
    if (ks == 0 && (rc = ws_get(w, 1, sb, &ds)) != CBP_OK) return rc;
    if (ki == 0 && cudaMemcpyAsync(di, image, ib, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return CBP_ECUDA;
    if ((rc = launch_fp(*g, t, (const float*)di, (float*)ds, batch, view_begin, view_count,
                        stream)) != CBP_OK)
        return rc;
    if (ks == 0 && cudaMemcpyAsync(sino, ds, sb, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return CBP_ECUDA;
    return cudaStreamSynchronize(stream) == cudaSuccess ? CBP_OK : CBP_ECUDA;
}

int cbp_back(const cbp_geometry_t* g, const float* sino, float* image, int32_t batch,
             int32_t view_begin, int32_t view_count, int32_t accumulate, void* stream_)
{
    int rc = check_common(g, sino, image, batch, view_begin, view_count);
    if (rc != CBP_OK) return rc;
    if (accumulate < 0 || accumulate > CBP_ACC_MULTIMEM) return CBP_EINVAL;
    cudaStream_t stream = (cudaStream_t)stream_;
    cbp::Tables t;
    if ((rc = get_tables(*g, stream, t)) != CBP_OK) return rc;
    const int ks = pointer_kind(sino);
    if (accumulate == CBP_ACC_MULTIMEM) {  // image: a device multicast address (not checked)
        if (ks != 1) return CBP_EINVAL;
        return launch_bp(*g, t, sino, image, batch, view_begin, view_count, accumulate, stream);
    }
    const int ki = pointer_kind(image);
    if (ki < 0 || ks < 0) return CBP_EINVAL;
    if (ki == 1 && ks == 1)
        return launch_bp(*g, t, sino, image, batch, view_begin, view_count, accumulate, stream);

    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_ws_mu);
    Workspace& w = g_ws[dev];
    const size_t ib = sizeof(float) * (size_t)batch * g->n * g->n;
    const size_t sb = sizeof(float) * (size_t)batch * view_count * g->n_det;
    void *di = (void*)image, *ds = (void*)sino;
    if (ks == 0 && (rc = ws_get(w, 1, sb, &ds)) != CBP_OK) return rc;
    if (ki == 0 && (rc = ws_get(w, 0, ib, &di)) != CBP_OK) return rc;
    if (ks == 0 && cudaMemcpyAsync(ds, sino, sb, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return CBP_ECUDA;
    if (ki == 0 && accumulate &&
        cudaMemcpyAsync(di, image, ib, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return CBP_ECUDA;
    if ((rc = launch_bp(*g, t, (const float*)ds, (float*)di, batch, view_begin, view_count,
                        accumulate, stream)) != CBP_OK)
        return rc;
    if (ki == 0 && cudaMemcpyAsync(image, di, ib, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return CBP_ECUDA;
    return cudaStreamSynchronize(stream) == cudaSuccess ? CBP_OK : CBP_ECUDA;
}

int cbp_normal(const cbp_geometry_t* g, const float* image, float* out, int32_t batch, void* stream_)
{
    int rc = check_common(g, image, out, batch, 0, g ? g->n_views : 0);
    if (rc != CBP_OK) return rc;
    cudaStream_t stream = (cudaStream_t)stream_;
    cbp::Tables t;
    if ((rc = get_tables(*g, stream, t)) != CBP_OK) return rc;
    const int ki = pointer_kind(image), ko = pointer_kind(out);
    if (ki < 0 || ko < 0) return CBP_EINVAL;
    const size_t ib = sizeof(float) * (size_t)batch * g->n * g->n;
    float* sino = nullptr;  // A c stays on the device
    if ((rc = scratch_alloc((void**)&sino, sizeof(float) * (size_t)batch * g->n_views * g->n_det, stream)) !=
        CBP_OK)
        return rc;
    std::unique_lock<std::mutex> lock(g_ws_mu, std::defer_lock);
    void *di = (void*)image, *dout = (void*)out;
    if (ki == 0 || ko == 0) {  // host buffers: stage through the device workspace
        lock.lock();
        int dev = 0;
        cudaGetDevice(&dev);
        Workspace& w = g_ws[dev];
        if ((ki == 0 && (rc = ws_get(w, 0, ib, &di)) != CBP_OK) || (ko == 0 && (rc = ws_get(w, 1, ib, &dout)) != CBP_OK)) {
            cudaFreeAsync(sino, stream);
            return rc;
        }
        if (ki == 0 && cudaMemcpyAsync(di, image, ib, cudaMemcpyHostToDevice, stream) != cudaSuccess) {
            cudaFreeAsync(sino, stream);
            return CBP_ECUDA;
        }
    }
    rc = launch_fp(*g, t, (const float*)di, sino, batch, 0, g->n_views, stream);
    if (rc == CBP_OK) rc = launch_bp(*g, t, sino, (float*)dout, batch, 0, g->n_views, 0, stream);
    cudaFreeAsync(sino, stream);
    if (rc != CBP_OK) return rc;
    if (ko == 0 && cudaMemcpyAsync(out, dout, ib, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return CBP_ECUDA;
    if (ki == 0 || ko == 0) return cudaStreamSynchronize(stream) == cudaSuccess ? CBP_OK : CBP_ECUDA;
    return CBP_OK;
}

// ---- the streamed normal operator: a copy / compute / copy pipeline ------
// Per device: an H2D and a D2H stream (non-blocking) beside the caller's
// compute stream, double-buffered device images, one sinogram, and events
// that order slot reuse: image i+1 crosses PCIe while image i is projected,
// and image i-1's result returns meanwhile.
struct Pipe {
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t start, done, in_ready[2], in_free[2], out_ready[2], out_free[2];
    void* buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // in0, in1, out0, out1, sino
    size_t cap[5] = {0, 0, 0, 0, 0};
};
std::mutex g_pipe_mu;
std::map<int, Pipe> g_pipes;

static int pipe_get(int dev, Pipe** out)
{
    auto it = g_pipes.find(dev);
    if (it == g_pipes.end()) {
        Pipe p;
        bool ok = cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaEventCreateWithFlags(&p.start, cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreateWithFlags(&p.done, cudaEventDisableTiming) == cudaSuccess;
        for (int k = 0; k < 2 && ok; ++k)
            ok = cudaEventCreateWithFlags(&p.in_ready[k], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&p.in_free[k], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&p.out_ready[k], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&p.out_free[k], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) {
            cudaGetLastError();
            return CBP_ECUDA;
        }
        it = g_pipes.emplace(dev, p).first;
    }
    *out = &it->second;
    return CBP_OK;
}

static int pipe_buf(Pipe& p, int k, size_t bytes)
{
    if (p.cap[k] >= bytes) return CBP_OK;
    cudaFree(p.buf[k]);
    p.buf[k] = nullptr;
    p.cap[k] = 0;
    if (cudaMalloc(&p.buf[k], bytes) != cudaSuccess) {
        cudaGetLastError();
        return CBP_ECUDA;
    }
    p.cap[k] = bytes;
    return CBP_OK;
}

int cbp_normal_stream(const cbp_geometry_t* g, const float* images, float* out, int32_t count, int32_t batch,
                      void* stream_)
{
    int rc = check_common(g, images, out, batch, 0, g ? g->n_views : 0);
    if (rc != CBP_OK) return rc;
    if (count < 1) return CBP_EINVAL;
    cudaStream_t stream = (cudaStream_t)stream_;
    const int ki = pointer_kind(images), ko = pointer_kind(out);
    if (ki < 0 || ko < 0 || ki != ko) return CBP_EINVAL;
    cbp::Tables t;
    if ((rc = get_tables(*g, stream, t)) != CBP_OK) return rc;
    const size_t ni = (size_t)batch * g->n * g->n;
    const size_t ib = sizeof(float) * ni, sb = sizeof(float) * (size_t)batch * g->n_views * g->n_det;
    if (ki == 1) {
        // device buffers: the pairs back to back on `stream`, asynchronous -- the
        // sinogram is stream-ordered scratch of this call (a buffer shared between
        // calls would race with a later call on another stream)
        float* sino = nullptr;
        if ((rc = scratch_alloc((void**)&sino, sb, stream)) != CBP_OK) return rc;
        for (int32_t i = 0; i < count && rc == CBP_OK; ++i) {
            rc = launch_fp(*g, t, images + i * ni, sino, batch, 0, g->n_views, stream);
            if (rc == CBP_OK) rc = launch_bp(*g, t, sino, out + i * ni, batch, 0, g->n_views, 0, stream);
        }
        cudaFreeAsync(sino, stream);
        return rc;
    }
    // host buffers: the call is synchronous, so the per-device pipe buffers
    // are free again when it returns (the mutex serialises callers)
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_pipe_mu);
    Pipe* P = nullptr;
    if ((rc = pipe_get(dev, &P)) != CBP_OK) return rc;
    if ((rc = pipe_buf(*P, 4, sb)) != CBP_OK) return rc;
    float* sino = (float*)P->buf[4];
    for (int k = 0; k < 4 && rc == CBP_OK; ++k) rc = pipe_buf(*P, k, ib);
    if (rc != CBP_OK) return rc;
    // everything after the work already queued on `stream`
    if (cudaEventRecord(P->start, stream) != cudaSuccess || cudaStreamWaitEvent(P->h2d, P->start, 0) != cudaSuccess ||
        cudaStreamWaitEvent(P->d2h, P->start, 0) != cudaSuccess)
        return CBP_ECUDA;
    bool ok = true;
    for (int32_t i = 0; i < count && ok; ++i) {
        const int k = i & 1;
        float* din = (float*)P->buf[k];
        float* dout = (float*)P->buf[2 + k];
        // H2D of image i once image i-2's FP has read the slot
        if (i >= 2) ok = ok && cudaStreamWaitEvent(P->h2d, P->in_free[k], 0) == cudaSuccess;
        ok = ok && cudaMemcpyAsync(din, images + i * ni, ib, cudaMemcpyHostToDevice, P->h2d) == cudaSuccess;
        ok = ok && cudaEventRecord(P->in_ready[k], P->h2d) == cudaSuccess;
        // FP + BP on the caller's stream once the image is in and result slot i-2 has left
        ok = ok && cudaStreamWaitEvent(stream, P->in_ready[k], 0) == cudaSuccess;
        if (i >= 2) ok = ok && cudaStreamWaitEvent(stream, P->out_free[k], 0) == cudaSuccess;
        if (!ok) break;
        if ((rc = launch_fp(*g, t, din, sino, batch, 0, g->n_views, stream)) != CBP_OK) break;
        ok = ok && cudaEventRecord(P->in_free[k], stream) == cudaSuccess;
        if ((rc = launch_bp(*g, t, sino, dout, batch, 0, g->n_views, 0, stream)) != CBP_OK) break;
        ok = ok && cudaEventRecord(P->out_ready[k], stream) == cudaSuccess;
        // D2H of result i
        ok = ok && cudaStreamWaitEvent(P->d2h, P->out_ready[k], 0) == cudaSuccess;
        ok = ok && cudaMemcpyAsync(out + i * ni, dout, ib, cudaMemcpyDeviceToHost, P->d2h) == cudaSuccess;
        ok = ok && cudaEventRecord(P->out_free[k], P->d2h) == cudaSuccess;
    }
    if (rc != CBP_OK || !ok) {
        // nothing may still write the caller's host buffers after an error return
        cudaStreamSynchronize(P->h2d);
        cudaStreamSynchronize(stream);
        cudaStreamSynchronize(P->d2h);
        cudaGetLastError();
        return rc != CBP_OK ? rc : CBP_ECUDA;
    }
    ok = cudaEventRecord(P->done, P->d2h) == cudaSuccess && cudaStreamWaitEvent(stream, P->done, 0) == cudaSuccess &&
         cudaEventSynchronize(P->done) == cudaSuccess;
    return ok ? CBP_OK : CBP_ECUDA;
}

int cbp_symmetry_fold(const cbp_geometry_t* g, int32_t batch, int32_t view_begin,
                      int32_t view_count)
{
    if (cbp_validate(g) != CBP_OK) return CBP_EINVAL;
    if (precise(*g)) return 1;
    if (use_mag_sym4(*g, batch, view_begin, view_count)) return mag_bp_fold(*g);  // the BP's (the FP uses 4)
    if (use_sym8(*g, 1, view_begin, view_count)) return 8;  // the BP of any batch (per image)
    return use_sym4(*g, batch, view_begin, view_count) ? 4 : 1;
}

static int check_orbit(const cbp_geometry_t* g, const void* a, const void* b, int32_t base_begin,
                       int32_t base_count, bool mc_image = false)
{
    if (cbp_validate(g) != CBP_OK || g->n_views % 4 != 0) return CBP_EINVAL;
    if (!a || !b || base_count < 1 || base_begin < 0 || (int64_t)base_begin + base_count > g->n_views / 4)
        return CBP_EINVAL;
    if (((uintptr_t)a & 3) || ((uintptr_t)b & 3)) return CBP_EINVAL;
    if ((!mc_image && pointer_kind(a) != 1) || pointer_kind(b) != 1) return CBP_EINVAL;
    return CBP_OK;
}

int cbp_forward_orbit(const cbp_geometry_t* g, const float* image, float* sino, int32_t base_begin,
                      int32_t base_count, void* stream_)
{
    int rc = check_orbit(g, image, sino, base_begin, base_count);
    if (rc != CBP_OK) return rc;
    cudaStream_t stream = (cudaStream_t)stream_;
    cbp::Tables t;
    if ((rc = get_tables(*g, stream, t)) != CBP_OK) return rc;
    if (g->model == CBP_MODEL_MAG || precise(*g)) {  // no shared weights: the 4 view blocks one by one
        for (int q = 0; q < 4 && rc == CBP_OK; ++q)
            rc = launch_fp(*g, t, image, sino + (size_t)q * base_count * g->n_det, 1,
                           base_begin + q * (g->n_views / 4), base_count, stream);
        return rc;
    }
    return launch_fp_sym4(*g, t, image, sino, base_begin, base_count, stream);
}

int cbp_back_orbit(const cbp_geometry_t* g, const float* sino, float* image, int32_t base_begin,
                   int32_t base_count, int32_t accumulate, void* stream_)
{
    if (accumulate < 0 || accumulate > CBP_ACC_MULTIMEM) return CBP_EINVAL;
    int rc = check_orbit(g, image, sino, base_begin, base_count, accumulate == CBP_ACC_MULTIMEM);
    if (rc != CBP_OK) return rc;
    cudaStream_t stream = (cudaStream_t)stream_;
    cbp::Tables t;
    if ((rc = get_tables(*g, stream, t)) != CBP_OK) return rc;
    if (g->model == CBP_MODEL_MAG || precise(*g)) {
        for (int q = 0; q < 4 && rc == CBP_OK; ++q)
            rc = launch_bp(*g, t, sino + (size_t)q * base_count * g->n_det, image, 1,
                           base_begin + q * (g->n_views / 4), base_count, q > 0 ? acc_next(accumulate) : accumulate,
                           stream);
        return rc;
    }
    return launch_bp_s<4>(*g, t, sino, image, 1, base_begin, base_count, accumulate, stream, 4);
}

// ---- dihedral shards (views sharded over GPUs keeping the 8-fold symmetry)
// The magnified-footprint model and the precise mode run the shard's views as
// contiguous blocks of the natural layout: the 4 rotations of the base block
// [b0, b0 + nb) and of its mirror images N/4 - b for b in [max(b0, 1), min(b0 + nb, N/8)).
static int block_dihedral(const cbp_geometry_t& g, const cbp::Tables& t, const float* image, float* sino,
                          int32_t b0, int32_t nb, int32_t accumulate, cudaStream_t stream, bool fp)
{
    const int N = g.n_views, q = N / 4, e = N / 8;
    const int lo = std::max(b0, 1), hi = std::min(b0 + nb, e);
    const int starts[2] = {b0, q - hi + 1}, counts[2] = {nb, hi - lo};
    int rc = CBP_OK, done = 0;
    for (int blk = 0; blk < 2; ++blk) {
        if (counts[blk] < 1) continue;
        for (int r = 0; r < 4 && rc == CBP_OK; ++r, ++done) {
            const int v = starts[blk] + r * q;
            rc = fp ? launch_fp(g, t, image, sino + (size_t)v * g.n_det, 1, v, counts[blk], stream)
                    : launch_bp(g, t, sino + (size_t)v * g.n_det, const_cast<float*>(image), 1, v, counts[blk],
                                done > 0 ? acc_next(accumulate) : accumulate, stream);
        }
    }
    return rc;
}

static int check_dihedral(const cbp_geometry_t* g, const void* a, const void* b, int32_t base_begin,
                          int32_t base_count, bool mc_image = false)
{
    if (cbp_validate(g) != CBP_OK || g->n_views % 8 != 0) return CBP_EINVAL;
    if (!a || !b || base_count < 1 || base_begin < 0 || (int64_t)base_begin + base_count > g->n_views / 8 + 1)
        return CBP_EINVAL;
    if (((uintptr_t)a & 3) || ((uintptr_t)b & 3)) return CBP_EINVAL;
    if ((!mc_image && pointer_kind(a) != 1) || pointer_kind(b) != 1) return CBP_EINVAL;
    return CBP_OK;
}

int cbp_forward_dihedral(const cbp_geometry_t* g, const float* image, float* sino, int32_t base_begin,
                         int32_t base_count, void* stream_)
{
    int rc = check_dihedral(g, image, sino, base_begin, base_count);
    if (rc != CBP_OK) return rc;
    cudaStream_t stream = (cudaStream_t)stream_;
    cbp::Tables t;
    if ((rc = get_tables(*g, stream, t)) != CBP_OK) return rc;
    const int N = g->n_views, q = N / 4, e = N / 8;
    if (g->model == CBP_MODEL_MAG || precise(*g))
        return block_dihedral(*g, t, image, sino, base_begin, base_count, 0, stream, true);
    // the 4 rotations of the base block, then those of its mirror images
    // N/4 - v (v = 0 and v = N/8 are their own mirror orbits)
    // one pad and one launch for both blocks (the grid of a small shard is far short of a wave)
    // (one 8-frame launch over the base block instead, launch_fp_sym8(..., base_begin,
    // base_count): measured slower at every shard size)
    const int lo = std::max(base_begin, 1), hi = std::min(base_begin + base_count, e);  // [lo, hi)
    return launch_fp_sym4(*g, t, image, sino, base_begin, base_count, stream, q, q - hi + 1, hi > lo ? hi - lo : 0);
}

int cbp_back_dihedral(const cbp_geometry_t* g, const float* sino, float* image, int32_t base_begin,
                      int32_t base_count, int32_t accumulate, void* stream_)
{
    if (accumulate < 0 || accumulate > CBP_ACC_MULTIMEM) return CBP_EINVAL;
    int rc = check_dihedral(g, sino, image, base_begin, base_count, accumulate == CBP_ACC_MULTIMEM);
    if (rc != CBP_OK) return rc;
    cudaStream_t stream = (cudaStream_t)stream_;
    cbp::Tables t;
    if ((rc = get_tables(*g, stream, t)) != CBP_OK) return rc;
    if (g->model == CBP_MODEL_MAG || precise(*g))
        return block_dihedral(*g, t, image, const_cast<float*>(sino), base_begin, base_count, accumulate, stream,
                              false);
    return launch_bp_sym8(*g, t, sino, image, 1, base_begin, base_count, accumulate, stream, 1);
}

// ---- row f1: SART / CGLS building blocks ---------------------------------
static int vec_grid(int64_t count)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t b = (count + cbp::VEC_BLOCK - 1) / cbp::VEC_BLOCK;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)sms * 8));
}

static int launched()
{
    ++g_launches;
    return cudaGetLastError() == cudaSuccess ? CBP_OK : CBP_ECUDA;
}

int cbp_sart_residual(const float* y, const float* ay, const float* rowsum, float* r, int64_t count,
                      void* stream)
{
    if (!y || !ay || !rowsum || !r || count < 0) return CBP_EINVAL;
    if (count == 0) return CBP_OK;
    cbp::cbp_sart_residual_kernel<<<vec_grid(count), cbp::VEC_BLOCK, 0, (cudaStream_t)stream>>>(
        y, ay, rowsum, r, count);
    return launched();
}

int cbp_sart_update(float* c, const float* bp, const float* colsum, float beta, int32_t nonneg,
                    int64_t count, void* stream)
{
    if (!c || !bp || !colsum || count < 0 || !std::isfinite(beta)) return CBP_EINVAL;
    if (count == 0) return CBP_OK;
    cbp::cbp_sart_update_kernel<<<vec_grid(count), cbp::VEC_BLOCK, 0, (cudaStream_t)stream>>>(
        c, bp, colsum, beta, nonneg ? 1 : 0, count);
    return launched();
}

int cbp_fill(float* x, float value, int64_t count, void* stream)
{
    if (!x || count < 0) return CBP_EINVAL;
    if (count == 0) return CBP_OK;
    cbp::cbp_fill_kernel<<<vec_grid(count), cbp::VEC_BLOCK, 0, (cudaStream_t)stream>>>(x, value, count);
    return launched();
}

int cbp_dot(const float* a, const float* b, int64_t count, double* out, void* stream_)
{
    if (!a || !b || !out || count < 0) return CBP_EINVAL;
    cudaStream_t stream = (cudaStream_t)stream_;
    double* part = nullptr;
    int rc = scratch_alloc((void**)&part, sizeof(double) * cbp::DOT_BLOCKS, stream);
    if (rc != CBP_OK) return rc;
    cbp::cbp_dot_partial_kernel<<<cbp::DOT_BLOCKS, cbp::VEC_BLOCK, 0, stream>>>(a, b, count, part);
    ++g_launches;
    cbp::cbp_dot_final_kernel<<<1, cbp::VEC_BLOCK, 0, stream>>>(part, cbp::DOT_BLOCKS, out);
    rc = launched();
    cudaFreeAsync(part, stream);
    return rc;
}

// ---- row f4: TV and the ASD-POCS steps ---------------------------------------
static int sum_reduce(const float* a, const float* b, int n, int64_t count, double eps, int mode,
                      double* out, cudaStream_t stream)
{
    double* part = nullptr;
    int rc = scratch_alloc((void**)&part, sizeof(double) * cbp::DOT_BLOCKS, stream);
    if (rc != CBP_OK) return rc;
    cbp::cbp_sum_partial_kernel<<<cbp::DOT_BLOCKS, cbp::VEC_BLOCK, 0, stream>>>(a, b, n, count, eps, mode,
                                                                               part);
    ++g_launches;
    cbp::cbp_dot_final_kernel<<<1, cbp::VEC_BLOCK, 0, stream>>>(part, cbp::DOT_BLOCKS, out);
    rc = launched();
    cudaFreeAsync(part, stream);
    return rc;
}

int cbp_tv_value(const float* x, int32_t n, int32_t batch, double eps, double* out, void* stream)
{
    if (!x || !out || n < 1 || batch < 1 || !(eps >= 0.0)) return CBP_EINVAL;
    return sum_reduce(x, nullptr, n, (int64_t)batch * n * n, eps, 0, out, (cudaStream_t)stream);
}

int cbp_tv_gradient(const float* x, float* grad, int32_t n, int32_t batch, double eps, void* stream)
{
    if (!x || !grad || n < 1 || batch < 1 || !(eps >= 0.0)) return CBP_EINVAL;
    const int64_t count = (int64_t)batch * n * n;
    cbp::cbp_tv_gradient_kernel<<<vec_grid(count), cbp::VEC_BLOCK, 0, (cudaStream_t)stream>>>(x, grad, n,
                                                                                              count, eps);
    return launched();
}

int cbp_diff_norm2(const float* a, const float* b, int64_t count, double* out, void* stream)
{
    if (!a || !b || !out || count < 0) return CBP_EINVAL;
    return sum_reduce(a, b, 1, count, 0.0, 1, out, (cudaStream_t)stream);
}

int cbp_tv_step(float* x, const float* g, int64_t count, const double* gg, const double* alpha,
                const double* dp2, void* stream)
{
    if (!x || !g || !gg || !alpha || !dp2 || count < 0) return CBP_EINVAL;
    cbp::cbp_tv_step_kernel<<<vec_grid(count), cbp::VEC_BLOCK, 0, (cudaStream_t)stream>>>(x, g, count, gg,
                                                                                          alpha, dp2);
    return launched();
}

int cbp_asd_adapt(double* alpha, const double* dp2, const double* dg2, double r_max, double alpha_red,
                  void* stream)
{
    if (!alpha || !dp2 || !dg2) return CBP_EINVAL;
    cbp::cbp_asd_adapt_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(alpha, dp2, dg2, r_max, alpha_red);
    return launched();
}

int cbp_cgls_step(float* x, const float* p, float* r, const float* q, const double* num,
                  const double* den, int64_t nx, int64_t nr, void* stream)
{
    if (!x || !p || !r || !q || !num || !den || nx < 0 || nr < 0) return CBP_EINVAL;
    cbp::cbp_cgls_step_kernel<<<vec_grid(std::max(nx, nr)), cbp::VEC_BLOCK, 0, (cudaStream_t)stream>>>(
        x, p, r, q, num, den, nx, nr);
    return launched();
}

int cbp_cgls_direction(float* p, const float* s, const double* num, const double* den, int64_t count,
                       void* stream)
{
    if (!p || !s || !num || !den || count < 0) return CBP_EINVAL;
    cbp::cbp_cgls_dir_kernel<<<vec_grid(count), cbp::VEC_BLOCK, 0, (cudaStream_t)stream>>>(
        p, s, num, den, count);
    return launched();
}

static uint64_t splitmix64(uint64_t& x)
{
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int cbp_adjoint_check(const cbp_geometry_t* g, uint64_t seed, double* rel_defect)
{
    if (cbp_validate(g) != CBP_OK || !rel_defect) return CBP_EINVAL;
    const size_t ni = (size_t)g->n * g->n, ns = (size_t)g->n_views * g->n_det;
    std::vector<float> c(ni), y(ns), Ac(ns), Aty(ni);
    uint64_t st = seed;
    for (auto& x : c) x = (float)((splitmix64(st) >> 40) * 0x1p-24);
    for (auto& x : y) x = (float)((splitmix64(st) >> 40) * 0x1p-24);
    float *dc = nullptr, *dy = nullptr, *dAc = nullptr, *dAty = nullptr;
    int rc = CBP_ECUDA;
    if (cudaMalloc(&dc, ni * 4) == cudaSuccess && cudaMalloc(&dy, ns * 4) == cudaSuccess &&
        cudaMalloc(&dAc, ns * 4) == cudaSuccess && cudaMalloc(&dAty, ni * 4) == cudaSuccess &&
        cudaMemcpy(dc, c.data(), ni * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
        cudaMemcpy(dy, y.data(), ns * 4, cudaMemcpyHostToDevice) == cudaSuccess) {
        rc = cbp_forward(g, dc, dAc, 1, 0, g->n_views, nullptr);
        if (rc == CBP_OK) rc = cbp_back(g, dy, dAty, 1, 0, g->n_views, 0, nullptr);
        if (rc == CBP_OK) {
            if (cudaMemcpy(Ac.data(), dAc, ns * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
                cudaMemcpy(Aty.data(), dAty, ni * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
                rc = CBP_ECUDA;
        }
    }
    cudaFree(dc);
    cudaFree(dy);
    cudaFree(dAc);
    cudaFree(dAty);
    cudaGetLastError();
    if (rc != CBP_OK) return rc;
    double lhs = 0.0, rhs = 0.0;
    for (size_t i = 0; i < ns; ++i) lhs += (double)Ac[i] * (double)y[i];
    for (size_t i = 0; i < ni; ++i) rhs += (double)c[i] * (double)Aty[i];
    *rel_defect = lhs != 0.0 ? std::fabs(lhs - rhs) / std::fabs(lhs) : std::fabs(rhs);
    return CBP_OK;
}

const char* cbp_strerror(int code)
{
    switch (code) {
        case CBP_OK: return "ok";
        case CBP_EINVAL: return "invalid geometry or argument";
        case CBP_ECUDA: return "CUDA error";
        case CBP_ENOMEM: return "out of host memory";
        default: return "unknown error";
    }
}

// ---- row f2: the reference projector ---------------------------------------
int cbp_ref_forward(const cbp_geometry_t* g, const float* image, double* sino, int32_t batch,
                    int32_t view_begin, int32_t view_count, void* stream_)
{
    int rc = check_common(g, image, sino, batch, view_begin, view_count);
    if (rc != CBP_OK) return rc;
    if (((uintptr_t)sino & 7) || pointer_kind(image) != 1 || pointer_kind(sino) != 1) return CBP_EINVAL;
    cudaStream_t stream = (cudaStream_t)stream_;
    cbp::Tables t;
    if ((rc = get_tables(*g, stream, t)) != CBP_OK) return rc;
    cbp::RefParams P;
    P.g = to_dev(*g);
    P.t = t;
    P.img = image;
    P.sino = sino;
    P.view_begin = view_begin;
    P.view_count = view_count;
    P.batch = batch;
    dim3 grid((g->n_det + cbp::REF_BLOCK - 1) / cbp::REF_BLOCK, view_count, batch);
    cbp::cbp_ref_fp_kernel<<<grid, cbp::REF_BLOCK, 0, stream>>>(P);
    return launched();
}

int cbp_ref_back(const cbp_geometry_t* g, const double* sino, double* image, int32_t batch,
                 int32_t view_begin, int32_t view_count, void* stream_)
{
    int rc = check_common(g, sino, image, batch, view_begin, view_count);
    if (rc != CBP_OK) return rc;
    if (((uintptr_t)sino & 7) || ((uintptr_t)image & 7) || pointer_kind(image) != 1 || pointer_kind(sino) != 1)
        return CBP_EINVAL;
    cudaStream_t stream = (cudaStream_t)stream_;
    cbp::Tables t;
    if ((rc = get_tables(*g, stream, t)) != CBP_OK) return rc;
    cbp::RefBackParams P;
    P.g = to_dev(*g);
    P.t = t;
    P.sino = sino;
    P.img = image;
    P.view_begin = view_begin;
    P.view_count = view_count;
    P.batch = batch;
    dim3 grid((unsigned)(((int64_t)g->n * g->n + cbp::REF_BLOCK - 1) / cbp::REF_BLOCK), batch);
    cbp::cbp_ref_bp_kernel<<<grid, cbp::REF_BLOCK, 0, stream>>>(P);
    return launched();
}

int cbp_version(void) { return 140; }

uint64_t cbp_launch_count(void) { return g_launches.load(); }

}  // extern "C"
