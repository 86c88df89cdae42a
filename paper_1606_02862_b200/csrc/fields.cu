// Yee FDTD field update and field-side validation on sm_100a.
//
// Reference: pic/kernels.py:253-288 (`_faraday`, `_ampere`), pic/fields.py
// :145-169 (div B, div J, field energy), pic/sim.py:168-175 (continuity
// residual).  The reference walks cells per super cell; here one thread
// owns one cell of the x-fastest lattice, so every neighbour read along x is
// coalesced and +-y/+-z neighbours hit L1/L2.  Arithmetic follows the
// reference bit for bit: differences in the storage type, everything after
// the divide by a Python float in double, rounding on store.
#include <algorithm>
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace kwb {

template <typename F>
struct F3 {
    F *x, *y, *z;
};

// Reciprocals of the cell sizes (RN(1/delta), host IEEE division) for the
// Yee quotients through div_rcp: bit for bit (double)a / delta.
struct Rcp3 {
    double x, y, z;
};
static Rcp3 rcp3(const kwb_grid *g) { return Rcp3{1.0 / g->dx, 1.0 / g->dy, 1.0 / g->dz}; }

// One thread per cell of an x row, blocks over (x tiles, y, z): no 64-bit
// index division; x neighbours coalesced, y/z neighbours from L1/L2.
// B -= half_dt * curl E (forward differences), pic/kernels.py:264-269.
template <typename F>
__global__ void __launch_bounds__(256) faraday_kernel(Geo g, Rcp3 r, F3<F> E, F3<F> B, double half_dt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.nx) return;
    const int j = blockIdx.y, k = blockIdx.z;
    const int64_t c = fidx(i, j, k, g.nx, g.ny);
    const int64_t ip = c + (i + 1 == g.nx ? 1 - g.nx : 1);
    const int64_t jp = c + (j + 1 == g.ny ? (int64_t)(1 - g.ny) * g.nx : g.nx);
    const int64_t kp = c + (k + 1 == g.nz ? (int64_t)(1 - g.nz) * g.ny * g.nx : (int64_t)g.ny * g.nx);
    const F exc = E.x[c], eyc = E.y[c], ezc = E.z[c];
    F a = E.z[jp] - ezc, b = E.y[kp] - eyc;
    B.x[c] = (F)((double)B.x[c] - half_dt * (div_rcp((double)a, g.dy, r.y) - div_rcp((double)b, g.dz, r.z)));
    a = E.x[kp] - exc; b = E.z[ip] - ezc;
    B.y[c] = (F)((double)B.y[c] - half_dt * (div_rcp((double)a, g.dz, r.z) - div_rcp((double)b, g.dx, r.x)));
    a = E.y[ip] - eyc; b = E.x[jp] - exc;
    B.z[c] = (F)((double)B.z[c] - half_dt * (div_rcp((double)a, g.dx, r.x) - div_rcp((double)b, g.dy, r.y)));
}

// E += dt * (curl B - J) (backward differences), pic/kernels.py:283-288.
template <typename F>
__global__ void __launch_bounds__(256) ampere_kernel(Geo g, Rcp3 r, F3<F> E, F3<F> B, F3<F> J, double dt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.nx) return;
    const int j = blockIdx.y, k = blockIdx.z;
    const int64_t c = fidx(i, j, k, g.nx, g.ny);
    const int64_t im = c - (i == 0 ? 1 - g.nx : 1);
    const int64_t jm = c - (j == 0 ? (int64_t)(1 - g.ny) * g.nx : g.nx);
    const int64_t km = c - (k == 0 ? (int64_t)(1 - g.nz) * g.ny * g.nx : (int64_t)g.ny * g.nx);
    const F bxc = B.x[c], byc = B.y[c], bzc = B.z[c];
    F a = bzc - B.z[jm], b = byc - B.y[km];
    E.x[c] = (F)((double)E.x[c] + dt * ((div_rcp((double)a, g.dy, r.y) - div_rcp((double)b, g.dz, r.z)) - (double)J.x[c]));
    a = bxc - B.x[km]; b = bzc - B.z[im];
    E.y[c] = (F)((double)E.y[c] + dt * ((div_rcp((double)a, g.dz, r.z) - div_rcp((double)b, g.dx, r.x)) - (double)J.y[c]));
    a = byc - B.y[im]; b = bxc - B.x[jm];
    E.z[c] = (F)((double)E.z[c] + dt * ((div_rcp((double)a, g.dx, r.x) - div_rcp((double)b, g.dy, r.y)) - (double)J.z[c]));
}

static dim3 row_grid(const kwb_grid *g) {
    return dim3((unsigned)((g->nx + 255) / 256), (unsigned)g->ny, (unsigned)g->nz);
}
static int row_threads(const kwb_grid *g) { return g->nx < 256 ? (g->nx + 31) / 32 * 32 : 256; }

// Backward-difference divergence at the charge sites, computed the way numpy
// evaluates pic/fields.py:154-160 on F arrays (NEP 50: the Python-float
// delta is cast to F, all arithmetic in F).
template <typename F>
__device__ __forceinline__ F div_back(const F3<F> &A, int64_t c, int64_t im, int64_t jm, int64_t km,
                                      F dx, F dy, F dz) {
    const F a = (A.x[c] - A.x[im]) / dx;
    const F b = (A.y[c] - A.y[jm]) / dy;
    const F d = (A.z[c] - A.z[km]) / dz;
    return (a + b) + d;
}

template <typename F>
__global__ void __launch_bounds__(256)
residual_kernel(Geo g, const double *__restrict__ rho_new, const double *__restrict__ rho_prev,
                F3<F> J, F3<F> E, double *__restrict__ G_prev, double *__restrict__ out) {
    const int64_t ncell = (int64_t)g.nx * g.ny * g.nz;
    const F dx = (F)g.dx, dy = (F)g.dy, dz = (F)g.dz;
    double rmax = 0.0, gmax = 0.0;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(c % g.nx);
        const int j = (int)((c / g.nx) % g.ny);
        const int k = (int)(c / ((int64_t)g.nx * g.ny));
        const int64_t im = fidx(i == 0 ? g.nx - 1 : i - 1, j, k, g.nx, g.ny);
        const int64_t jm = fidx(i, j == 0 ? g.ny - 1 : j - 1, k, g.nx, g.ny);
        const int64_t km = fidx(i, j, k == 0 ? g.nz - 1 : k - 1, g.nx, g.ny);
        const double rn = rho_new[c];
        if (rho_prev) {
            const double dj = (double)div_back<F>(J, c, im, jm, km, dx, dy, dz);
            const double r = fabs((rn - rho_prev[c]) / g.dt + dj);
            rmax = fmax(rmax, r);
        }
        if (G_prev) {
            const double G = (double)div_back<F>(E, c, im, jm, km, dx, dy, dz) - rn;
            gmax = fmax(gmax, fabs(G - G_prev[c]));
            G_prev[c] = G;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(out + 0, rmax);
        atomic_max_nonneg(out + 1, gmax);
    }
}

// out[0] += sum(E^2 + B^2) in float64; out[1] = max |div B| with the forward
// face divergence of pic/fields.py:145-151 (numpy F arithmetic).
template <typename F>
__global__ void __launch_bounds__(256) field_stats_kernel(Geo g, F3<F> E, F3<F> B, double *out) {
    __shared__ double red[8];
    const int64_t ncell = (int64_t)g.nx * g.ny * g.nz;
    const F dx = (F)g.dx, dy = (F)g.dy, dz = (F)g.dz;
    double s = 0.0, dmax = 0.0;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(c % g.nx);
        const int j = (int)((c / g.nx) % g.ny);
        const int k = (int)(c / ((int64_t)g.nx * g.ny));
        const int64_t ip = fidx(i + 1 == g.nx ? 0 : i + 1, j, k, g.nx, g.ny);
        const int64_t jp = fidx(i, j + 1 == g.ny ? 0 : j + 1, k, g.nx, g.ny);
        const int64_t kp = fidx(i, j, k + 1 == g.nz ? 0 : k + 1, g.nx, g.ny);
        const double ex = E.x[c], ey = E.y[c], ez = E.z[c], bx = B.x[c], by = B.y[c], bz = B.z[c];
        s += ((ex * ex + ey * ey) + ez * ez) + ((bx * bx + by * by) + bz * bz);
        const F a = (B.x[ip] - B.x[c]) / dx, b = (B.y[jp] - B.y[c]) / dy,
                d = (B.z[kp] - B.z[c]) / dz;
        dmax = fmax(dmax, fabs((double)((a + b) + d)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[wid] = s;
        atomic_max_nonneg(out + 1, dmax);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        atomicAdd(out + 0, t);
    }
}

static int grid_blocks(int64_t ncell) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    int64_t need = (ncell + 255) / 256;
    int64_t cap = (int64_t)sms * 8;
    return (int)(need < cap ? (need > 0 ? need : 1) : cap);
}

template <typename F>
static F3<F> f3(void *const a[3]) {
    F3<F> r;
    r.x = (F *)a[0]; r.y = (F *)a[1]; r.z = (F *)a[2];
    return r;
}

}  // namespace kwb

// ============================ C ABI =======================================
using namespace kwb;

static thread_local char g_err[512] = "";

void kwb_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int kwb_check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        kwb_set_error("%s: %s", what, cudaGetErrorString(e));
        return KWB_ECUDA;
    }
    return KWB_OK;
}

extern "C" int kwb_version(void) { return KWB_VERSION; }
extern "C" const char *kwb_last_error(void) { return g_err; }

static int check_fields(const kwb_grid *g, const char *what) {
    if (!g || g->nx <= 0 || g->ny <= 0 || g->nz <= 0 ||
        (g->dtype != KWB_F32 && g->dtype != KWB_F64)) {
        kwb_set_error("%s: invalid grid", what);
        return KWB_EINVAL;
    }
    return KWB_OK;
}

static bool all3(void *const a[3]) { return a && a[0] && a[1] && a[2]; }

// E and B at arbitrary points (the reference's gather_fields,
// pic/fields.py:95-118, with the advance kernel's recipe pic/kernels.py:26-77:
// trilinear weights of the Yee-staggered lattices in double, periodic wrap,
// rounded to the storage type).  One thread per point.
template <typename F>
__device__ __forceinline__ double sample_global(const F *__restrict__ a, const Geo &g, double px,
                                                double py, double pz, double sx, double sy,
                                                double sz) {
    const double tx = px - sx, ty = py - sy, tz = pz - sz;
    const int64_t ix = (int64_t)floor(tx), iy = (int64_t)floor(ty), iz = (int64_t)floor(tz);
    const double fx = tx - (double)ix, fy = ty - (double)iy, fz = tz - (double)iz;
    auto md = [](int64_t v, int n) { int64_t r = v % n; return r < 0 ? r + n : r; };
    const int64_t i0 = md(ix, g.nx), i1 = md(ix + 1, g.nx), j0 = md(iy, g.ny),
                  j1 = md(iy + 1, g.ny), k0 = md(iz, g.nz), k1 = md(iz + 1, g.nz);
    auto A = [&](int64_t i, int64_t j, int64_t k) { return (double)a[(k * g.ny + j) * g.nx + i]; };
    const double c00 = A(i0, j0, k0) * (1.0 - fx) + A(i1, j0, k0) * fx;
    const double c10 = A(i0, j1, k0) * (1.0 - fx) + A(i1, j1, k0) * fx;
    const double c01 = A(i0, j0, k1) * (1.0 - fx) + A(i1, j0, k1) * fx;
    const double c11 = A(i0, j1, k1) * (1.0 - fx) + A(i1, j1, k1) * fx;
    return (c00 * (1.0 - fy) + c10 * fy) * (1.0 - fz) + (c01 * (1.0 - fy) + c11 * fy) * fz;
}

template <typename F>
__global__ void gather_points_kernel(Geo g, F3<F> E, F3<F> B, int64_t n,
                                     const int32_t *__restrict__ cells,
                                     const double *__restrict__ offsets, F *__restrict__ out) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const double px = (double)cells[3 * q] + offsets[3 * q];
    const double py = (double)cells[3 * q + 1] + offsets[3 * q + 1];
    const double pz = (double)cells[3 * q + 2] + offsets[3 * q + 2];
    // staggers, pic/fields.py:24-31
    out[6 * q + 0] = (F)sample_global(E.x, g, px, py, pz, 1.0, 0.5, 0.5);
    out[6 * q + 1] = (F)sample_global(E.y, g, px, py, pz, 0.5, 1.0, 0.5);
    out[6 * q + 2] = (F)sample_global(E.z, g, px, py, pz, 0.5, 0.5, 1.0);
    out[6 * q + 3] = (F)sample_global(B.x, g, px, py, pz, 0.5, 1.0, 1.0);
    out[6 * q + 4] = (F)sample_global(B.y, g, px, py, pz, 1.0, 0.5, 1.0);
    out[6 * q + 5] = (F)sample_global(B.z, g, px, py, pz, 1.0, 1.0, 0.5);
}

extern "C" int kwb_fields_gather(const kwb_grid *g, void *const E[3], void *const B[3], int64_t n,
                                 const int32_t *cells, const double *offsets, void *out,
                                 kwb_stream_t stream) {
    int rc = check_fields(g, "gather");
    if (rc) return rc;
    if (!all3(E) || !all3(B) || (n > 0 && (!cells || !offsets || !out)) || n < 0) {
        kwb_set_error("gather: NULL or invalid argument");
        return KWB_EINVAL;
    }
    if (n == 0) return KWB_OK;
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = (int)((n + 255) / 256);
    if (g->dtype == KWB_F32)
        gather_points_kernel<float><<<blocks, 256, 0, s>>>(geo, f3<float>(E), f3<float>(B), n, cells,
                                                          offsets, (float *)out);
    else
        gather_points_kernel<double><<<blocks, 256, 0, s>>>(geo, f3<double>(E), f3<double>(B), n,
                                                            cells, offsets, (double *)out);
    return kwb_check_launch("gather_points_kernel");
}

// Start-of-step clear: J = 0 (pic/sim.py:138-140) and the per-species status
// words, one kernel instead of two eager fills.  16-byte stores where the
// lattices allow (each is a separate pointer; their sizes are multiples of
// 16 bytes whenever nx * ny * nz * sizeof(F) is).
__global__ void __launch_bounds__(256) zero_step_kernel(uint4 *j0, uint4 *j1, uint4 *j2,
                                                       int64_t n16, int32_t *status, int nstatus) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
        j0[i] = z;
        j1[i] = z;
        j2[i] = z;
    }
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < nstatus; i += blockDim.x) status[i] = 0;
}

__global__ void __launch_bounds__(256) zero_tail_kernel(unsigned char *j0, unsigned char *j1,
                                                       unsigned char *j2, int64_t from, int64_t bytes) {
    for (int64_t i = from + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < bytes;
         i += (int64_t)gridDim.x * blockDim.x) {
        j0[i] = 0;
        j1[i] = 0;
        j2[i] = 0;
    }
}

extern "C" int kwb_zero_step(const kwb_grid *g, void *const J[3], int32_t *status, int32_t n_status,
                             kwb_stream_t stream) {
    int rc = check_fields(g, "zero_step");
    if (rc) return rc;
    if ((J && !all3(J)) || (n_status > 0 && !status) || n_status < 0) {
        kwb_set_error("zero_step: NULL argument");
        return KWB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t bytes = J ? (int64_t)g->nx * g->ny * g->nz * (g->dtype == KWB_F32 ? 4 : 8) : 0;
    bool aligned = true;
    for (int c = 0; J && c < 3; ++c) aligned = aligned && ((uintptr_t)J[c] & 15) == 0;
    const int64_t n16 = aligned ? bytes / 16 : 0;
    const int64_t blocks = std::min<int64_t>((n16 + 255) / 256 + 1, 148 * 8);
    zero_step_kernel<<<(int)blocks, 256, 0, s>>>(J ? (uint4 *)J[0] : nullptr, J ? (uint4 *)J[1] : nullptr,
                                                 J ? (uint4 *)J[2] : nullptr, n16, status, n_status);
    if ((rc = kwb_check_launch("zero_step_kernel"))) return rc;
    if (bytes > n16 * 16) {
        zero_tail_kernel<<<148, 256, 0, s>>>((unsigned char *)J[0], (unsigned char *)J[1],
                                             (unsigned char *)J[2], n16 * 16, bytes);
        return kwb_check_launch("zero_tail_kernel");
    }
    return KWB_OK;
}

// ---- multi-GPU plumbing (z-slab fused halo, pic/decomp.py) ---------------

// Let THIS process's current device access `peer_device`'s memory (the
// advance kernel red.adds into the neighbour's J planes, the guard pulls
// read the neighbour's planes).  Already-enabled is success.
extern "C" int kwb_enable_peer_access(int32_t peer_device) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return kwb_check_launch("cudaGetDevice");
    if (peer_device == dev) return KWB_OK;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, dev, peer_device) != cudaSuccess || !can) {
        kwb_set_error("device %d cannot access peer device %d (no P2P / NVLink path)", dev,
                      peer_device);
        cudaGetLastError();
        return KWB_ECUDA;
    }
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();   // clear the sticky-free "already enabled" error
        return KWB_OK;
    }
    if (e != cudaSuccess) {
        kwb_set_error("cudaDeviceEnablePeerAccess(%d -> %d): %s", dev, peer_device,
                      cudaGetErrorString(e));
        return KWB_ECUDA;
    }
    return KWB_OK;
}

// bytes from src to dst on `stream` (the caller's own stream: a cross-GPU
// plane pull then runs on this GPU, reading the peer over NVLink, instead
// of being launched on the peer's stream).  Unified addressing.
extern "C" int kwb_copy_async(void *dst, const void *src, int64_t bytes, kwb_stream_t stream) {
    if (bytes < 0 || (bytes > 0 && (!dst || !src))) {
        kwb_set_error("copy_async: invalid argument");
        return KWB_EINVAL;
    }
    if (bytes == 0) return KWB_OK;
    const cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault,
                                          (cudaStream_t)stream);
    if (e != cudaSuccess) {
        kwb_set_error("cudaMemcpyAsync: %s", cudaGetErrorString(e));
        return KWB_ECUDA;
    }
    return KWB_OK;
}

extern "C" int kwb_fields_faraday_half(const kwb_grid *g, void *const E[3], void *const B[3],
                                       double half_dt, kwb_stream_t stream) {
    int rc = check_fields(g, "faraday");
    if (rc) return rc;
    if (!all3(E) || !all3(B)) { kwb_set_error("faraday: NULL field"); return KWB_EINVAL; }
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    if (g->dtype == KWB_F32)
        faraday_kernel<float><<<row_grid(g), row_threads(g), 0, s>>>(geo, rcp3(g), f3<float>(E), f3<float>(B), half_dt);
    else
        faraday_kernel<double><<<row_grid(g), row_threads(g), 0, s>>>(geo, rcp3(g), f3<double>(E), f3<double>(B), half_dt);
    return kwb_check_launch("faraday_kernel");
}

extern "C" int kwb_fields_ampere(const kwb_grid *g, void *const E[3], void *const B[3],
                                 void *const J[3], double dt, kwb_stream_t stream) {
    int rc = check_fields(g, "ampere");
    if (rc) return rc;
    if (!all3(E) || !all3(B) || !all3(J)) { kwb_set_error("ampere: NULL field"); return KWB_EINVAL; }
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    if (g->dtype == KWB_F32)
        ampere_kernel<float><<<row_grid(g), row_threads(g), 0, s>>>(geo, rcp3(g), f3<float>(E), f3<float>(B), f3<float>(J), dt);
    else
        ampere_kernel<double><<<row_grid(g), row_threads(g), 0, s>>>(geo, rcp3(g), f3<double>(E), f3<double>(B), f3<double>(J), dt);
    return kwb_check_launch("ampere_kernel");
}

extern "C" int kwb_continuity_residual(const kwb_grid *g, const double *rho_new,
                                       const double *rho_prev, void *const J[3], void *const E[3],
                                       double *G_prev, double *out, kwb_stream_t stream) {
    int rc = check_fields(g, "residual");
    if (rc) return rc;
    if (!rho_new || !out || !all3(J) || !all3(E)) {
        kwb_set_error("residual: NULL argument");
        return KWB_EINVAL;
    }
    Geo geo = geo_of(*g);
    const int64_t ncell = (int64_t)g->nx * g->ny * g->nz;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(out, 0, 2 * sizeof(double), s) != cudaSuccess)
        return kwb_check_launch("residual reset");
    if (g->dtype == KWB_F32)
        residual_kernel<float><<<grid_blocks(ncell), 256, 0, s>>>(geo, rho_new, rho_prev, f3<float>(J),
                                                                  f3<float>(E), G_prev, out);
    else
        residual_kernel<double><<<grid_blocks(ncell), 256, 0, s>>>(geo, rho_new, rho_prev, f3<double>(J),
                                                                   f3<double>(E), G_prev, out);
    return kwb_check_launch("residual_kernel");
}

extern "C" int kwb_field_stats(const kwb_grid *g, void *const E[3], void *const B[3], double *out,
                               kwb_stream_t stream) {
    int rc = check_fields(g, "field_stats");
    if (rc) return rc;
    if (!out || !all3(E) || !all3(B)) { kwb_set_error("field_stats: NULL argument"); return KWB_EINVAL; }
    Geo geo = geo_of(*g);
    const int64_t ncell = (int64_t)g->nx * g->ny * g->nz;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(out, 0, 2 * sizeof(double), s) != cudaSuccess)
        return kwb_check_launch("field_stats reset");
    if (g->dtype == KWB_F32)
        field_stats_kernel<float><<<grid_blocks(ncell), 256, 0, s>>>(geo, f3<float>(E), f3<float>(B), out);
    else
        field_stats_kernel<double><<<grid_blocks(ncell), 256, 0, s>>>(geo, f3<double>(E), f3<double>(B), out);
    return kwb_check_launch("field_stats_kernel");
}

unsigned long long kwb_chk_read_fields(int reset) {
#ifdef KWB_CHECKS
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, kwb::kwb_chk_count, sizeof(v));
    if (reset) {
        const unsigned long long z = 0;
        cudaMemcpyToSymbol(kwb::kwb_chk_count, &z, sizeof(z));
    }
    return v;
#else
    (void)reset;
    return 0;
#endif
}
