// Yee FDTD field update and field-side validation on sm_100a.
//
// Reference: pic/kernels.py:253-288 (`_faraday`, `_ampere`), pic/fields.py
// :145-169 (div B, div J, field energy), pic/sim.py:168-175 (continuity
// residual).  The reference walks cells per super cell; here one thread
// owns one cell of the x-fastest lattice, so every neighbour read along x is
// coalesced and +-y/+-z neighbours hit L1/L2.  Arithmetic follows the
// reference bit for bit: differences in the storage type, everything after
// the divide by a Python float in double, rounding on store.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace kwb {

template <typename F>
struct F3 {
    F *x, *y, *z;
};

// B -= half_dt * curl E (forward differences), pic/kernels.py:264-269.
template <typename F>
__global__ void __launch_bounds__(256) faraday_kernel(Geo g, F3<F> E, F3<F> B, double half_dt) {
    const int64_t ncell = (int64_t)g.nx * g.ny * g.nz;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(c % g.nx);
        const int j = (int)((c / g.nx) % g.ny);
        const int k = (int)(c / ((int64_t)g.nx * g.ny));
        const int64_t ip = fidx(i + 1 == g.nx ? 0 : i + 1, j, k, g.nx, g.ny);
        const int64_t jp = fidx(i, j + 1 == g.ny ? 0 : j + 1, k, g.nx, g.ny);
        const int64_t kp = fidx(i, j, k + 1 == g.nz ? 0 : k + 1, g.nx, g.ny);
        const F exc = E.x[c], eyc = E.y[c], ezc = E.z[c];
        F a = E.z[jp] - ezc, b = E.y[kp] - eyc;
        B.x[c] = (F)((double)B.x[c] - half_dt * ((double)a / g.dy - (double)b / g.dz));
        a = E.x[kp] - exc; b = E.z[ip] - ezc;
        B.y[c] = (F)((double)B.y[c] - half_dt * ((double)a / g.dz - (double)b / g.dx));
        a = E.y[ip] - eyc; b = E.x[jp] - exc;
        B.z[c] = (F)((double)B.z[c] - half_dt * ((double)a / g.dx - (double)b / g.dy));
    }
}

// E += dt * (curl B - J) (backward differences), pic/kernels.py:283-288.
template <typename F>
__global__ void __launch_bounds__(256) ampere_kernel(Geo g, F3<F> E, F3<F> B, F3<F> J, double dt) {
    const int64_t ncell = (int64_t)g.nx * g.ny * g.nz;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(c % g.nx);
        const int j = (int)((c / g.nx) % g.ny);
        const int k = (int)(c / ((int64_t)g.nx * g.ny));
        const int64_t im = fidx(i == 0 ? g.nx - 1 : i - 1, j, k, g.nx, g.ny);
        const int64_t jm = fidx(i, j == 0 ? g.ny - 1 : j - 1, k, g.nx, g.ny);
        const int64_t km = fidx(i, j, k == 0 ? g.nz - 1 : k - 1, g.nx, g.ny);
        const F bxc = B.x[c], byc = B.y[c], bzc = B.z[c];
        F a = bzc - B.z[jm], b = byc - B.y[km];
        E.x[c] = (F)((double)E.x[c] + dt * (((double)a / g.dy - (double)b / g.dz) - (double)J.x[c]));
        a = bxc - B.x[km]; b = bzc - B.z[im];
        E.y[c] = (F)((double)E.y[c] + dt * (((double)a / g.dz - (double)b / g.dx) - (double)J.y[c]));
        a = byc - B.y[im]; b = bxc - B.x[jm];
        E.z[c] = (F)((double)E.z[c] + dt * (((double)a / g.dx - (double)b / g.dy) - (double)J.z[c]));
    }
}

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

extern "C" int kwb_fields_faraday_half(const kwb_grid *g, void *const E[3], void *const B[3],
                                       double half_dt, kwb_stream_t stream) {
    int rc = check_fields(g, "faraday");
    if (rc) return rc;
    if (!all3(E) || !all3(B)) { kwb_set_error("faraday: NULL field"); return KWB_EINVAL; }
    Geo geo = geo_of(*g);
    const int64_t ncell = (int64_t)g->nx * g->ny * g->nz;
    cudaStream_t s = (cudaStream_t)stream;
    if (g->dtype == KWB_F32)
        faraday_kernel<float><<<grid_blocks(ncell), 256, 0, s>>>(geo, f3<float>(E), f3<float>(B), half_dt);
    else
        faraday_kernel<double><<<grid_blocks(ncell), 256, 0, s>>>(geo, f3<double>(E), f3<double>(B), half_dt);
    return kwb_check_launch("faraday_kernel");
}

extern "C" int kwb_fields_ampere(const kwb_grid *g, void *const E[3], void *const B[3],
                                 void *const J[3], double dt, kwb_stream_t stream) {
    int rc = check_fields(g, "ampere");
    if (rc) return rc;
    if (!all3(E) || !all3(B) || !all3(J)) { kwb_set_error("ampere: NULL field"); return KWB_EINVAL; }
    Geo geo = geo_of(*g);
    const int64_t ncell = (int64_t)g->nx * g->ny * g->nz;
    cudaStream_t s = (cudaStream_t)stream;
    if (g->dtype == KWB_F32)
        ampere_kernel<float><<<grid_blocks(ncell), 256, 0, s>>>(geo, f3<float>(E), f3<float>(B), f3<float>(J), dt);
    else
        ampere_kernel<double><<<grid_blocks(ncell), 256, 0, s>>>(geo, f3<double>(E), f3<double>(B), f3<double>(J), dt);
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
