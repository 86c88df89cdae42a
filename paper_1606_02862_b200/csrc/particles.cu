// Particle path of the PIC cycle on sm_100a: the fused advance (gather,
// Boris push, move, Esirkepov deposit, in-super-cell shift), the cross-
// super-cell shift, and store load/export/repack.
//
// Reference: pic/kernels.py:26-250 (stage loops) and :329-412 (kernel
// objects), kw/atomics.py:147-163 (deposit-halo merge), pic/particles.py
// :214-345 (migration).  As in the reference one block owns one super cell
// (§2.1), but here ONE kernel does all four particle stages:
//
//  * Store = cell-column frames (include/kwb200.h): thread t of the CTA owns
//    local cell t and walks column t, so every particle a thread touches is
//    in its own cell.  Frame k of 32 adjacent cells is one coalesced 128-B
//    load per SoA column.
//  * E/B of the super cell + one guard cell are staged in shared memory once
//    per CTA (the trilinear support of cell c is c-1..c+1).
//  * Deposit of particles that stay in their cell (~94 %): accumulated in
//    54 registers per thread (the 2 x 3 x 3 non-closing running-sum entries
//    per component), reduced into a shared J tile once per super cell in
//    conflict-free barrier-separated sweeps -- no atomics at all.  Shared
//    fp32 atomicAdd is a CAS loop on sm_100a (~2.6 ops/clk/SM measured), so
//    this is the design's central choice.
//  * Particles that cross a cell face are queued per warp in shared memory
//    and deposited by the whole warp (anchor-shifted 4-point supports, CAS
//    into the J tile); PCS and float64 use this path for every particle.
//  * The J tile (super cell + shape halo) is flushed once with coalesced
//    red.global.add; leavers of the super cell go to an exchange buffer.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace kwb {

#include "advance.cuh"
#include "push.cuh"

// Append leavers to the back of their new column (the cross-super-cell
// shift, pic/particles.py:316-345).  Slot claims are atomic per column.
// All species of a step at once: dest = super cell + species * n_sc.
constexpr int kMaxSpecies = 4;
template <typename F>
struct ShiftOut {
    StoreT<F> out[kMaxSpecies];
};
template <typename F>
__global__ void shift_kernel(ShiftOut<F> so, int n_species, ExchT<F> ex, Geo g,
                             int32_t *__restrict__ status) {
    int n = *ex.count;
    if (n > ex.capacity) n = ex.capacity;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&status[KWB_ST_LEAVERS], n);
    const int V = g.scx * g.scy * g.scz, n_sc = g.gx * g.gy * g.gz;
    int fill_max[kMaxSpecies] = {};   // warp-aggregated: one atomicMax per warp and species
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int d = ex.dest[i];
        const int s = d / n_sc;
        d -= s * n_sc;
        if (!KWB_IN(s >= 0 && s < n_species)) continue;
        // compile-time indices: a runtime index into the parameter array
        // would copy it to local memory
        const StoreT<F> o_ = s == 0 ? so.out[0] : s == 1 ? so.out[1] : s == 2 ? so.out[2]
                                                                      : so.out[kMaxSpecies - 1];
        const int K = o_.frames;
        const int bx = d % g.gx, by = (d / g.gx) % g.gy, bz = d / (g.gx * g.gy);
        const int c = (ex.cx[i] - bx * g.scx) +
                      g.scx * ((ex.cy[i] - by * g.scy) + g.scy * (ex.cz[i] - bz * g.scz));
        if (!KWB_IN(d >= 0 && d < n_sc && c >= 0 && c < V)) continue;
        const int64_t colx = (int64_t)d * V + c;
        const int slot = atomicAdd(&o_.back[colx], 1);
        const int fill = o_.front[colx] + slot + 1;
        if (fill > K) {
            atomicSub(&o_.back[colx], 1);
            atomicAdd(&status[s * KWB_STATUS_WORDS + KWB_ST_STORE_OVERFLOW], 1);
            continue;
        }
#pragma unroll
        for (int k = 0; k < kMaxSpecies; ++k)
            if (k == s) fill_max[k] = max(fill_max[k], fill);
        const int64_t o = ((int64_t)d * K + (K - 1 - slot)) * V + c;
        o_.ox[o] = ex.ox[i]; o_.oy[o] = ex.oy[i]; o_.oz[o] = ex.oz[i];
        o_.ux[o] = ex.ux[i]; o_.uy[o] = ex.uy[i]; o_.uz[o] = ex.uz[i];
        o_.w[o] = ex.w[i];
    }
#pragma unroll
    for (int k = 0; k < kMaxSpecies; ++k) {
        const int m = __reduce_max_sync(0xffffffffu, fill_max[k]);
        if ((threadIdx.x & 31) == 0 && m > 0 && k < n_species)
            atomicMax(&status[k * KWB_STATUS_WORDS + KWB_ST_MAX_COUNT], m);
    }
}

// ---- store load / export / repack ---------------------------------------

// n_dev != NULL: the record count is read on the device (min(*n_dev, n)),
// so a received message can be appended without a host round trip.
template <typename F>
__global__ void load_kernel(Geo g, StoreT<F> st, int64_t n, const int64_t *__restrict__ n_dev,
                            const int32_t *__restrict__ cx,
                            const int32_t *__restrict__ cy, const int32_t *__restrict__ cz,
                            const F *__restrict__ ox, const F *__restrict__ oy,
                            const F *__restrict__ oz, const F *__restrict__ ux,
                            const F *__restrict__ uy, const F *__restrict__ uz,
                            const F *__restrict__ w, int32_t *__restrict__ status) {
    const int V = g.scx * g.scy * g.scz, K = st.frames;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (n_dev) n = min(n, *n_dev);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int x = cx[i], y = cy[i], z = cz[i];
        if (x < 0 || x >= g.nx || y < 0 || y >= g.ny || z < 0 || z >= g.nz) {
            atomicAdd(&status[KWB_ST_LOAD_ERRORS], 1);
            continue;
        }
        const int s = (x / g.scx) + g.gx * ((y / g.scy) + g.gy * (z / g.scz));
        const int c = (x % g.scx) + g.scx * ((y % g.scy) + g.scy * (z % g.scz));
        const int64_t colx = (int64_t)s * V + c;
        const int k = atomicAdd(&st.front[colx], 1);
        if (k + st.back[colx] >= K) {
            atomicSub(&st.front[colx], 1);
            atomicAdd(&status[KWB_ST_LOAD_ERRORS], 1);
            continue;
        }
        const int64_t o = ((int64_t)s * K + k) * V + c;
        st.ox[o] = ox[i]; st.oy[o] = oy[i]; st.oz[o] = oz[i];
        st.ux[o] = ux[i]; st.uy[o] = uy[i]; st.uz[o] = uz[i];
        st.w[o] = w[i];
    }
}

template <typename F>
__global__ void export_kernel(Geo g, StoreT<F> st, int64_t col0, int64_t col1,
                              const int64_t *__restrict__ cell_start, int clear, int32_t *cx,
                              int32_t *cy, int32_t *cz, F *ox, F *oy, F *oz, F *ux, F *uy, F *uz,
                              F *w, int64_t capacity, int64_t *count_out, int32_t *status) {
    const int V = g.scx * g.scy * g.scz, K = st.frames;
    if (capacity >= 0) {   // bounded: all or nothing for the whole column range
        const int64_t total = cell_start[col1 - col0];
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            *count_out = total <= capacity ? total : 0;
            if (total > capacity) atomicAdd(&status[KWB_ST_GUARD_OVERFLOW], (int)(total - capacity));
        }
        if (total > capacity) return;
    }
    for (int64_t colx = col0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; colx < col1;
         colx += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(colx / V), c = (int)(colx % V);
        const int bx = s % g.gx, by = (s / g.gx) % g.gy, bz = s / (g.gx * g.gy);
        const int x = bx * g.scx + c % g.scx, y = by * g.scy + (c / g.scx) % g.scy,
                  z = bz * g.scz + c / (g.scx * g.scy);
        const int f = st.front[colx], b = st.back[colx];
        int64_t o = cell_start[colx - col0];
        if (!KWB_IN(f >= 0 && b >= 0 && f + b <= K)) continue;
        for (int j = 0; j < f + b; ++j, ++o) {
            const int k = j < f ? j : K - b + (j - f);
            const int64_t q = ((int64_t)s * K + k) * V + c;
            cx[o] = x; cy[o] = y; cz[o] = z;
            ox[o] = st.ox[q]; oy[o] = st.oy[q]; oz[o] = st.oz[q];
            ux[o] = st.ux[q]; uy[o] = st.uy[q]; uz[o] = st.uz[q];
            w[o] = st.w[q];
        }
        if (clear) { st.front[colx] = 0; st.back[colx] = 0; }
    }
}

// Export of whole super cells, one CTA each: the CTA's records occupy one
// contiguous output range (canonical order), so each array is staged in
// shared memory -- threads scatter their column's records to their output
// offsets there -- and written out with coalesced stores.  The column-per-
// thread export_kernel writes 32 scattered records per warp store.
template <typename F>
__global__ void export_sc_kernel(Geo g, StoreT<F> st, int64_t col0, const int64_t *__restrict__ cell_start,
                                 int clear, int32_t *cx, int32_t *cy, int32_t *cz, F *ox, F *oy,
                                 F *oz, F *ux, F *uy, F *uz, F *w, int chunk) {
    extern __shared__ __align__(16) unsigned char xs_raw[];
    const int V = g.scx * g.scy * g.scz, K = st.frames, t = threadIdx.x;
    const int64_t s = col0 / V + blockIdx.x;
    const int64_t sc_first = s * V - col0;               // local index of this super cell's column 0
    const int64_t S0 = cell_start[sc_first], S1 = cell_start[sc_first + V];
    const bool owner = t < V;
    int f = 0, b = 0;
    int64_t my0 = 0;
    int x = 0, y = 0, z = 0;
    if (owner) {
        const int64_t colx = s * V + t;
        f = st.front[colx]; b = st.back[colx];
        my0 = cell_start[sc_first + t];
        const int bx = (int)(s % g.gx), by = (int)((s / g.gx) % g.gy), bz = (int)(s / ((int64_t)g.gx * g.gy));
        x = bx * g.scx + t % g.scx; y = by * g.scy + (t / g.scx) % g.scy;
        z = bz * g.scz + t / (g.scx * g.scy);
    }
    const int n = f + b;
    F *bf = reinterpret_cast<F *>(xs_raw);
    int32_t *bi = reinterpret_cast<int32_t *>(xs_raw);
    for (int64_t base = S0; base < S1; base += chunk) {
        const int64_t m = min((int64_t)chunk, S1 - base);
        const int j0 = (int)max((int64_t)0, base - my0), j1 = (int)min((int64_t)n, base + chunk - my0);
        // three cell arrays (constant per column), then the seven F arrays
        for (int a = 0; a < 10; ++a) {
            if (a < 3) {
                const int v = a == 0 ? x : a == 1 ? y : z;
                for (int j = j0; j < j1; ++j)
                    if (KWB_IN(my0 + j - base >= 0 && my0 + j - base < m)) bi[my0 + j - base] = v;
            } else {
                const F *src = a == 3 ? st.ox : a == 4 ? st.oy : a == 5 ? st.oz : a == 6 ? st.ux
                             : a == 7 ? st.uy : a == 8 ? st.uz : st.w;
                for (int j = j0; j < j1; ++j) {
                    const int k = j < f ? j : K - b + (j - f);
                    if (KWB_IN(my0 + j - base >= 0 && my0 + j - base < m && k >= 0 && k < K))
                        bf[my0 + j - base] = src[(s * K + k) * V + t];
                }
            }
            __syncthreads();
            if (a < 3) {
                int32_t *dst = a == 0 ? cx : a == 1 ? cy : cz;
                for (int i = t; i < m; i += blockDim.x) dst[base - cell_start[0] + i] = bi[i];
            } else {
                F *dst = a == 3 ? ox : a == 4 ? oy : a == 5 ? oz : a == 6 ? ux : a == 7 ? uy
                       : a == 8 ? uz : w;
                for (int i = t; i < m; i += blockDim.x) dst[base - cell_start[0] + i] = bf[i];
            }
            __syncthreads();
        }
    }
    if (clear && owner) {
        st.front[s * V + t] = 0;
        st.back[s * V + t] = 0;
    }
}

template <typename F>
__global__ void repack_kernel(Geo g, StoreT<F> src, StoreT<F> dst) {
    const int V = g.scx * g.scy * g.scz, Ks = src.frames, Kd = dst.frames;
    const int64_t ncol = (int64_t)g.gx * g.gy * g.gz * V;
    for (int64_t colx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; colx < ncol;
         colx += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(colx / V), c = (int)(colx % V);
        const int f = src.front[colx], b = src.back[colx];
        if (!KWB_IN(f >= 0 && b >= 0 && f + b <= Ks)) continue;
        const int n = min(f + b, Kd);
        for (int j = 0; j < n; ++j) {
            const int k = j < f ? j : Ks - b + (j - f);
            const int64_t a = ((int64_t)s * Ks + k) * V + c, o = ((int64_t)s * Kd + j) * V + c;
            dst.ox[o] = src.ox[a]; dst.oy[o] = src.oy[a]; dst.oz[o] = src.oz[a];
            dst.ux[o] = src.ux[a]; dst.uy[o] = src.uy[a]; dst.uz[o] = src.uz[a];
            dst.w[o] = src.w[a];
        }
        dst.front[colx] = n;
        dst.back[colx] = 0;
    }
}

// Visit every particle of a store: f(colx, s, c, q) with q the slot index.
template <typename F, typename Fn>
__device__ __forceinline__ void for_column(const StoreT<F> &st, int s, int c, int V, Fn fn) {
    const int64_t colx = (int64_t)s * V + c;
    const int f = st.front[colx], b = st.back[colx], K = st.frames;
    if (!KWB_IN(f >= 0 && b >= 0 && f + b <= K)) return;
    for (int j = 0; j < f + b; ++j) {
        const int k = j < f ? j : K - b + (j - f);
        fn(((int64_t)s * K + k) * V + c);
    }
}

// ---- validation charge density and particle moments --------------------

// pic/kernels.py:291-326 `_rho_tsc` (order 2) and the matching CIC/PCS shape
// deposits; float64 accumulation with global atomics.
template <typename F, int ORDER>
__global__ void rho_kernel(Geo g, StoreT<F> st, double q_inv_vol, double *__restrict__ rho) {
    const int V = g.scx * g.scy * g.scz;
    const int s = blockIdx.x, c = threadIdx.x;
    if (c >= V) return;
    const int bx = s % g.gx, by = (s / g.gx) % g.gy, bz = s / (g.gx * g.gy);
    const int cx = bx * g.scx + c % g.scx, cy = by * g.scy + (c / g.scx) % g.scy,
              cz = bz * g.scz + c / (g.scx * g.scy);
    for_column(st, s, c, V, [&](int64_t q) {
        const double qw = q_inv_vol * (double)st.w[q];
        if (ORDER == 2) {
            double wx[3], wy[3], wz[3], o, l, r;
            o = (double)st.ox[q] - 0.5; l = 0.5 * ((0.5 - o) * (0.5 - o)); r = 0.5 * ((0.5 + o) * (0.5 + o));
            wx[0] = l; wx[1] = (1.0 - l) - r; wx[2] = r;
            o = (double)st.oy[q] - 0.5; l = 0.5 * ((0.5 - o) * (0.5 - o)); r = 0.5 * ((0.5 + o) * (0.5 + o));
            wy[0] = l; wy[1] = (1.0 - l) - r; wy[2] = r;
            o = (double)st.oz[q] - 0.5; l = 0.5 * ((0.5 - o) * (0.5 - o)); r = 0.5 * ((0.5 + o) * (0.5 + o));
            wz[0] = l; wz[1] = (1.0 - l) - r; wz[2] = r;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int ia = pymod(cx - 1 + a, g.nx);
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    const int jb = pymod(cy - 1 + b, g.ny);
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        const int kd = pymod(cz - 1 + d, g.nz);
                        atomicAdd(rho + fidx(ia, jb, kd, g.nx, g.ny), ((qw * wx[a]) * wy[b]) * wz[d]);
                    }
                }
            }
        } else {
            constexpr int NP = Shape<ORDER>::NP, H = Shape<ORDER>::H;
            F sx[NP], sy[NP], sz[NP];
            shape_into<F, ORDER>((double)st.ox[q], sx);
            shape_into<F, ORDER>((double)st.oy[q], sy);
            shape_into<F, ORDER>((double)st.oz[q], sz);
#pragma unroll
            for (int a = 0; a < NP; ++a) {
                if (sx[a] == F(0)) continue;
                const int ia = pymod(cx - H + a, g.nx);
#pragma unroll
                for (int b = 0; b < NP; ++b) {
                    if (sy[b] == F(0)) continue;
                    const int jb = pymod(cy - H + b, g.ny);
#pragma unroll
                    for (int d = 0; d < NP; ++d) {
                        if (sz[d] == F(0)) continue;
                        const int kd = pymod(cz - H + d, g.nz);
                        atomicAdd(rho + fidx(ia, jb, kd, g.nx, g.ny),
                                  ((qw * (double)sx[a]) * (double)sy[b]) * (double)sz[d]);
                    }
                }
            }
        }
    });
}

__device__ __forceinline__ double block_sum(double v, double *red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
    return t;  // valid on thread 0
}

// census, sum q w, sum m (gamma - 1) w (pic/sim.py:191-214)
template <typename F>
__global__ void __launch_bounds__(256)
moments_kernel(Geo g, StoreT<F> st, double charge, double mass, double *__restrict__ out) {
    __shared__ double red[8];
    const int V = g.scx * g.scy * g.scz;
    const int64_t ncol = (int64_t)g.gx * g.gy * g.gz * V;
    double cen = 0.0, qw = 0.0, ke = 0.0;
    for (int64_t colx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; colx < ncol;
         colx += (int64_t)gridDim.x * blockDim.x) {
        for_column(st, (int)(colx / V), (int)(colx % V), V, [&](int64_t q) {
            const double ux = (double)st.ux[q], uy = (double)st.uy[q], uz = (double)st.uz[q];
            const double ww = (double)st.w[q];
            const double gm = sqrt(((1.0 + ux * ux) + uy * uy) + uz * uz);
            cen += 1.0;
            qw += ww;
            ke += (gm - 1.0) * ww;
        });
    }
    const double a = block_sum(cen, red);
    const double b = block_sum(qw, red);
    const double c = block_sum(ke, red);
    if (threadIdx.x == 0) {
        atomicAdd(out + 0, a);
        atomicAdd(out + 1, charge * b);
        atomicAdd(out + 2, mass * c);
    }
}

}  // namespace kwb

// ============================ C ABI =======================================
using namespace kwb;

static int check_grid(const kwb_grid *g) {
    if (!g) { kwb_set_error("grid is NULL"); return KWB_EINVAL; }
    if (g->nx <= 0 || g->ny <= 0 || g->nz <= 0 || g->scx <= 0 || g->scy <= 0 || g->scz <= 0) {
        kwb_set_error("non-positive grid extent");
        return KWB_EINVAL;
    }
    if (g->nx % g->scx || g->ny % g->scy || g->nz % g->scz || g->gx != g->nx / g->scx ||
        g->gy != g->ny / g->scy || g->gz != g->nz / g->scz) {
        kwb_set_error("super cell (%d,%d,%d) does not tile cells (%d,%d,%d)", g->scx, g->scy,
                      g->scz, g->nx, g->ny, g->nz);
        return KWB_EINVAL;
    }
    if (g->scx * g->scy * g->scz > kMaxCells || g->scx > 255 || g->scy > 255 || g->scz > 255) {
        kwb_set_error("super-cell volume %d exceeds %d cells (one thread per cell)",
                      g->scx * g->scy * g->scz, kMaxCells);
        return KWB_EINVAL;
    }
    if (g->dtype != KWB_F32 && g->dtype != KWB_F64) {
        kwb_set_error("dtype must be KWB_F32 or KWB_F64");
        return KWB_EINVAL;
    }
    return KWB_OK;
}

static int check_store(const kwb_store *s, const char *what) {
    if (!s || !s->ox || !s->oy || !s->oz || !s->ux || !s->uy || !s->uz || !s->w || !s->front ||
        !s->back || s->frames_per_sc <= 0) {
        kwb_set_error("%s store is incomplete", what);
        return KWB_EINVAL;
    }
    return KWB_OK;
}

// KWB_CHECKS counters of the three modules (0 in a normal build).
#ifdef KWB_CHECKS
static unsigned long long chk_read(int reset) {
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, kwb_chk_count, sizeof(v));
    if (reset) {
        const unsigned long long z = 0;
        cudaMemcpyToSymbol(kwb_chk_count, &z, sizeof(z));
    }
    return v;
}
#endif
unsigned long long kwb_chk_read_fields(int reset);
unsigned long long kwb_chk_read_init(int reset);

extern "C" int64_t kwb_check_failures(int32_t reset) {
#ifdef KWB_CHECKS
    cudaDeviceSynchronize();
    return (int64_t)(chk_read(reset) + kwb_chk_read_fields(reset) + kwb_chk_read_init(reset));
#else
    (void)reset;
    return -1;   // not a checks build
#endif
}

static int block_threads(const kwb_grid *g) {
    const int V = g->scx * g->scy * g->scz;
    return (V + 31) / 32 * 32;
}

// ---- TMA tensor maps of the field lattices ---------------------------------
// The encoder is a driver entry point (no -lcuda): cudaGetDriverEntryPoint.
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
        cudaGetLastError();
    }
    return fn;
}

// n lattices at base, base + L, ..., L = one lattice's bytes, each (nx, ny,
// nz) x fastest: a 4-D map (x, y, z, lattice) with the given box.  false when
// the layout does not qualify (not equally spaced / not 16-byte multiples).
template <typename F>
static bool lattice_map(CUtensorMap *m, void *const *ptrs, int n, const kwb_grid *g,
                        const cuuint32_t box[4]) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn || getenv("KWB_NO_TMA")) return false;
    const cuuint64_t L = (cuuint64_t)g->nx * g->ny * g->nz * sizeof(F);
    const uintptr_t base = (uintptr_t)ptrs[0];
    for (int i = 0; i < n; ++i)
        if ((uintptr_t)ptrs[i] != base + i * L) return false;
    if (base % 16 || ((cuuint64_t)g->nx * sizeof(F)) % 16 || L % 16 || (box[0] * sizeof(F)) % 16)
        return false;
    const cuuint64_t dims[4] = {(cuuint64_t)g->nx, (cuuint64_t)g->ny, (cuuint64_t)g->nz,
                                (cuuint64_t)n};
    const cuuint64_t strides[3] = {(cuuint64_t)g->nx * sizeof(F),
                                   (cuuint64_t)g->nx * g->ny * sizeof(F), L};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(m, sizeof(F) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
              4, (void *)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int sm_count();
template <typename F>
static int shift_launch(const kwb_grid *g, int n, const kwb_store *out, const kwb_exchange *ex,
                        int32_t *status, cudaStream_t s) {
    ShiftOut<F> so;
    memset(&so, 0, sizeof(so));
    for (int i = 0; i < n; ++i) so.out[i] = store_of<F>(out[i]);
    shift_kernel<F><<<sm_count() * 4, 256, 0, s>>>(so, n, exch_of<F>(*ex), geo_of(*g), status);
    return kwb_check_launch("shift_kernel");
}
static int shift_all(const kwb_grid *g, int n, const kwb_store *out, const kwb_exchange *ex,
                     int32_t *status, kwb_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    return g->dtype == KWB_F32 ? shift_launch<float>(g, n, out, ex, status, s)
                               : shift_launch<double>(g, n, out, ex, status, s);
}

// sp / in / out: NS entries; status: NS x KWB_STATUS_WORDS
// SPLIT: push_kernel (gather/push/move into the workspace store ws) then
// the deposit/shift kernel reading it (csrc/push.cuh).
template <typename F, int ORDER, bool REGACC, int SX, int SY, int SZ, int NS, bool SPLIT = false>
static int launch_advance(const kwb_grid *g, const kwb_species *sp, const kwb_store *in,
                          const kwb_store *out, const kwb_exchange *ex, void *const E[3],
                          void *const B[3], void *const J[3], void *const *jpl,
                          int32_t *status, cudaStream_t stream, int sp0, bool reset,
                          const kwb_store *ws = nullptr) {
    Geo geo = geo_of(*g);
    const int threads = block_threads(g);
    const size_t smem = adv_layout<F, ORDER, NS, SPLIT>(g->scx, g->scy, g->scz).bytes;
    auto kern = advance_kernel<F, ORDER, REGACC, SX, SY, SZ, NS, SPLIT>;
    if (smem > 227 * 1024) {
        kwb_set_error("super cell too large for the shared-memory tiles (%zu B)", smem);
        return KWB_EINVAL;
    }
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    FieldPtrs fp;
    for (int c = 0; c < 3; ++c) { fp.E[c] = E[c]; fp.B[c] = B[c]; fp.J[c] = J[c]; }
    fp.jpl = jpl;
    if (reset && cudaMemsetAsync(ex->count, 0, sizeof(int32_t), stream) != cudaSuccess)
        return kwb_check_launch("exchange counter reset");
    const int n_sc = g->gx * g->gy * g->gz;
    // E/B box: the tile (super cell + 1 guard) from a 16-byte aligned x start
    // (origin - 4 for f32, origin - 2 for f64; csrc/advance.cuh kTmaX0)
    CUtensorMap tm_eb;
    memset(&tm_eb, 0, sizeof(tm_eb));
    int tma = 0;
    const size_t stage_room =
        SPLIT ? (size_t)6 * push_layout<F>(g->scx, g->scy, g->scz).boxx * (g->scy + 2) *
                    (g->scz + 2) * sizeof(F)
              : adv_layout<F, ORDER, NS>(g->scx, g->scy, g->scz).off_arr -
                    adv_layout<F, ORDER, NS>(g->scx, g->scy, g->scz).off_qf;
    if (REGACC) {
        const cuuint32_t vec = 16 / sizeof(F), x0 = sizeof(F) == 4 ? 4 : 2;
        const cuuint32_t need = (cuuint32_t)g->scx + 1 + x0;   // origin - x0 .. origin + scx
        const cuuint32_t ebox[4] = {(need + vec - 1) / vec * vec, (cuuint32_t)g->scy + 2,
                                    (cuuint32_t)g->scz + 2, 6};
        void *eb[6] = {E[0], E[1], E[2], B[0], B[1], B[2]};
        // the box start origin - x0 is 16-byte aligned when scx is a multiple of x0
        if (g->scx % x0 == 0 && ebox[0] <= 256 && ebox[1] <= 256 && ebox[2] <= 256 &&
            (size_t)6 * ebox[0] * ebox[1] * ebox[2] * sizeof(F) <= stage_room &&
            lattice_map<F>(&tm_eb, eb, 6, g, ebox))
            tma |= TMA_EB;
        if (const char *m = getenv("KWB_TMA_MASK")) tma &= atoi(m);   // debugging / A/B
    }
    SpeciesB<F> sb;
    memset(&sb, 0, sizeof(sb));
    if (NS == 2) {
        sb.in = store_of<F>(in[1]);
        sb.out = store_of<F>(out[1]);
        sb.sp = sp[1];
        sb.status = status + KWB_STATUS_WORDS;
    }
    if constexpr (SPLIT) {
        const StoreT<F> wst = store_of<F>(ws[0]);
        auto pk = push_kernel<F, SX, SY, SZ>;
        const size_t psm = push_layout<F>(g->scx, g->scy, g->scz).bytes;
        if (psm > 48 * 1024)
            cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
        pk<<<n_sc, threads, psm, stream>>>(geo, sp[0], store_of<F>(in[0]), wst, fp, tm_eb, tma);
        if (int rc = kwb_check_launch("push_kernel")) return rc;
        sb.in = wst;
        tma = 0;
    }
    kern<<<n_sc, threads, smem, stream>>>(geo, sp[0], store_of<F>(in[0]), store_of<F>(out[0]),
                                          exch_of<F>(*ex), fp, status, tm_eb, tma, sb, sp0);
    return kwb_check_launch("advance_kernel");
}

// Compile-time (8,8,4) super cell (the reference default, every BASELINE
// config) or a runtime-shaped generic instance.
template <typename F, int ORDER, bool REGACC, int NS>
static int dispatch_advance(const kwb_grid *g, const kwb_species *sp, const kwb_store *in,
                            const kwb_store *out, const kwb_exchange *ex, void *const E[3],
                            void *const B[3], void *const J[3], void *const *jpl,
                            int32_t *status, cudaStream_t stream, int sp0, bool reset) {
    if (g->scx == 8 && g->scy == 8 && g->scz == 4)
        return launch_advance<F, ORDER, REGACC, 8, 8, 4, NS>(g, sp, in, out, ex, E, B, J, jpl,
                                                             status, stream, sp0, reset);
    return launch_advance<F, ORDER, REGACC, 0, 0, 0, NS>(g, sp, in, out, ex, E, B, J, jpl, status,
                                                         stream, sp0, reset);
}

template <int NS>
static int advance_ns(const kwb_grid *g, const kwb_species *sp, const kwb_store *in,
                      const kwb_store *out, const kwb_exchange *ex, void *const E[3],
                      void *const B[3], void *const J[3], void *const *jpl, int shape_order,
                      int32_t *status, cudaStream_t s, int sp0 = 0, bool reset = true) {
    if (g->dtype == KWB_F32) {
        switch (shape_order) {
            case 1: return dispatch_advance<float, 1, true, NS>(g, sp, in, out, ex, E, B, J, jpl, status, s, sp0, reset);
            case 2: return dispatch_advance<float, 2, true, NS>(g, sp, in, out, ex, E, B, J, jpl, status, s, sp0, reset);
            case 3: return dispatch_advance<float, 3, false, NS>(g, sp, in, out, ex, E, B, J, jpl, status, s, sp0, reset);
        }
    } else {
        switch (shape_order) {
            case 1: return dispatch_advance<double, 1, true, NS>(g, sp, in, out, ex, E, B, J, jpl, status, s, sp0, reset);
            case 2: return dispatch_advance<double, 2, true, NS>(g, sp, in, out, ex, E, B, J, jpl, status, s, sp0, reset);
            case 3: return dispatch_advance<double, 3, false, NS>(g, sp, in, out, ex, E, B, J, jpl, status, s, sp0, reset);
        }
    }
    kwb_set_error("shape_order must be 1 (CIC), 2 (TSC) or 3 (PCS), got %d", shape_order);
    return KWB_EINVAL;
}

extern "C" int kwb_particles_advance(const kwb_grid *g, const kwb_species *sp,
                                     const kwb_store *in, const kwb_store *out,
                                     const kwb_exchange *ex, void *const E[3], void *const B[3],
                                     void *const J[3], int shape_order, int32_t *status,
                                     kwb_stream_t stream) {
    return kwb_particles_advance_zslab(g, sp, in, out, ex, E, B, J, nullptr, shape_order, status,
                                       stream);
}

extern "C" int kwb_particles_advance_zslab(const kwb_grid *g, const kwb_species *sp,
                                           const kwb_store *in, const kwb_store *out,
                                           const kwb_exchange *ex, void *const E[3],
                                           void *const B[3], void *const J[3],
                                           void *const *j_planes, int shape_order,
                                           int32_t *status, kwb_stream_t stream) {
    void *const *jpl = j_planes;
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(in, "input")) || (rc = check_store(out, "output"))) return rc;
    if (!sp || !ex || !ex->count || !status || !E || !B || !J) {
        kwb_set_error("advance: NULL argument");
        return KWB_EINVAL;
    }
    if (out->frames_per_sc != in->frames_per_sc) {
        kwb_set_error("advance: input and output stores differ in frames_per_sc");
        return KWB_EINVAL;
    }
    return advance_ns<1>(g, sp, in, out, ex, E, B, J, jpl, shape_order, status,
                         (cudaStream_t)stream);
}

// All species of a Simulation in as few launches as possible: two species
// share one fused launch (lane-level fusion, csrc/advance.cuh SpeciesB);
// otherwise one launch per species.  The exchange buffer is shared (a fused
// launch encodes the species in dest, see kwb_particles_shift_species).
extern "C" int kwb_particles_advance_species(const kwb_grid *g, int32_t n_species,
                                             const kwb_species *sp, const kwb_store *in,
                                             const kwb_store *out, const kwb_exchange *ex,
                                             void *const E[3], void *const B[3],
                                             void *const J[3], void *const *j_planes,
                                             int shape_order, int32_t *status,
                                             kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if (n_species < 1 || !sp || !in || !out || !ex || !ex->count || !status || !E || !B || !J) {
        kwb_set_error("advance_species: NULL argument or no species");
        return KWB_EINVAL;
    }
    for (int i = 0; i < n_species; ++i) {
        if ((rc = check_store(in + i, "input")) || (rc = check_store(out + i, "output"))) return rc;
        if (out[i].frames_per_sc != in[i].frames_per_sc) {
            kwb_set_error("advance_species: input and output stores differ in frames_per_sc");
            return KWB_EINVAL;
        }
    }
    if (n_species > kMaxSpecies) {
        kwb_set_error("advance_species: at most %d species", kMaxSpecies);
        return KWB_EINVAL;
    }
    // The species-fused launch (lane-level fusion, NS = 2) is opt-in: on C2
    // it issues as many warp instructions as the two per-species launches
    // (+1.5 %: the species selects eat the lane-balance gain, active lanes
    // 25.6 -> 26.4 of 32) and stalls more (7.8 vs 6.7 cycles per issue:
    // 9 spilled registers in the hot loop, L1 is ~3 KB next to 2 x 112 KB of
    // shared memory): 8.14 ms vs 2 x 3.48 ms (ncu, tools/gpurun/r02i_ncu.sh).
    if (n_species == 2 && getenv("KWB_SPECIES_FUSION") && getenv("KWB_SPECIES_FUSION")[0] == '1')
        return advance_ns<2>(g, sp, in, out, ex, E, B, J, j_planes, shape_order, status,
                             (cudaStream_t)stream);
    // one launch per species, all appending their leavers to the one
    // exchange buffer (dest carries the species; counter reset once)
    for (int i = 0; i < n_species; ++i) {
        rc = advance_ns<1>(g, sp + i, in + i, out + i, ex, E, B, J, j_planes, shape_order,
                           status + i * KWB_STATUS_WORDS, (cudaStream_t)stream, i, i == 0);
        if (rc) return rc;
    }
    return KWB_OK;
}

template <typename F, int ORDER>
static int split_one(const kwb_grid *g, const kwb_species *sp, const kwb_store *in,
                     const kwb_store *out, const kwb_store *ws, const kwb_exchange *ex,
                     void *const E[3], void *const B[3], void *const J[3], void *const *jpl,
                     int32_t *status, cudaStream_t s, int sp0, bool reset) {
    if (g->scx == 8 && g->scy == 8 && g->scz == 4)
        return launch_advance<F, ORDER, true, 8, 8, 4, 1, true>(g, sp, in, out, ex, E, B, J, jpl,
                                                               status, s, sp0, reset, ws);
    return launch_advance<F, ORDER, true, 0, 0, 0, 1, true>(g, sp, in, out, ex, E, B, J, jpl,
                                                           status, s, sp0, reset, ws);
}

// kwb_particles_advance_species with the advance split in two kernels per
// species (csrc/push.cuh): ws[i] is a workspace store of in[i]'s geometry
// (same frames_per_sc; its front/back are not used).  PCS keeps the fused
// kernel (ws ignored).
extern "C" int kwb_particles_advance_split(const kwb_grid *g, int32_t n_species,
                                           const kwb_species *sp, const kwb_store *in,
                                           const kwb_store *out, const kwb_store *ws,
                                           const kwb_exchange *ex, void *const E[3],
                                           void *const B[3], void *const J[3],
                                           void *const *j_planes, int shape_order,
                                           int32_t *status, kwb_stream_t stream) {
    if (shape_order == 3 || !ws)
        return kwb_particles_advance_species(g, n_species, sp, in, out, ex, E, B, J, j_planes,
                                             shape_order, status, stream);
    int rc = check_grid(g);
    if (rc) return rc;
    if (n_species < 1 || n_species > kMaxSpecies || !sp || !in || !out || !ex || !ex->count ||
        !status || !E || !B || !J) {
        kwb_set_error("advance_split: NULL argument or bad species count");
        return KWB_EINVAL;
    }
    if (shape_order != 1 && shape_order != 2) {
        kwb_set_error("shape_order must be 1 (CIC), 2 (TSC) or 3 (PCS), got %d", shape_order);
        return KWB_EINVAL;
    }
    for (int i = 0; i < n_species; ++i) {
        if ((rc = check_store(in + i, "input")) || (rc = check_store(out + i, "output")) ||
            (rc = check_store(ws + i, "workspace")))
            return rc;
        if (out[i].frames_per_sc != in[i].frames_per_sc ||
            ws[i].frames_per_sc != in[i].frames_per_sc) {
            kwb_set_error("advance_split: input, output and workspace differ in frames_per_sc");
            return KWB_EINVAL;
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    for (int i = 0; i < n_species; ++i) {
        int32_t *st = status + i * KWB_STATUS_WORDS;
        const bool f32 = g->dtype == KWB_F32;
        rc = shape_order == 1
                 ? (f32 ? split_one<float, 1>(g, sp + i, in + i, out + i, ws + i, ex, E, B, J,
                                              j_planes, st, s, i, i == 0)
                        : split_one<double, 1>(g, sp + i, in + i, out + i, ws + i, ex, E, B, J,
                                               j_planes, st, s, i, i == 0))
                 : (f32 ? split_one<float, 2>(g, sp + i, in + i, out + i, ws + i, ex, E, B, J,
                                              j_planes, st, s, i, i == 0)
                        : split_one<double, 2>(g, sp + i, in + i, out + i, ws + i, ex, E, B, J,
                                               j_planes, st, s, i, i == 0));
        if (rc) return rc;
    }
    return KWB_OK;
}

static int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

static int col_blocks(const kwb_grid *g) {
    const int64_t ncol = (int64_t)g->gx * g->gy * g->gz * g->scx * g->scy * g->scz;
    const int64_t need = (ncol + 255) / 256, cap = (int64_t)sm_count() * 16;
    return (int)(need < cap ? (need > 0 ? need : 1) : cap);
}

extern "C" int kwb_particles_shift(const kwb_grid *g, const kwb_store *out,
                                   const kwb_exchange *ex, int32_t *status,
                                   kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(out, "output"))) return rc;
    if (!ex || !ex->count || !status) {
        kwb_set_error("shift: NULL argument");
        return KWB_EINVAL;
    }
    return shift_all(g, 1, out, ex, status, stream);
}

// The shift of every species after kwb_particles_advance_species.
extern "C" int kwb_particles_shift_species(const kwb_grid *g, int32_t n_species,
                                           const kwb_store *out, const kwb_exchange *ex,
                                           int32_t *status, kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if (n_species < 1 || n_species > kMaxSpecies || !out || !ex || !ex->count || !status) {
        kwb_set_error("shift_species: NULL argument or 1..%d species", kMaxSpecies);
        return KWB_EINVAL;
    }
    for (int i = 0; i < n_species; ++i)
        if ((rc = check_store(out + i, "output"))) return rc;
    return shift_all(g, n_species, out, ex, status, stream);
}

static int store_load(const kwb_grid *g, const kwb_store *st, int64_t n, const int64_t *n_dev,
                      const int32_t *cx, const int32_t *cy, const int32_t *cz,
                      void *const f7[7], int32_t *status, kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(st, "target"))) return rc;
    if (!status || (n > 0 && (!cx || !cy || !cz || !f7))) {
        kwb_set_error("store_load: NULL argument");
        return KWB_EINVAL;
    }
    if (n <= 0) return KWB_OK;
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t need = (n + 255) / 256, cap = (int64_t)sm_count() * 16;
    const int blocks = (int)(need < cap ? need : cap);
    if (g->dtype == KWB_F32) {
        const float *const *f = (const float *const *)f7;
        load_kernel<float><<<blocks, 256, 0, s>>>(geo, store_of<float>(*st), n, n_dev, cx, cy, cz,
                                                  f[0], f[1], f[2], f[3], f[4], f[5], f[6], status);
    } else {
        const double *const *f = (const double *const *)f7;
        load_kernel<double><<<blocks, 256, 0, s>>>(geo, store_of<double>(*st), n, n_dev, cx, cy, cz,
                                                   f[0], f[1], f[2], f[3], f[4], f[5], f[6], status);
    }
    return kwb_check_launch("load_kernel");
}

extern "C" int kwb_store_load(const kwb_grid *g, const kwb_store *st, int64_t n,
                              const int32_t *cx, const int32_t *cy, const int32_t *cz,
                              void *const f7[7], int32_t *status, kwb_stream_t stream) {
    return store_load(g, st, n, nullptr, cx, cy, cz, f7, status, stream);
}

extern "C" int kwb_store_load_counted(const kwb_grid *g, const kwb_store *st, const int64_t *n_dev,
                                      int64_t capacity, const int32_t *cx, const int32_t *cy,
                                      const int32_t *cz, void *const f7[7], int32_t *status,
                                      kwb_stream_t stream) {
    if (!n_dev) {
        kwb_set_error("store_load_counted: NULL count");
        return KWB_EINVAL;
    }
    return store_load(g, st, capacity, n_dev, cx, cy, cz, f7, status, stream);
}

static int store_export(const kwb_grid *g, const kwb_store *st, int64_t col_begin,
                        int64_t col_end, const int64_t *cell_start, int clear, int32_t *cx,
                        int32_t *cy, int32_t *cz, void *const f7[7], int64_t capacity,
                        int64_t *count_out, int32_t *status, kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(st, "source"))) return rc;
    const int64_t ncol = (int64_t)g->gx * g->gy * g->gz * g->scx * g->scy * g->scz;
    if (col_begin < 0 || col_end > ncol || col_begin > col_end) {
        kwb_set_error("store_export: column range [%lld, %lld) outside [0, %lld)",
                      (long long)col_begin, (long long)col_end, (long long)ncol);
        return KWB_EINVAL;
    }
    if (!cell_start || !cx || !cy || !cz || !f7 ||
        (capacity >= 0 && (!count_out || !status))) {
        kwb_set_error("store_export: NULL argument");
        return KWB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (col_begin == col_end) {
        if (capacity >= 0) return cudaMemsetAsync(count_out, 0, sizeof(int64_t), s) == cudaSuccess
                                      ? KWB_OK : kwb_check_launch("store_export memset");
        return KWB_OK;
    }
    Geo geo = geo_of(*g);
    const int V = g->scx * g->scy * g->scz;
    if (capacity < 0 && col_begin % V == 0 && col_end % V == 0) {
        // whole super cells: shared-memory staged, coalesced stores
        const int64_t nsc = (col_end - col_begin) / V;
        const int chunk = g->dtype == KWB_F32 ? 8192 : 4096;
        const size_t smem = (size_t)chunk * (g->dtype == KWB_F32 ? 4 : 8);
        const int th = block_threads(g);
        if (g->dtype == KWB_F32) {
            float *const *f = (float *const *)f7;
            export_sc_kernel<float><<<(unsigned)nsc, th, smem, s>>>(
                geo, store_of<float>(*st), col_begin, cell_start, clear, cx, cy, cz, f[0], f[1],
                f[2], f[3], f[4], f[5], f[6], chunk);
        } else {
            double *const *f = (double *const *)f7;
            export_sc_kernel<double><<<(unsigned)nsc, th, smem, s>>>(
                geo, store_of<double>(*st), col_begin, cell_start, clear, cx, cy, cz, f[0], f[1],
                f[2], f[3], f[4], f[5], f[6], chunk);
        }
        return kwb_check_launch("export_sc_kernel");
    }
    const int64_t need = (col_end - col_begin + 255) / 256, cap = (int64_t)sm_count() * 16;
    const int blocks = (int)(need < cap ? need : cap);
    if (g->dtype == KWB_F32) {
        float *const *f = (float *const *)f7;
        export_kernel<float><<<blocks, 256, 0, s>>>(geo, store_of<float>(*st), col_begin, col_end,
                                                    cell_start, clear, cx, cy, cz, f[0], f[1], f[2],
                                                    f[3], f[4], f[5], f[6], capacity, count_out,
                                                    status);
    } else {
        double *const *f = (double *const *)f7;
        export_kernel<double><<<blocks, 256, 0, s>>>(geo, store_of<double>(*st), col_begin, col_end,
                                                     cell_start, clear, cx, cy, cz, f[0], f[1], f[2],
                                                     f[3], f[4], f[5], f[6], capacity, count_out,
                                                     status);
    }
    return kwb_check_launch("export_kernel");
}

extern "C" int kwb_store_export(const kwb_grid *g, const kwb_store *st, int64_t col_begin,
                                int64_t col_end, const int64_t *cell_start, int clear,
                                int32_t *cx, int32_t *cy, int32_t *cz, void *const f7[7],
                                kwb_stream_t stream) {
    return store_export(g, st, col_begin, col_end, cell_start, clear, cx, cy, cz, f7, -1, nullptr,
                        nullptr, stream);
}

extern "C" int kwb_store_extract(const kwb_grid *g, const kwb_store *st, int64_t col_begin,
                                 int64_t col_end, const int64_t *cell_start, int64_t capacity,
                                 int32_t *cx, int32_t *cy, int32_t *cz, void *const f7[7],
                                 int64_t *count_out, int32_t *status, kwb_stream_t stream) {
    if (capacity < 0) {
        kwb_set_error("store_extract: negative capacity");
        return KWB_EINVAL;
    }
    return store_export(g, st, col_begin, col_end, cell_start, 1, cx, cy, cz, f7, capacity,
                        count_out, status, stream);
}

extern "C" int kwb_store_repack(const kwb_grid *g, const kwb_store *src, const kwb_store *dst,
                                kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(src, "source")) || (rc = check_store(dst, "target"))) return rc;
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    if (g->dtype == KWB_F32)
        repack_kernel<float><<<col_blocks(g), 256, 0, s>>>(geo, store_of<float>(*src), store_of<float>(*dst));
    else
        repack_kernel<double><<<col_blocks(g), 256, 0, s>>>(geo, store_of<double>(*src), store_of<double>(*dst));
    return kwb_check_launch("repack_kernel");
}

// CIC/TSC charge density with the current deposit's strategy: a thread owns
// a cell, so every particle it reads deposits into the same 3x3x3 stencil
// around that cell -- 27 float64 register accumulators, reduced into a
// shared (scx+2)(scy+2)(scz+2) tile in 27 barrier-separated conflict-free
// sweeps, the tile flushed with one global red.add per entry.  Same terms
// as rho_kernel (pic/kernels.py:291-326), summed in a different order
// (float64; the validation compares rho within tolerance).  The per-particle
// atomic version costs ~27 random float64 atomics per particle.
template <typename F, int ORDER>
__global__ void __launch_bounds__(256) rho_reg_kernel(Geo g, StoreT<F> st, double q_inv_vol,
                                                      double *__restrict__ rho) {
    static_assert(ORDER == 1 || ORDER == 2, "3-point stencils only");
    constexpr int H = Shape<ORDER>::H;
    __shared__ double tile[(16 + 2) * (16 + 2) * (16 + 2)];
    const int V = g.scx * g.scy * g.scz;
    const int tx = g.scx + 2, ty = g.scy + 2, tz = g.scz + 2, T = tx * ty * tz;
    const int s = blockIdx.x, c = threadIdx.x;
    const bool owner = c < V;
    const int bx = s % g.gx, by = (s / g.gx) % g.gy, bz = s / (g.gx * g.gy);
    const int lx = c % g.scx, ly = (c / g.scx) % g.scy, lz = c / (g.scx * g.scy);
    for (int i = c; i < T; i += blockDim.x) tile[i] = 0.0;
    double acc[3][3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int d = 0; d < 3; ++d) acc[a][b][d] = 0.0;
    if (owner) {
        for_column(st, s, c, V, [&](int64_t q) {
            const double qw = q_inv_vol * (double)st.w[q];
            double wx[3], wy[3], wz[3];
            if (ORDER == 2) {
                double o, l, r;
                o = (double)st.ox[q] - 0.5; l = 0.5 * ((0.5 - o) * (0.5 - o)); r = 0.5 * ((0.5 + o) * (0.5 + o));
                wx[0] = l; wx[1] = (1.0 - l) - r; wx[2] = r;
                o = (double)st.oy[q] - 0.5; l = 0.5 * ((0.5 - o) * (0.5 - o)); r = 0.5 * ((0.5 + o) * (0.5 + o));
                wy[0] = l; wy[1] = (1.0 - l) - r; wy[2] = r;
                o = (double)st.oz[q] - 0.5; l = 0.5 * ((0.5 - o) * (0.5 - o)); r = 0.5 * ((0.5 + o) * (0.5 + o));
                wz[0] = l; wz[1] = (1.0 - l) - r; wz[2] = r;
            } else {
                constexpr int NP = Shape<ORDER>::NP;
                F sx[NP], sy[NP], sz[NP];
                shape_into<F, ORDER>((double)st.ox[q], sx);
                shape_into<F, ORDER>((double)st.oy[q], sy);
                shape_into<F, ORDER>((double)st.oz[q], sz);
#pragma unroll
                for (int a = 0; a < 3; ++a) {   // CIC support: indices H-1 .. H+1
                    wx[a] = (double)sx[H - 1 + a];
                    wy[a] = (double)sy[H - 1 + a];
                    wz[a] = (double)sz[H - 1 + a];
                }
            }
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
#pragma unroll
                    for (int d = 0; d < 3; ++d) acc[a][b][d] += ((qw * wx[a]) * wy[b]) * wz[d];
        });
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                if (owner) tile[((lz + d) * ty + (ly + b)) * tx + (lx + a)] += acc[a][b][d];
                __syncthreads();
            }
    const int ox = bx * g.scx - 1, oy = by * g.scy - 1, oz = bz * g.scz - 1;
    for (int i = c; i < T; i += blockDim.x) {
        const double v = tile[i];
        if (v != 0.0) {
            const int a = i % tx, b = (i / tx) % ty, d = i / (tx * ty);
            atomicAdd(rho + fidx(pymod(ox + a, g.nx), pymod(oy + b, g.ny), pymod(oz + d, g.nz),
                                 g.nx, g.ny), v);
        }
    }
}

extern "C" int kwb_charge_density(const kwb_grid *g, const kwb_species *sp, const kwb_store *st,
                                  int shape_order, double *rho, kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(st, "source"))) return rc;
    if (!sp || !rho) {
        kwb_set_error("charge_density: NULL argument");
        return KWB_EINVAL;
    }
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    const int n_sc = g->gx * g->gy * g->gz, th = block_threads(g);
    // register/tile kernel for CIC/TSC when the super cell fits its static tile
    const bool reg = g->scx <= 16 && g->scy <= 16 && g->scz <= 16;
#define KWB_RHO(T, O) rho_kernel<T, O><<<n_sc, th, 0, s>>>(geo, store_of<T>(*st), sp->q_inv_vol, rho)
#define KWB_RHOR(T, O) rho_reg_kernel<T, O><<<n_sc, th, 0, s>>>(geo, store_of<T>(*st), sp->q_inv_vol, rho)
    if (g->dtype == KWB_F32) {
        if (shape_order == 1) { if (reg) KWB_RHOR(float, 1); else KWB_RHO(float, 1); }
        else if (shape_order == 2) { if (reg) KWB_RHOR(float, 2); else KWB_RHO(float, 2); }
        else if (shape_order == 3) KWB_RHO(float, 3);
        else { kwb_set_error("bad shape_order %d", shape_order); return KWB_EINVAL; }
    } else {
        if (shape_order == 1) { if (reg) KWB_RHOR(double, 1); else KWB_RHO(double, 1); }
        else if (shape_order == 2) { if (reg) KWB_RHOR(double, 2); else KWB_RHO(double, 2); }
        else if (shape_order == 3) KWB_RHO(double, 3);
        else { kwb_set_error("bad shape_order %d", shape_order); return KWB_EINVAL; }
    }
#undef KWB_RHO
#undef KWB_RHOR
    return kwb_check_launch("rho_kernel");
}

extern "C" int kwb_particle_moments(const kwb_grid *g, const kwb_species *sp, const kwb_store *st,
                                    double *out, kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(st, "source"))) return rc;
    if (!sp || !out) {
        kwb_set_error("particle_moments: NULL argument");
        return KWB_EINVAL;
    }
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    if (g->dtype == KWB_F32)
        moments_kernel<float><<<col_blocks(g), 256, 0, s>>>(geo, store_of<float>(*st), sp->charge, sp->mass, out);
    else
        moments_kernel<double><<<col_blocks(g), 256, 0, s>>>(geo, store_of<double>(*st), sp->charge, sp->mass, out);
    return kwb_check_launch("moments_kernel");
}
