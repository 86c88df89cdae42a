// Shared device helpers for libkwb200 (sm_100a).
//
// The whole library is compiled with --fmad=false: the reference kernels
// (Numba/LLVM, no fast-math) never contract a*b+c, so neither may we if the
// particle state is to stay bitwise equal.
#pragma once

#include <cuda.h>   // CUtensorMap (types only; the encoder comes from cudaGetDriverEntryPoint)
#include <cuda_runtime.h>
#include <cstdio>
#include <stdint.h>

#include "kwb200.h"

namespace kwb {

constexpr int kThreads = 256;  // one CTA per super cell, 8 warps

// ---- KWB_CHECKS: the bounds-checked debug build --------------------------
// (compute-sanitizer is not available on the GPU pool.)  Every shared- and
// global-memory index the kernels compute is checked against its array
// before the access; a failing check skips the access, counts into a
// per-module device counter and prints its first occurrence.  Read and reset
// through kwb_check_failures() (tests/conftest.py asserts 0 after every GPU
// test when the library was built with the checks).  Compiled out otherwise.
#ifdef KWB_CHECKS
static __device__ unsigned long long kwb_chk_count;
__device__ __forceinline__ bool kwb_chk(bool ok, const char *what, int line) {
    if (!ok && atomicAdd(&kwb_chk_count, 1ull) == 0ull)
        printf("KWB_CHECK failed: %s (line %d) block %d thread %d\n", what, line, blockIdx.x,
               threadIdx.x);
    return ok;
}
#define KWB_IN(cond) kwb::kwb_chk((cond), #cond, __LINE__)
#else
#define KWB_IN(cond) true
#endif

// Python floor-mod (non-negative for n > 0).
__host__ __device__ __forceinline__ int pymod(int a, int n) {
    int r = a % n;
    return r < 0 ? r + n : r;
}

// a / b correctly rounded from r = RN(1 / b) (one IEEE division): q0 =
// RN(a r) is within 1 ulp of a / b, the residual a - b q0 is exact with an
// FMA, and RN(q0 + r (a - b q0)) is the correctly rounded quotient
// (Markstein's theorem) -- so the push's and the move's three quotients by
// one divisor (gamma, 1 + t^2, gamma') cost one division each, and the Yee
// updates' quotients by the cell sizes none, bit for bit the reference's
// a / b (checked against IEEE division over 2^24 kernel-like pairs in the
// CPU suite, oracle orc_div_rcp_check).  An exact q0 is returned as is (the
// FMA would turn -0 into +0).  The theorem needs no overflow or subnormal
// intermediates: the operands are O(1) momenta, fields and cell sizes.
// Every divisor here is positive (gamma, 1 + t^2, cell sizes, 6), so the
// quotient has the numerator's sign -- zeros included, where the FMA alone
// would turn -0 / b into +0: the sign is copied from a (one LOP3 instead of
// a compare and two selects).
__device__ __forceinline__ double div_rcp(double a, double b, double r) {
    const double q0 = a * r;
    const double e = __fma_rn(-q0, b, a);
#ifdef KWB_DIV_SELECT
    return e == 0.0 ? q0 : __fma_rn(e, r, q0);   // e == 0: q0 exact, keeps -0 / b = -0
#else
    return copysign(__fma_rn(e, r, q0), a);
#endif
}

// Field index for the x-fastest layout: (k * ny + j) * nx + i.
__device__ __forceinline__ int64_t fidx(int i, int j, int k, int nx, int ny) {
    return ((int64_t)k * ny + j) * nx + i;
}

template <typename F>
struct StoreT {
    F *ox, *oy, *oz, *ux, *uy, *uz, *w;
    int32_t *front, *back;
    int32_t frames;
};

template <typename F>
__host__ inline StoreT<F> store_of(const kwb_store &s) {
    StoreT<F> t;
    t.ox = (F *)s.ox; t.oy = (F *)s.oy; t.oz = (F *)s.oz;
    t.ux = (F *)s.ux; t.uy = (F *)s.uy; t.uz = (F *)s.uz;
    t.w = (F *)s.w;
    t.front = s.front;
    t.back = s.back;
    t.frames = s.frames_per_sc;
    return t;
}

template <typename F>
struct ExchT {
    F *ox, *oy, *oz, *ux, *uy, *uz, *w;
    int32_t *cx, *cy, *cz, *dest, *count;
    int32_t capacity;
};

template <typename F>
__host__ inline ExchT<F> exch_of(const kwb_exchange &e) {
    ExchT<F> t;
    t.ox = (F *)e.ox; t.oy = (F *)e.oy; t.oz = (F *)e.oz;
    t.ux = (F *)e.ux; t.uy = (F *)e.uy; t.uz = (F *)e.uz;
    t.w = (F *)e.w;
    t.cx = e.cx; t.cy = e.cy; t.cz = e.cz; t.dest = e.dest; t.count = e.count;
    t.capacity = e.capacity;
    return t;
}

struct Geo {
    int nx, ny, nz, scx, scy, scz, gx, gy, gz;
    double dx, dy, dz, dt;
};

__host__ inline Geo geo_of(const kwb_grid &g) {
    Geo o;
    o.nx = g.nx; o.ny = g.ny; o.nz = g.nz;
    o.scx = g.scx; o.scy = g.scy; o.scz = g.scz;
    o.gx = g.gx; o.gy = g.gy; o.gz = g.gz;
    o.dx = g.dx; o.dy = g.dy; o.dz = g.dz; o.dt = g.dt;
    return o;
}

// Atomic max on a non-negative double via its bit pattern.
__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
    atomicMax((unsigned long long *)addr, (unsigned long long)__double_as_longlong(v));
}

// Shape orders: 1 CIC, 2 TSC (reference), 3 PCS.  NP = support array length,
// H = tile halo (and array centre offset).
template <int ORDER>
struct Shape {
    static constexpr int NP = (ORDER == 3) ? 7 : 5;
    static constexpr int H = (ORDER == 3) ? 3 : 2;
};

// pic/kernels.py:138-150 `_shape5_into` (TSC) and the CIC/PCS extension
// (SURVEY.md §8c): out[idx] = (F) W(|x - ((idx - H) + 0.5)|).
template <typename F, int ORDER>
__device__ __forceinline__ void shape_into(double x, F (&out)[Shape<ORDER>::NP]) {
    constexpr int NP = Shape<ORDER>::NP, H = Shape<ORDER>::H;
#pragma unroll
    for (int idx = 0; idx < NP; ++idx) {
        double d = x - ((double)(idx - H) + 0.5);
        if (d < 0) d = -d;
        double v;
        if (ORDER == 2) {
            if (d < 0.5) v = 0.75 - d * d;
            else if (d < 1.5) { double e = 1.5 - d; v = (0.5 * e) * e; }
            else v = 0.0;
        } else if (ORDER == 1) {
            v = (d < 1.0) ? 1.0 - d : 0.0;
        } else {
            if (d < 1.0) v = ((4.0 - (6.0 * d) * d) + ((3.0 * d) * d) * d) / 6.0;
            else if (d < 2.0) { double e = 2.0 - d; v = ((e * e) * e) / 6.0; }
            else v = 0.0;
        }
        out[idx] = (F)v;
    }
}

// Transverse factor, pic/kernels.py:215-218, evaluated left to right:
// ((F(a0*b0) + (0.5*da)*b0) + (0.5*a0)*db) + F(da*db)/3.0
template <typename F>
__device__ __forceinline__ double transverse(F a0, F da, F b0, F db) {
    F p00 = a0 * b0, pdd = da * db;
    return (((double)p00 + (0.5 * (double)da) * (double)b0) + (0.5 * (double)a0) * (double)db) +
           (double)pdd / 3.0;
}

}  // namespace kwb

// thread-local error text for kwb_last_error()
void kwb_set_error(const char *fmt, ...);
int kwb_check_launch(const char *what);
