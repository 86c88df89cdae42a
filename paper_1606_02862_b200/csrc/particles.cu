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
//  * Particles that cross a cell boundary are queued in shared memory and
//    deposited with the reference's exact per-contribution arithmetic by
//    all threads together (CAS into the J tile); PCS and float64 use this
//    path for every particle.
//  * The J tile (super cell + shape halo) is flushed once with coalesced
//    red.global.add; leavers of the super cell go to an exchange buffer.
#include <cstdio>

#include "common.cuh"

namespace kwb {

struct FieldPtrs {
    const void *E[3], *B[3];
    void *J[3];
};

constexpr int kMaxCells = 256;       // super-cell volume limit (= max CTA size)
constexpr int kQueue = 2 * kMaxCells; // crossing-particle queue capacity

// Yee staggers in cell units, pic/fields.py:24-31 (Ex Ey Ez Bx By Bz).
__host__ __device__ constexpr double stagger(int c, int a) {
    return (c == 0) ? (a == 0 ? 1.0 : 0.5)
         : (c == 1) ? (a == 1 ? 1.0 : 0.5)
         : (c == 2) ? (a == 2 ? 1.0 : 0.5)
         : (c == 3) ? (a == 0 ? 0.5 : 1.0)
         : (c == 4) ? (a == 1 ? 0.5 : 1.0)
                    : (a == 2 ? 0.5 : 1.0);
}

template <typename F, int ORDER>
struct AdvanceSmem {
    static size_t bytes(const Geo &g, int threads) {
        constexpr int H = Shape<ORDER>::H;
        size_t tv = (size_t)(g.scx + 2) * (g.scy + 2) * (g.scz + 2);
        size_t jv = (size_t)(g.scx + 2 * H) * (g.scy + 2 * H) * (g.scz + 2 * H);
        size_t b = (6 * tv + 3 * jv) * sizeof(F);
        b = (b + 15) & ~size_t(15);
        b += (size_t)kQueue * (7 * sizeof(F) + sizeof(int));  // crossing queue
        b += (size_t)threads * sizeof(int);                   // intra-super-cell arrivals
        return b;
    }
};

// Trilinear sample of one staged component (pic/kernels.py:26-47).  The tile
// origin is the super-cell origin minus one guard cell.
template <typename F, int C>
__device__ __forceinline__ double sample_tile(const F *__restrict__ T, double px, double py,
                                              double pz, int ox0, int oy0, int oz0, int tx,
                                              int ty) {
    const double ttx = px - stagger(C, 0), tty = py - stagger(C, 1), ttz = pz - stagger(C, 2);
    const double flx = floor(ttx), fly = floor(tty), flz = floor(ttz);
    const int ix = (int)flx, iy = (int)fly, iz = (int)flz;
    const double fx = ttx - (double)ix, fy = tty - (double)iy, fz = ttz - (double)iz;
    const F *r00 = T + (((iz - oz0) * ty) + (iy - oy0)) * tx + (ix - ox0);
    const F *r10 = r00 + tx;
    const F *r01 = r00 + tx * ty;
    const F *r11 = r01 + tx;
    const double gx = 1.0 - fx;
    const double c00 = (double)r00[0] * gx + (double)r00[1] * fx;
    const double c10 = (double)r10[0] * gx + (double)r10[1] * fx;
    const double c01 = (double)r01[0] * gx + (double)r01[1] * fx;
    const double c11 = (double)r11[0] * gx + (double)r11[1] * fx;
    return (c00 * (1.0 - fy) + c10 * fy) * (1.0 - fz) + (c01 * (1.0 - fy) + c11 * fy) * fz;
}

// Reference-exact deposit of one particle into the shared J tile
// (pic/kernels.py:173-248): double transverse factor and running sum,
// storage-type contributions.  Shared float atomics (CAS on sm_100a).
template <typename F, int ORDER>
__device__ void deposit_exact(F *__restrict__ jt, int jx, int jy, int JV, int lx, int ly, int lz,
                              int dcx, int dcy, int dcz, F oox, F ooy, F ooz, F nox, F noy,
                              F noz, F w, const double fac[3]) {
    constexpr int NP = Shape<ORDER>::NP, TOP = NP - 2;
    F s0x[NP], s0y[NP], s0z[NP], s1x[NP], s1y[NP], s1z[NP];
    shape_into<F, ORDER>((double)oox, s0x);
    shape_into<F, ORDER>((double)ooy, s0y);
    shape_into<F, ORDER>((double)ooz, s0z);
    shape_into<F, ORDER>((double)dcx + (double)nox, s1x);
    shape_into<F, ORDER>((double)dcy + (double)noy, s1y);
    shape_into<F, ORDER>((double)dcz + (double)noz, s1z);
    const double ww = (double)w;
    const int lox = 1 + min(dcx, 0), hix = TOP + max(dcx, 0), ex_ = min(hix, TOP);
    const int loy = 1 + min(dcy, 0), hiy = TOP + max(dcy, 0), ey_ = min(hiy, TOP);
    const int loz = 1 + min(dcz, 0), hiz = TOP + max(dcz, 0), ez_ = min(hiz, TOP);
    F *J0 = jt + ((lz * jy) + ly) * jx + lx;
    // x currents: tile[0][lx+ja][ly+j1][lz+j2]
#pragma unroll
    for (int j1 = 0; j1 < NP; ++j1) {
        if (j1 < loy || j1 > hiy) continue;
        const F dsy = s1y[j1] - s0y[j1];
#pragma unroll
        for (int j2 = 0; j2 < NP; ++j2) {
            if (j2 < loz || j2 > hiz) continue;
            const F dsz = s1z[j2] - s0z[j2];
            const double tr = (transverse<F>(s0y[j1], dsy, s0z[j2], dsz) * fac[0]) * ww;
            double acc = 0.0;
#pragma unroll
            for (int ja = 0; ja <= TOP; ++ja) {
                if (ja < lox || ja > ex_) continue;
                const F d = s1x[ja] - s0x[ja];
                acc += (double)d * tr;
                atomicAdd(J0 + (j2 * jy + j1) * jx + ja, (F)acc);
            }
        }
    }
    // y currents: tile[1][lx+j2][ly+ja][lz+j1]
    F *J1 = J0 + JV;
#pragma unroll
    for (int j1 = 0; j1 < NP; ++j1) {
        if (j1 < loz || j1 > hiz) continue;
        const F dsz = s1z[j1] - s0z[j1];
#pragma unroll
        for (int j2 = 0; j2 < NP; ++j2) {
            if (j2 < lox || j2 > hix) continue;
            const F dsx = s1x[j2] - s0x[j2];
            const double tr = (transverse<F>(s0z[j1], dsz, s0x[j2], dsx) * fac[1]) * ww;
            double acc = 0.0;
#pragma unroll
            for (int ja = 0; ja <= TOP; ++ja) {
                if (ja < loy || ja > ey_) continue;
                const F d = s1y[ja] - s0y[ja];
                acc += (double)d * tr;
                atomicAdd(J1 + (j1 * jy + ja) * jx + j2, (F)acc);
            }
        }
    }
    // z currents: tile[2][lx+j1][ly+j2][lz+ja]
    F *J2 = J0 + 2 * JV;
#pragma unroll
    for (int j1 = 0; j1 < NP; ++j1) {
        if (j1 < lox || j1 > hix) continue;
        const F dsx = s1x[j1] - s0x[j1];
#pragma unroll
        for (int j2 = 0; j2 < NP; ++j2) {
            if (j2 < loy || j2 > hiy) continue;
            const F dsy = s1y[j2] - s0y[j2];
            const double tr = (transverse<F>(s0x[j1], dsx, s0y[j2], dsy) * fac[2]) * ww;
            double acc = 0.0;
#pragma unroll
            for (int ja = 0; ja <= TOP; ++ja) {
                if (ja < loz || ja > ez_) continue;
                const F d = s1z[ja] - s0z[ja];
                acc += (double)d * tr;
                atomicAdd(J2 + (ja * jy + j2) * jx + j1, (F)acc);
            }
        }
    }
}

// Shape values at support indices 1..3 (the whole support of a CIC/TSC
// particle whose offset is in [0, 1]); identical arithmetic to shape_into.
template <int ORDER>
__device__ __forceinline__ void shape123(double x, float (&o)[3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double d = x - ((double)(i + 1 - 2) + 0.5);
        if (d < 0) d = -d;
        double v;
        if (ORDER == 2) {
            if (d < 0.5) v = 0.75 - d * d;
            else if (d < 1.5) { double e = 1.5 - d; v = (0.5 * e) * e; }
            else v = 0.0;
        } else {
            v = (d < 1.0) ? 1.0 - d : 0.0;
        }
        o[i] = (float)v;
    }
}

// Register accumulation of a particle that stays in its cell (dc = 0):
// J_a(along ja, transverse j1, j2) += P_ja * fw * T(j1, j2), ja in {1, 2}
// (the closing ja = 3 entry is a rounding residue of sum(s1) - sum(s0) and
// is dropped), T = (s0 + ds/2)_1 s0_2 + (s0/2 + ds/3)_1 ds_2.  fp32 with
// FMA: J is compared within tolerance, never bitwise (atomic order).
struct RegAcc {
    float a[3][2][3][3];  // [component][ja-1][j1-1][j2-1]
};

template <int ORDER>
__device__ __forceinline__ void deposit_stay(RegAcc &R, float oox, float ooy, float ooz,
                                             float nox, float noy, float noz, float fwx,
                                             float fwy, float fwz) {
    float s0[3][3], ds[3][3];
    {
        float s1[3];
        shape123<ORDER>((double)oox, s0[0]);
        shape123<ORDER>((double)nox, s1);
#pragma unroll
        for (int i = 0; i < 3; ++i) ds[0][i] = s1[i] - s0[0][i];
        shape123<ORDER>((double)ooy, s0[1]);
        shape123<ORDER>((double)noy, s1);
#pragma unroll
        for (int i = 0; i < 3; ++i) ds[1][i] = s1[i] - s0[1][i];
        shape123<ORDER>((double)ooz, s0[2]);
        shape123<ORDER>((double)noz, s1);
#pragma unroll
        for (int i = 0; i < 3; ++i) ds[2][i] = s1[i] - s0[2][i];
    }
    const float fw[3] = {fwx, fwy, fwz};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int a1 = (c + 1) % 3, a2 = (c + 2) % 3;  // transverse axes (x: y,z; y: z,x; z: x,y)
        const float p1 = ds[c][0], p2 = __fadd_rn(ds[c][0], ds[c][1]);
#pragma unroll
        for (int j1 = 0; j1 < 3; ++j1) {
            const float u = __fmul_rn(fw[c], __fmaf_rn(0.5f, ds[a1][j1], s0[a1][j1]));
            const float v = __fmul_rn(fw[c], __fmaf_rn(1.0f / 3.0f, ds[a1][j1], 0.5f * s0[a1][j1]));
#pragma unroll
            for (int j2 = 0; j2 < 3; ++j2) {
                const float T = __fmaf_rn(u, s0[a2][j2], __fmul_rn(v, ds[a2][j2]));
                R.a[c][0][j1][j2] = __fmaf_rn(p1, T, R.a[c][0][j1][j2]);
                R.a[c][1][j1][j2] = __fmaf_rn(p2, T, R.a[c][1][j1][j2]);
            }
        }
    }
}

// Tile offsets of accumulator (c, ja, j1, j2) relative to the owner cell.
__device__ __forceinline__ int regacc_offset(int c, int ja, int j1, int j2, int jx, int jy) {
    int ox, oy, oz;
    if (c == 0) { ox = ja; oy = j1; oz = j2; }
    else if (c == 1) { ox = j2; oy = ja; oz = j1; }
    else { ox = j1; oy = j2; oz = ja; }
    return (oz * jy + oy) * jx + ox;
}

template <typename F, int ORDER, bool REGACC>
__global__ void __launch_bounds__(kMaxCells)
advance_kernel(Geo g, kwb_species sp, StoreT<F> in, StoreT<F> out, ExchT<F> ex, FieldPtrs fp,
               int32_t *__restrict__ status) {
    constexpr int H = Shape<ORDER>::H;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_qcount, s_nmax, s_maxcol;

    const int V = g.scx * g.scy * g.scz;
    const int K = in.frames;
    const int t = threadIdx.x;
    const bool owner = t < V;
    const int sc = blockIdx.x;
    const int bx = sc % g.gx, by = (sc / g.gx) % g.gy, bz = sc / (g.gx * g.gy);
    const int orgx = bx * g.scx, orgy = by * g.scy, orgz = bz * g.scz;
    const int lx = t % g.scx, ly = (t / g.scx) % g.scy, lz = t / (g.scx * g.scy);

    const int tx = g.scx + 2, ty = g.scy + 2, tz = g.scz + 2, TV = tx * ty * tz;
    const int jx = g.scx + 2 * H, jy = g.scy + 2 * H, jz = g.scz + 2 * H, JV = jx * jy * jz;
    F *eb = reinterpret_cast<F *>(smem_raw);
    F *jt = eb + 6 * TV;
    size_t off = ((size_t)(6 * TV + 3 * JV) * sizeof(F) + 15) & ~size_t(15);
    F *q_f = reinterpret_cast<F *>(smem_raw + off);           // [7][kQueue]
    int *q_info = reinterpret_cast<int *>(q_f + 7 * kQueue);  // [kQueue]
    int *arr = q_info + kQueue;                               // [blockDim]

    // ---- stage E/B (+1 guard cell, periodic), clear J tile and counters --
    for (int i = t; i < 6 * TV; i += blockDim.x) {
        const int c = i / TV, r = i - c * TV;
        const int a = r % tx, b = (r / tx) % ty, d = r / (tx * ty);
        const int gi = pymod(orgx - 1 + a, g.nx), gj = pymod(orgy - 1 + b, g.ny),
                  gk = pymod(orgz - 1 + d, g.nz);
        const F *src = (const F *)(c < 3 ? fp.E[c] : fp.B[c - 3]);
        eb[i] = src[fidx(gi, gj, gk, g.nx, g.ny)];
    }
    for (int i = t; i < 3 * JV; i += blockDim.x) jt[i] = F(0);
    arr[t] = 0;
    if (t == 0) { s_qcount = 0; s_nmax = 0; s_maxcol = 0; }

    const int64_t col = (int64_t)sc * V + t;
    const int front_in = owner ? in.front[col] : 0;
    const int back_in = owner ? in.back[col] : 0;
    const int n_t = front_in + back_in;
    __syncthreads();
    atomicMax(&s_nmax, n_t);
    __syncthreads();
    const int n_max = s_nmax;

    RegAcc R;
    if (REGACC) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
#pragma unroll
                    for (int d = 0; d < 3; ++d) R.a[c][a][b][d] = 0.f;
    }
    const double qm = sp.qm_half_dt;
    const int lane = t & 31;
    const int cx = orgx + lx, cy = orgy + ly, cz = orgz + lz;
    int fo = 0;      // stayers written to the front of this column
    int n_err = 0;

    for (int i = 0; i < n_max; ++i) {
        bool active = owner && i < n_t;
        bool queue = false, leave = false, mover = false, stay = false;
        F ox = 0, oy = 0, oz = 0, nox = 0, noy = 0, noz = 0, nux = 0, nuy = 0, nuz = 0, w = 0;
        int dcx = 0, dcy = 0, dcz = 0, ncx = 0, ncy = 0, ncz = 0, dest = 0, nlc = 0;
        if (active) {
            const int k = i < front_in ? i : K - back_in + (i - front_in);
            const int64_t q = ((int64_t)sc * K + k) * V + t;
            ox = in.ox[q]; oy = in.oy[q]; oz = in.oz[q];
            const F ux = in.ux[q], uy = in.uy[q], uz = in.uz[q];
            w = in.w[q];

            // -- gather (pic/kernels.py:53-77): f64 compute, F store --------
            const double px = (double)cx + (double)ox;
            const double py = (double)cy + (double)oy;
            const double pz = (double)cz + (double)oz;
            const F e0 = (F)sample_tile<F, 0>(eb + 0 * TV, px, py, pz, orgx - 1, orgy - 1, orgz - 1, tx, ty);
            const F e1 = (F)sample_tile<F, 1>(eb + 1 * TV, px, py, pz, orgx - 1, orgy - 1, orgz - 1, tx, ty);
            const F e2 = (F)sample_tile<F, 2>(eb + 2 * TV, px, py, pz, orgx - 1, orgy - 1, orgz - 1, tx, ty);
            const F b0 = (F)sample_tile<F, 3>(eb + 3 * TV, px, py, pz, orgx - 1, orgy - 1, orgz - 1, tx, ty);
            const F b1 = (F)sample_tile<F, 4>(eb + 4 * TV, px, py, pz, orgx - 1, orgy - 1, orgz - 1, tx, ty);
            const F b2 = (F)sample_tile<F, 5>(eb + 5 * TV, px, py, pz, orgx - 1, orgy - 1, orgz - 1, tx, ty);

            // -- Boris push (pic/kernels.py:80-104), all in double ---------
            const double umx = (double)ux + qm * (double)e0;
            const double umy = (double)uy + qm * (double)e1;
            const double umz = (double)uz + qm * (double)e2;
            const double gm = sqrt(((1.0 + umx * umx) + umy * umy) + umz * umz);
            const double ttx = (qm * (double)b0) / gm;
            const double tty = (qm * (double)b1) / gm;
            const double ttz = (qm * (double)b2) / gm;
            const double tsq = (ttx * ttx + tty * tty) + ttz * ttz;
            const double ssx = (2.0 * ttx) / (1.0 + tsq);
            const double ssy = (2.0 * tty) / (1.0 + tsq);
            const double ssz = (2.0 * ttz) / (1.0 + tsq);
            const double upx = umx + (umy * ttz - umz * tty);
            const double upy = umy + (umz * ttx - umx * ttz);
            const double upz = umz + (umx * tty - umy * ttx);
            nux = (F)((umx + (upy * ssz - upz * ssy)) + qm * (double)e0);
            nuy = (F)((umy + (upz * ssx - upx * ssz)) + qm * (double)e1);
            nuz = (F)((umz + (upx * ssy - upy * ssx)) + qm * (double)e2);

            // -- move (pic/kernels.py:107-135): gamma from F squares -------
            const F sxx = nux * nux, syy = nuy * nuy, szz = nuz * nuz;
            const double gv = sqrt(((1.0 + (double)sxx) + (double)syy) + (double)szz);
            const double mpx = (double)ox + ((double)nux / gv) * sp.dt_d[0];
            const double mpy = (double)oy + ((double)nuy / gv) * sp.dt_d[1];
            const double mpz = (double)oz + ((double)nuz / gv) * sp.dt_d[2];
            const int dxi = (int)floor(mpx), dyi = (int)floor(mpy), dzi = (int)floor(mpz);
            nox = (F)(mpx - (double)dxi);
            noy = (F)(mpy - (double)dyi);
            noz = (F)(mpz - (double)dzi);
            ncx = pymod(cx + dxi, g.nx);
            ncy = pymod(cy + dyi, g.ny);
            ncz = pymod(cz + dzi, g.nz);

            // -- deposit dispatch (pic/kernels.py:173-191) ------------------
            dcx = ncx - cx; dcy = ncy - cy; dcz = ncz - cz;
            if (dcx > 1) dcx -= g.nx; else if (dcx < -1) dcx += g.nx;
            if (dcy > 1) dcy -= g.ny; else if (dcy < -1) dcy += g.ny;
            if (dcz > 1) dcz -= g.nz; else if (dcz < -1) dcz += g.nz;
            if (dcx > 1 || dcx < -1 || dcy > 1 || dcy < -1 || dcz > 1 || dcz < -1) {
                ++n_err;
            } else if (REGACC && dcx == 0 && dcy == 0 && dcz == 0) {
                const double ww = (double)w;
                deposit_stay<ORDER>(R, (float)ox, (float)oy, (float)oz, (float)nox, (float)noy,
                                    (float)noz, (float)(sp.fac[0] * ww), (float)(sp.fac[1] * ww),
                                    (float)(sp.fac[2] * ww));
            } else {
                queue = true;
            }

            // -- membership (pic/particles.py:226-228) ----------------------
            dest = (ncx / g.scx) + g.gx * ((ncy / g.scy) + g.gy * (ncz / g.scz));
            if (dest == sc) {
                nlc = (ncx - orgx) + g.scx * ((ncy - orgy) + g.scy * (ncz - orgz));
                if (nlc == t) stay = true; else mover = true;
            } else {
                leave = true;
            }
        }

        // ---- enqueue crossing particles (warp-aggregated slot claim) ------
        {
            const unsigned qm_ = __ballot_sync(0xffffffffu, queue);
            if (qm_) {
                int base = 0;
                const int leader = __ffs(qm_) - 1;
                if (lane == leader) base = atomicAdd(&s_qcount, __popc(qm_));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (queue) {
                    const int j = base + __popc(qm_ & ((1u << lane) - 1u));
                    q_f[0 * kQueue + j] = ox; q_f[1 * kQueue + j] = oy; q_f[2 * kQueue + j] = oz;
                    q_f[3 * kQueue + j] = nox; q_f[4 * kQueue + j] = noy; q_f[5 * kQueue + j] = noz;
                    q_f[6 * kQueue + j] = w;
                    q_info[j] = lx | (ly << 8) | (lz << 16) | ((dcx + 1) << 24) | ((dcy + 1) << 26) |
                                ((dcz + 1) << 28);
                }
            }
        }
        // ---- write the particle to its column / exchange ----------------
        if (stay) {
            const int64_t o = ((int64_t)sc * K + fo) * V + t;
            ++fo;
            out.ox[o] = nox; out.oy[o] = noy; out.oz[o] = noz;
            out.ux[o] = nux; out.uy[o] = nuy; out.uz[o] = nuz;
            out.w[o] = w;
        } else if (mover) {
            const int slot = atomicAdd(&arr[nlc], 1);
            const int64_t o = ((int64_t)sc * K + (K - 1 - slot)) * V + nlc;
            if (slot < K) {
                out.ox[o] = nox; out.oy[o] = noy; out.oz[o] = noz;
                out.ux[o] = nux; out.uy[o] = nuy; out.uz[o] = nuz;
                out.w[o] = w;
            }
        }
        {
            const unsigned lm = __ballot_sync(0xffffffffu, leave);
            if (lm) {
                int basek = 0;
                const int leader = __ffs(lm) - 1;
                if (lane == leader) basek = atomicAdd(ex.count, __popc(lm));
                basek = __shfl_sync(0xffffffffu, basek, leader);
                if (leave) {
                    const int k = basek + __popc(lm & ((1u << lane) - 1u));
                    if (k < ex.capacity) {
                        ex.ox[k] = nox; ex.oy[k] = noy; ex.oz[k] = noz;
                        ex.ux[k] = nux; ex.uy[k] = nuy; ex.uz[k] = nuz;
                        ex.w[k] = w;
                        ex.cx[k] = ncx; ex.cy[k] = ncy; ex.cz[k] = ncz;
                        ex.dest[k] = dest;
                    } else {
                        atomicAdd(&status[KWB_ST_EXCH_OVERFLOW], 1);
                    }
                }
            }
        }
        __syncthreads();
        // ---- drain the crossing queue when another round could overflow it
        const int qn = s_qcount;
        if (qn > kQueue - (int)blockDim.x || (i == n_max - 1 && qn > 0)) {
            for (int j = t; j < qn; j += blockDim.x) {
                const int info = q_info[j];
                deposit_exact<F, ORDER>(jt, jx, jy, JV, info & 255, (info >> 8) & 255,
                                        (info >> 16) & 255, ((info >> 24) & 3) - 1,
                                        ((info >> 26) & 3) - 1, ((info >> 28) & 3) - 1,
                                        q_f[0 * kQueue + j], q_f[1 * kQueue + j], q_f[2 * kQueue + j],
                                        q_f[3 * kQueue + j], q_f[4 * kQueue + j], q_f[5 * kQueue + j],
                                        q_f[6 * kQueue + j], sp.fac);
            }
            __syncthreads();
            if (t == 0) s_qcount = 0;
            __syncthreads();
        }
    }
    if (n_err) atomicAdd(&status[KWB_ST_MOVE_ERRORS], n_err);

    // ---- reduce the register accumulators into the J tile ----------------
    // Sweep s adds accumulator s of every cell: targets cell + offset(s) are
    // distinct across threads, so plain read-modify-writes are race free;
    // the barrier orders consecutive sweeps.
    if (REGACC) {
        F *Jb = jt + ((lz * jy) + ly) * jx + lx;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        if (owner) {
                            F *p = Jb + c * JV + regacc_offset(c, a + 1, b + 1, d + 1, jx, jy);
                            *p = *p + (F)R.a[c][a][b][d];
                        }
                        __syncthreads();
                    }
    } else {
        __syncthreads();
    }

    // ---- flush the J tile: one red.global.add per non-zero entry ---------
    for (int i = t; i < 3 * JV; i += blockDim.x) {
        const F v = jt[i];
        if (v != F(0)) {
            const int c = i / JV, r = i - c * JV;
            const int a = r % jx, b = (r / jx) % jy, d = r / (jx * jy);
            const int gi = pymod(orgx - H + a, g.nx), gj = pymod(orgy - H + b, g.ny),
                      gk = pymod(orgz - H + d, g.nz);
            atomicAdd((F *)fp.J[c] + fidx(gi, gj, gk, g.nx, g.ny), v);
        }
    }
    if (owner) {
        const int nb = arr[t];
        out.front[col] = fo;
        out.back[col] = nb < K ? nb : K;
        if (fo + nb > K) atomicAdd(&status[KWB_ST_STORE_OVERFLOW], fo + nb - K);
        atomicMax(&s_maxcol, fo + nb);
    }
    __syncthreads();
    if (t == 0) atomicMax(&status[KWB_ST_MAX_COUNT], s_maxcol);
}

// Append leavers to the back of their new column (the cross-super-cell
// shift, pic/particles.py:316-345).  Slot claims are atomic per column.
template <typename F>
__global__ void shift_kernel(StoreT<F> out, ExchT<F> ex, Geo g, int32_t *__restrict__ status) {
    int n = *ex.count;
    if (n > ex.capacity) n = ex.capacity;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&status[KWB_ST_LEAVERS], n);
    const int V = g.scx * g.scy * g.scz, K = out.frames;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int d = ex.dest[i];
        const int bx = d % g.gx, by = (d / g.gx) % g.gy, bz = d / (g.gx * g.gy);
        const int c = (ex.cx[i] - bx * g.scx) +
                      g.scx * ((ex.cy[i] - by * g.scy) + g.scy * (ex.cz[i] - bz * g.scz));
        const int64_t colx = (int64_t)d * V + c;
        const int slot = atomicAdd(&out.back[colx], 1);
        const int fill = out.front[colx] + slot + 1;
        if (fill > K) {
            atomicSub(&out.back[colx], 1);
            atomicAdd(&status[KWB_ST_STORE_OVERFLOW], 1);
            continue;
        }
        atomicMax(&status[KWB_ST_MAX_COUNT], fill);
        const int64_t o = ((int64_t)d * K + (K - 1 - slot)) * V + c;
        out.ox[o] = ex.ox[i]; out.oy[o] = ex.oy[i]; out.oz[o] = ex.oz[i];
        out.ux[o] = ex.ux[i]; out.uy[o] = ex.uy[i]; out.uz[o] = ex.uz[i];
        out.w[o] = ex.w[i];
    }
}

// ---- store load / export / repack ---------------------------------------

template <typename F>
__global__ void load_kernel(Geo g, StoreT<F> st, int64_t n, const int32_t *__restrict__ cx,
                            const int32_t *__restrict__ cy, const int32_t *__restrict__ cz,
                            const F *__restrict__ ox, const F *__restrict__ oy,
                            const F *__restrict__ oz, const F *__restrict__ ux,
                            const F *__restrict__ uy, const F *__restrict__ uz,
                            const F *__restrict__ w, int32_t *__restrict__ status) {
    const int V = g.scx * g.scy * g.scz, K = st.frames;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
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
__global__ void export_kernel(Geo g, StoreT<F> st, const int64_t *__restrict__ cell_start,
                              int32_t *cx, int32_t *cy, int32_t *cz, F *ox, F *oy, F *oz, F *ux,
                              F *uy, F *uz, F *w) {
    const int V = g.scx * g.scy * g.scz, K = st.frames;
    const int64_t ncol = (int64_t)g.gx * g.gy * g.gz * V;
    for (int64_t colx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; colx < ncol;
         colx += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(colx / V), c = (int)(colx % V);
        const int bx = s % g.gx, by = (s / g.gx) % g.gy, bz = s / (g.gx * g.gy);
        const int x = bx * g.scx + c % g.scx, y = by * g.scy + (c / g.scx) % g.scy,
                  z = bz * g.scz + c / (g.scx * g.scy);
        const int f = st.front[colx], b = st.back[colx];
        int64_t o = cell_start[colx];
        for (int j = 0; j < f + b; ++j, ++o) {
            const int k = j < f ? j : K - b + (j - f);
            const int64_t q = ((int64_t)s * K + k) * V + c;
            cx[o] = x; cy[o] = y; cz[o] = z;
            ox[o] = st.ox[q]; oy[o] = st.oy[q]; oz[o] = st.oz[q];
            ux[o] = st.ux[q]; uy[o] = st.uy[q]; uz[o] = st.uz[q];
            w[o] = st.w[q];
        }
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

static int block_threads(const kwb_grid *g) {
    const int V = g->scx * g->scy * g->scz;
    return (V + 31) / 32 * 32;
}

template <typename F, int ORDER, bool REGACC>
static int launch_advance(const kwb_grid *g, const kwb_species *sp, const kwb_store *in,
                          const kwb_store *out, const kwb_exchange *ex, void *const E[3],
                          void *const B[3], void *const J[3], int32_t *status,
                          cudaStream_t stream) {
    Geo geo = geo_of(*g);
    const int threads = block_threads(g);
    size_t smem = AdvanceSmem<F, ORDER>::bytes(geo, threads);
    auto kern = advance_kernel<F, ORDER, REGACC>;
    if (smem > 227 * 1024) {
        kwb_set_error("super cell too large for the shared-memory tiles (%zu B)", smem);
        return KWB_EINVAL;
    }
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    FieldPtrs fp;
    for (int c = 0; c < 3; ++c) { fp.E[c] = E[c]; fp.B[c] = B[c]; fp.J[c] = J[c]; }
    if (cudaMemsetAsync(ex->count, 0, sizeof(int32_t), stream) != cudaSuccess)
        return kwb_check_launch("exchange counter reset");
    const int n_sc = g->gx * g->gy * g->gz;
    kern<<<n_sc, threads, smem, stream>>>(geo, *sp, store_of<F>(*in), store_of<F>(*out),
                                          exch_of<F>(*ex), fp, status);
    return kwb_check_launch("advance_kernel");
}

extern "C" int kwb_particles_advance(const kwb_grid *g, const kwb_species *sp,
                                     const kwb_store *in, const kwb_store *out,
                                     const kwb_exchange *ex, void *const E[3], void *const B[3],
                                     void *const J[3], int shape_order, int32_t *status,
                                     kwb_stream_t stream) {
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
    cudaStream_t s = (cudaStream_t)stream;
    if (g->dtype == KWB_F32) {
        switch (shape_order) {
            case 1: return launch_advance<float, 1, true>(g, sp, in, out, ex, E, B, J, status, s);
            case 2: return launch_advance<float, 2, true>(g, sp, in, out, ex, E, B, J, status, s);
            case 3: return launch_advance<float, 3, false>(g, sp, in, out, ex, E, B, J, status, s);
        }
    } else {
        switch (shape_order) {
            case 1: return launch_advance<double, 1, false>(g, sp, in, out, ex, E, B, J, status, s);
            case 2: return launch_advance<double, 2, false>(g, sp, in, out, ex, E, B, J, status, s);
            case 3: return launch_advance<double, 3, false>(g, sp, in, out, ex, E, B, J, status, s);
        }
    }
    kwb_set_error("shape_order must be 1 (CIC), 2 (TSC) or 3 (PCS), got %d", shape_order);
    return KWB_EINVAL;
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
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = sm_count() * 4;
    if (g->dtype == KWB_F32)
        shift_kernel<float><<<blocks, 256, 0, s>>>(store_of<float>(*out), exch_of<float>(*ex), geo, status);
    else
        shift_kernel<double><<<blocks, 256, 0, s>>>(store_of<double>(*out), exch_of<double>(*ex), geo, status);
    return kwb_check_launch("shift_kernel");
}

extern "C" int kwb_store_load(const kwb_grid *g, const kwb_store *st, int64_t n,
                              const int32_t *cx, const int32_t *cy, const int32_t *cz,
                              void *const f7[7], int32_t *status, kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(st, "target"))) return rc;
    if (!status || (n > 0 && (!cx || !cy || !cz || !f7))) {
        kwb_set_error("store_load: NULL argument");
        return KWB_EINVAL;
    }
    if (n == 0) return KWB_OK;
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t need = (n + 255) / 256, cap = (int64_t)sm_count() * 16;
    const int blocks = (int)(need < cap ? need : cap);
    if (g->dtype == KWB_F32) {
        const float *const *f = (const float *const *)f7;
        load_kernel<float><<<blocks, 256, 0, s>>>(geo, store_of<float>(*st), n, cx, cy, cz,
                                                  f[0], f[1], f[2], f[3], f[4], f[5], f[6], status);
    } else {
        const double *const *f = (const double *const *)f7;
        load_kernel<double><<<blocks, 256, 0, s>>>(geo, store_of<double>(*st), n, cx, cy, cz,
                                                   f[0], f[1], f[2], f[3], f[4], f[5], f[6], status);
    }
    return kwb_check_launch("load_kernel");
}

extern "C" int kwb_store_export(const kwb_grid *g, const kwb_store *st, const int64_t *cell_start,
                                int32_t *cx, int32_t *cy, int32_t *cz, void *const f7[7],
                                kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(st, "source"))) return rc;
    if (!cell_start || !cx || !cy || !cz || !f7) {
        kwb_set_error("store_export: NULL argument");
        return KWB_EINVAL;
    }
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    if (g->dtype == KWB_F32) {
        float *const *f = (float *const *)f7;
        export_kernel<float><<<col_blocks(g), 256, 0, s>>>(geo, store_of<float>(*st), cell_start, cx, cy, cz,
                                                           f[0], f[1], f[2], f[3], f[4], f[5], f[6]);
    } else {
        double *const *f = (double *const *)f7;
        export_kernel<double><<<col_blocks(g), 256, 0, s>>>(geo, store_of<double>(*st), cell_start, cx, cy, cz,
                                                            f[0], f[1], f[2], f[3], f[4], f[5], f[6]);
    }
    return kwb_check_launch("export_kernel");
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
#define KWB_RHO(T, O) rho_kernel<T, O><<<n_sc, th, 0, s>>>(geo, store_of<T>(*st), sp->q_inv_vol, rho)
    if (g->dtype == KWB_F32) {
        if (shape_order == 1) KWB_RHO(float, 1);
        else if (shape_order == 2) KWB_RHO(float, 2);
        else if (shape_order == 3) KWB_RHO(float, 3);
        else { kwb_set_error("bad shape_order %d", shape_order); return KWB_EINVAL; }
    } else {
        if (shape_order == 1) KWB_RHO(double, 1);
        else if (shape_order == 2) KWB_RHO(double, 2);
        else if (shape_order == 3) KWB_RHO(double, 3);
        else { kwb_set_error("bad shape_order %d", shape_order); return KWB_EINVAL; }
    }
#undef KWB_RHO
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
