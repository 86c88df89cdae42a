// Particle path of the PIC cycle on sm_100a: fused gather/push/move/deposit
// with in-kernel compaction, the super-cell shift, and store load/export.
//
// Reference: pic/kernels.py:26-250 (stage loops), :329-412 (kernel objects),
// kw/atomics.py:147-163 (deposit-halo merge), pic/particles.py:214-345
// (migration).  One CTA owns one super cell (the paper's "super cell is
// mapped to a block", §2.1), exactly as the reference's work
// division does, but all four particle stages run in ONE pass over the
// particle data:
//
//   * E/B of the super cell plus one guard cell are staged in shared memory
//     once per CTA (the gather support of a particle in cell c is c-1..c+1);
//   * the pre-move offset and cell never leave registers (the reference's
//     oo*/oc* scratch arrays are gone), nor do gathered E_p/B_p;
//   * current is accumulated in a shared-memory J tile covering the super
//     cell plus the shape halo (2 cells CIC/TSC, 3 PCS), flushed once to
//     global J with red.global.add (the reference merges the same tile with a
//     locked dense add);
//   * stayers are written densely (order-preserving block scan) into the
//     output store; leavers go to an exchange buffer (warp-aggregated slot
//     claim) which kwb_particles_shift appends to their new super cells.
#include <cstdio>

#include "common.cuh"

namespace kwb {

struct FieldPtrs {
    const void *E[3], *B[3];
    void *J[3];
};

// Yee staggers in cell units, pic/fields.py:24-31 (Ex Ey Ez Bx By Bz).
__constant__ double c_stagger[6][3] = {
    {1.0, 0.5, 0.5}, {0.5, 1.0, 0.5}, {0.5, 0.5, 1.0},
    {0.5, 1.0, 1.0}, {1.0, 0.5, 1.0}, {1.0, 1.0, 0.5},
};

template <typename F, int ORDER>
__host__ __device__ inline size_t advance_smem_bytes(const Geo &g) {
    constexpr int H = Shape<ORDER>::H;
    size_t tv = (size_t)(g.scx + 2) * (g.scy + 2) * (g.scz + 2);
    size_t jv = (size_t)(g.scx + 2 * H) * (g.scy + 2 * H) * (g.scz + 2 * H);
    return (6 * tv + 3 * jv) * sizeof(F);
}

// Trilinear sample of one staged component, pic/kernels.py:26-47; the tile
// origin is the super-cell origin minus one guard cell.
template <typename F>
__device__ __forceinline__ double sample_tile(const F *__restrict__ T, double px, double py,
                                              double pz, double sx, double sy, double sz,
                                              int ox0, int oy0, int oz0, int tx, int ty) {
    double ttx = px - sx, tty = py - sy, ttz = pz - sz;
    int ix = (int)floor(ttx), iy = (int)floor(tty), iz = (int)floor(ttz);
    double fx = ttx - (double)ix, fy = tty - (double)iy, fz = ttz - (double)iz;
    int a = ix - ox0, b = iy - oy0, c = iz - oz0;
    const F *r00 = T + ((c * ty) + b) * tx + a;  // (j0, k0)
    const F *r10 = r00 + tx;                     // (j1, k0)
    const F *r01 = r00 + tx * ty;                // (j0, k1)
    const F *r11 = r01 + tx;                     // (j1, k1)
    double c00 = (double)r00[0] * (1.0 - fx) + (double)r00[1] * fx;
    double c10 = (double)r10[0] * (1.0 - fx) + (double)r10[1] * fx;
    double c01 = (double)r01[0] * (1.0 - fx) + (double)r01[1] * fx;
    double c11 = (double)r11[0] * (1.0 - fx) + (double)r11[1] * fx;
    return (c00 * (1.0 - fy) + c10 * fy) * (1.0 - fz) + (c01 * (1.0 - fy) + c11 * fy) * fz;
}

template <typename F, int ORDER>
__global__ void __launch_bounds__(kThreads)
advance_kernel(Geo g, kwb_species sp, StoreT<F> in, StoreT<F> out, ExchT<F> ex, FieldPtrs fp,
               int32_t *__restrict__ status) {
    constexpr int NP = Shape<ORDER>::NP, H = Shape<ORDER>::H, TOP = NP - 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int warp_tot[kThreads / 32];

    const int sc = blockIdx.x;
    const int bx = sc % g.gx, by = (sc / g.gx) % g.gy, bz = sc / (g.gx * g.gy);
    const int orgx = bx * g.scx, orgy = by * g.scy, orgz = bz * g.scz;

    const int tx = g.scx + 2, ty = g.scy + 2, tz = g.scz + 2, TV = tx * ty * tz;
    const int jx = g.scx + 2 * H, jy = g.scy + 2 * H, jz = g.scz + 2 * H, JV = jx * jy * jz;
    F *eb = reinterpret_cast<F *>(smem_raw);
    F *jt = eb + 6 * TV;

    // ---- stage E/B (+1 guard cell, periodic) and clear the J tile -------
    for (int t = threadIdx.x; t < 6 * TV; t += kThreads) {
        int c = t / TV, r = t - c * TV;
        int a = r % tx, b = (r / tx) % ty, d = r / (tx * ty);
        int gi = pymod(orgx - 1 + a, g.nx), gj = pymod(orgy - 1 + b, g.ny),
            gk = pymod(orgz - 1 + d, g.nz);
        const F *src = (const F *)(c < 3 ? fp.E[c] : fp.B[c - 3]);
        eb[t] = src[fidx(gi, gj, gk, g.nx, g.ny)];
    }
    for (int t = threadIdx.x; t < 3 * JV; t += kThreads) jt[t] = F(0);
    __syncthreads();

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n = in.count[sc];
    const int64_t base_in = (int64_t)sc * in.slots;
    const int64_t base_out = (int64_t)sc * out.slots;
    const double qm = sp.qm_half_dt;
    int n_stay = 0;
    int n_err = 0;

    for (int c0 = 0; c0 < n; c0 += kThreads) {
        const int i = c0 + threadIdx.x;
        bool stay = false, leave = false;
        F nox = 0, noy = 0, noz = 0, nux = 0, nuy = 0, nuz = 0, w = 0;
        int ncx = 0, ncy = 0, ncz = 0, dest = 0;
        uint16_t nlc = 0;
        if (i < n) {
            const int64_t q = base_in + i;
            const int lc = in.cell[q];
            const int lx = lc % g.scx, ly = (lc / g.scx) % g.scy, lz = lc / (g.scx * g.scy);
            const int cx = orgx + lx, cy = orgy + ly, cz = orgz + lz;
            const F ox = in.ox[q], oy = in.oy[q], oz = in.oz[q];
            const F ux = in.ux[q], uy = in.uy[q], uz = in.uz[q];
            w = in.w[q];

            // -- gather (pic/kernels.py:53-77): f64 compute, F store --------
            const double px = (double)cx + (double)ox;
            const double py = (double)cy + (double)oy;
            const double pz = (double)cz + (double)oz;
            F e[3], b[3];
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                double v = sample_tile<F>(eb + c * TV, px, py, pz, c_stagger[c][0],
                                          c_stagger[c][1], c_stagger[c][2], orgx - 1, orgy - 1,
                                          orgz - 1, tx, ty);
                if (c < 3) e[c] = (F)v; else b[c - 3] = (F)v;
            }

            // -- Boris push (pic/kernels.py:80-104), all in double ---------
            const double umx = (double)ux + qm * (double)e[0];
            const double umy = (double)uy + qm * (double)e[1];
            const double umz = (double)uz + qm * (double)e[2];
            const double gm = sqrt(((1.0 + umx * umx) + umy * umy) + umz * umz);
            const double ttx = (qm * (double)b[0]) / gm;
            const double tty = (qm * (double)b[1]) / gm;
            const double ttz = (qm * (double)b[2]) / gm;
            const double tsq = (ttx * ttx + tty * tty) + ttz * ttz;
            const double ssx = (2.0 * ttx) / (1.0 + tsq);
            const double ssy = (2.0 * tty) / (1.0 + tsq);
            const double ssz = (2.0 * ttz) / (1.0 + tsq);
            const double upx = umx + (umy * ttz - umz * tty);
            const double upy = umy + (umz * ttx - umx * ttz);
            const double upz = umz + (umx * tty - umy * ttx);
            nux = (F)((umx + (upy * ssz - upz * ssy)) + qm * (double)e[0]);
            nuy = (F)((umy + (upz * ssx - upx * ssz)) + qm * (double)e[1]);
            nuz = (F)((umz + (upx * ssy - upy * ssx)) + qm * (double)e[2]);

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

            // -- Esirkepov deposit (pic/kernels.py:153-250) -----------------
            int dcx = ncx - cx, dcy = ncy - cy, dcz = ncz - cz;
            if (dcx > 1) dcx -= g.nx; else if (dcx < -1) dcx += g.nx;
            if (dcy > 1) dcy -= g.ny; else if (dcy < -1) dcy += g.ny;
            if (dcz > 1) dcz -= g.nz; else if (dcz < -1) dcz += g.nz;
            if (dcx > 1 || dcx < -1 || dcy > 1 || dcy < -1 || dcz > 1 || dcz < -1) {
                ++n_err;
            } else {
                F s0x[NP], s0y[NP], s0z[NP], s1x[NP], s1y[NP], s1z[NP];
                shape_into<F, ORDER>((double)ox, s0x);
                shape_into<F, ORDER>((double)oy, s0y);
                shape_into<F, ORDER>((double)oz, s0z);
                shape_into<F, ORDER>((double)dcx + (double)nox, s1x);
                shape_into<F, ORDER>((double)dcy + (double)noy, s1y);
                shape_into<F, ORDER>((double)dcz + (double)noz, s1z);
                const double ww = (double)w;
                const int lox = 1 + min(dcx, 0), hix = TOP + max(dcx, 0), ex_ = min(hix, TOP);
                const int loy = 1 + min(dcy, 0), hiy = TOP + max(dcy, 0), ey_ = min(hiy, TOP);
                const int loz = 1 + min(dcz, 0), hiz = TOP + max(dcz, 0), ez_ = min(hiz, TOP);
                // x currents: tile[0][lx+ja][ly+j1][lz+j2]
                F *J0 = jt + ((lz * jy) + ly) * jx + lx;
#pragma unroll
                for (int j1 = 0; j1 < NP; ++j1) {
                    if (j1 < loy || j1 > hiy) continue;
                    const F dsy = s1y[j1] - s0y[j1];
#pragma unroll
                    for (int j2 = 0; j2 < NP; ++j2) {
                        if (j2 < loz || j2 > hiz) continue;
                        const F dsz = s1z[j2] - s0z[j2];
                        const double tr = (transverse<F>(s0y[j1], dsy, s0z[j2], dsz) * sp.fac[0]) * ww;
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
                        const double tr = (transverse<F>(s0z[j1], dsz, s0x[j2], dsx) * sp.fac[1]) * ww;
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
                        const double tr = (transverse<F>(s0x[j1], dsx, s0y[j2], dsy) * sp.fac[2]) * ww;
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

            // -- super-cell membership (pic/particles.py:226-228) ----------
            dest = (ncx / g.scx) + g.gx * ((ncy / g.scy) + g.gy * (ncz / g.scz));
            stay = (dest == sc);
            leave = !stay;
            if (stay)
                nlc = (uint16_t)((ncx - orgx) + g.scx * ((ncy - orgy) + g.scy * (ncz - orgz)));
        }

        // ---- order-preserving compaction of stayers (ballot + block scan)
        const unsigned m = __ballot_sync(0xffffffffu, stay);
        if (lane == 0) warp_tot[wid] = __popc(m);
        __syncthreads();
        int off = 0, tot = 0;
#pragma unroll
        for (int k = 0; k < kThreads / 32; ++k) {
            const int v = warp_tot[k];
            off += (k < wid) ? v : 0;
            tot += v;
        }
        __syncthreads();
        if (stay) {
            const int64_t o = base_out + n_stay + off + __popc(m & ((1u << lane) - 1u));
            out.ox[o] = nox; out.oy[o] = noy; out.oz[o] = noz;
            out.ux[o] = nux; out.uy[o] = nuy; out.uz[o] = nuz;
            out.w[o] = w;
            out.cell[o] = nlc;
        }
        n_stay += tot;

        // ---- leavers: warp-aggregated claim in the exchange buffer -------
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
    if (n_err) atomicAdd(&status[KWB_ST_MOVE_ERRORS], n_err);
    __syncthreads();

    // ---- flush the J tile: one red.global.add per non-zero entry -------
    for (int t = threadIdx.x; t < 3 * JV; t += kThreads) {
        const F v = jt[t];
        if (v != F(0)) {
            const int c = t / JV, r = t - c * JV;
            const int a = r % jx, b = (r / jx) % jy, d = r / (jx * jy);
            const int gi = pymod(orgx - H + a, g.nx), gj = pymod(orgy - H + b, g.ny),
                      gk = pymod(orgz - H + d, g.nz);
            atomicAdd((F *)fp.J[c] + fidx(gi, gj, gk, g.nx, g.ny), v);
        }
    }
    if (threadIdx.x == 0) {
        out.count[sc] = n_stay;
        atomicMax(&status[KWB_ST_MAX_COUNT], n_stay);
    }
}

// Append leavers to their destination super cell (the shift/migration
// phase, pic/particles.py:316-345).  Slot claims are atomic per super cell.
template <typename F>
__global__ void shift_kernel(StoreT<F> out, ExchT<F> ex, Geo g, int32_t *__restrict__ status) {
    int n = *ex.count;
    if (n > ex.capacity) n = ex.capacity;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&status[KWB_ST_LEAVERS], n);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int d = ex.dest[i];
        const int k = atomicAdd(&out.count[d], 1);
        if (k >= out.slots) {
            atomicSub(&out.count[d], 1);
            atomicAdd(&status[KWB_ST_STORE_OVERFLOW], 1);
            continue;
        }
        atomicMax(&status[KWB_ST_MAX_COUNT], k + 1);
        const int bx = d % g.gx, by = (d / g.gx) % g.gy, bz = d / (g.gx * g.gy);
        const int64_t o = (int64_t)d * out.slots + k;
        out.ox[o] = ex.ox[i]; out.oy[o] = ex.oy[i]; out.oz[o] = ex.oz[i];
        out.ux[o] = ex.ux[i]; out.uy[o] = ex.uy[i]; out.uz[o] = ex.uz[i];
        out.w[o] = ex.w[i];
        out.cell[o] = (uint16_t)((ex.cx[i] - bx * g.scx) +
                                 g.scx * ((ex.cy[i] - by * g.scy) + g.scy * (ex.cz[i] - bz * g.scz)));
    }
}

// ---- store load / export / repack ---------------------------------------

template <typename F>
__global__ void load_kernel(Geo g, StoreT<F> st, int64_t n, const int64_t *__restrict__ sc_start,
                            const int32_t *__restrict__ cx, const int32_t *__restrict__ cy,
                            const int32_t *__restrict__ cz, const F *__restrict__ ox,
                            const F *__restrict__ oy, const F *__restrict__ oz,
                            const F *__restrict__ ux, const F *__restrict__ uy,
                            const F *__restrict__ uz, const F *__restrict__ w,
                            int32_t *__restrict__ status) {
    const int n_sc = g.gx * g.gy * g.gz;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_sc; s += stride) {
        const int64_t c = sc_start[s + 1] - sc_start[s];
        st.count[s] = (int32_t)(c < st.slots ? c : st.slots);
        if (c > st.slots) atomicAdd(&status[KWB_ST_LOAD_ERRORS], (int)(c - st.slots));
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        int lo = 0, hi = n_sc;  // sc_start[lo] <= i < sc_start[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (sc_start[mid] <= i) lo = mid; else hi = mid;
        }
        const int s = lo;
        const int64_t slot = i - sc_start[s];
        const int bx = s % g.gx, by = (s / g.gx) % g.gy, bz = s / (g.gx * g.gy);
        const int lx = cx[i] - bx * g.scx, ly = cy[i] - by * g.scy, lz = cz[i] - bz * g.scz;
        if (slot >= st.slots || lx < 0 || lx >= g.scx || ly < 0 || ly >= g.scy || lz < 0 ||
            lz >= g.scz) {
            if (slot < st.slots) atomicAdd(&status[KWB_ST_LOAD_ERRORS], 1);
            continue;
        }
        const int64_t o = (int64_t)s * st.slots + slot;
        st.ox[o] = ox[i]; st.oy[o] = oy[i]; st.oz[o] = oz[i];
        st.ux[o] = ux[i]; st.uy[o] = uy[i]; st.uz[o] = uz[i];
        st.w[o] = w[i];
        st.cell[o] = (uint16_t)(lx + g.scx * (ly + g.scy * lz));
    }
}

template <typename F>
__global__ void export_kernel(Geo g, StoreT<F> st, const int64_t *__restrict__ out_start,
                              int32_t *cx, int32_t *cy, int32_t *cz, F *ox, F *oy, F *oz, F *ux,
                              F *uy, F *uz, F *w) {
    const int n_sc = g.gx * g.gy * g.gz;
    for (int s = blockIdx.x; s < n_sc; s += gridDim.x) {
        const int n = st.count[s];
        const int bx = s % g.gx, by = (s / g.gx) % g.gy, bz = s / (g.gx * g.gy);
        const int64_t base = (int64_t)s * st.slots;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int64_t q = base + i, o = out_start[s] + i;
            const int lc = st.cell[q];
            cx[o] = bx * g.scx + lc % g.scx;
            cy[o] = by * g.scy + (lc / g.scx) % g.scy;
            cz[o] = bz * g.scz + lc / (g.scx * g.scy);
            ox[o] = st.ox[q]; oy[o] = st.oy[q]; oz[o] = st.oz[q];
            ux[o] = st.ux[q]; uy[o] = st.uy[q]; uz[o] = st.uz[q];
            w[o] = st.w[q];
        }
    }
}

template <typename F>
__global__ void repack_kernel(Geo g, StoreT<F> src, StoreT<F> dst) {
    const int n_sc = g.gx * g.gy * g.gz;
    for (int s = blockIdx.x; s < n_sc; s += gridDim.x) {
        const int n = min(src.count[s], dst.slots);
        const int64_t a = (int64_t)s * src.slots, b = (int64_t)s * dst.slots;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            dst.ox[b + i] = src.ox[a + i]; dst.oy[b + i] = src.oy[a + i];
            dst.oz[b + i] = src.oz[a + i]; dst.ux[b + i] = src.ux[a + i];
            dst.uy[b + i] = src.uy[a + i]; dst.uz[b + i] = src.uz[a + i];
            dst.w[b + i] = src.w[a + i]; dst.cell[b + i] = src.cell[a + i];
        }
        if (threadIdx.x == 0) dst.count[s] = n;
    }
}

// ---- validation charge density and particle moments --------------------

// pic/kernels.py:291-326 `_rho_tsc` (order 2) and the matching CIC/PCS shape
// deposits; float64 accumulation with global atomics.
template <typename F, int ORDER>
__global__ void __launch_bounds__(kThreads)
rho_kernel(Geo g, StoreT<F> st, double q_inv_vol, double *__restrict__ rho) {
    const int sc = blockIdx.x;
    const int bx = sc % g.gx, by = (sc / g.gx) % g.gy, bz = sc / (g.gx * g.gy);
    const int n = st.count[sc];
    const int64_t base = (int64_t)sc * st.slots;
    for (int i = threadIdx.x; i < n; i += kThreads) {
        const int64_t q = base + i;
        const int lc = st.cell[q];
        const int cx = bx * g.scx + lc % g.scx, cy = by * g.scy + (lc / g.scx) % g.scy,
                  cz = bz * g.scz + lc / (g.scx * g.scy);
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
                    for (int c = 0; c < 3; ++c) {
                        const int kc = pymod(cz - 1 + c, g.nz);
                        atomicAdd(rho + fidx(ia, jb, kc, g.nx, g.ny), ((qw * wx[a]) * wy[b]) * wz[c]);
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
                    for (int c = 0; c < NP; ++c) {
                        if (sz[c] == F(0)) continue;
                        const int kc = pymod(cz - H + c, g.nz);
                        atomicAdd(rho + fidx(ia, jb, kc, g.nx, g.ny),
                                  ((qw * (double)sx[a]) * (double)sy[b]) * (double)sz[c]);
                    }
                }
            }
        }
    }
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
__global__ void __launch_bounds__(kThreads)
moments_kernel(Geo g, StoreT<F> st, double charge, double mass, double *__restrict__ out) {
    __shared__ double red[kThreads / 32];
    const int n_sc = g.gx * g.gy * g.gz;
    double cen = 0.0, qw = 0.0, ke = 0.0;
    for (int sc = blockIdx.x; sc < n_sc; sc += gridDim.x) {
        const int n = st.count[sc];
        if (threadIdx.x == 0) cen += (double)n;
        const int64_t base = (int64_t)sc * st.slots;
        for (int i = threadIdx.x; i < n; i += kThreads) {
            const int64_t q = base + i;
            const double ux = (double)st.ux[q], uy = (double)st.uy[q], uz = (double)st.uz[q];
            const double ww = (double)st.w[q];
            const double gm = sqrt(((1.0 + ux * ux) + uy * uy) + uz * uz);
            qw += ww;
            ke += (gm - 1.0) * ww;
        }
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
    if (g->scx * g->scy * g->scz > 65535) {
        kwb_set_error("super-cell volume exceeds the 16-bit local cell index");
        return KWB_EINVAL;
    }
    if (g->dtype != KWB_F32 && g->dtype != KWB_F64) {
        kwb_set_error("dtype must be KWB_F32 or KWB_F64");
        return KWB_EINVAL;
    }
    return KWB_OK;
}

static int check_store(const kwb_store *s, const char *what) {
    if (!s || !s->ox || !s->oy || !s->oz || !s->ux || !s->uy || !s->uz || !s->w || !s->cell ||
        !s->count || s->slots_per_sc <= 0) {
        kwb_set_error("%s store is incomplete", what);
        return KWB_EINVAL;
    }
    return KWB_OK;
}

template <typename F, int ORDER>
static int launch_advance(const kwb_grid *g, const kwb_species *sp, const kwb_store *in,
                          const kwb_store *out, const kwb_exchange *ex, void *const E[3],
                          void *const B[3], void *const J[3], int32_t *status,
                          cudaStream_t stream) {
    Geo geo = geo_of(*g);
    size_t smem = advance_smem_bytes<F, ORDER>(geo);
    auto kern = advance_kernel<F, ORDER>;
    if (smem > 48 * 1024) {
        if (smem > 227 * 1024) {
            kwb_set_error("super cell too large for the shared-memory tiles (%zu B)", smem);
            return KWB_EINVAL;
        }
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    FieldPtrs fp;
    for (int c = 0; c < 3; ++c) { fp.E[c] = E[c]; fp.B[c] = B[c]; fp.J[c] = J[c]; }
    if (cudaMemsetAsync(ex->count, 0, sizeof(int32_t), stream) != cudaSuccess)
        return kwb_check_launch("exchange counter reset");
    const int n_sc = g->gx * g->gy * g->gz;
    kern<<<n_sc, kThreads, smem, stream>>>(geo, *sp, store_of<F>(*in), store_of<F>(*out),
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
    if (out->slots_per_sc < in->slots_per_sc) {
        kwb_set_error("advance: output store smaller than input store");
        return KWB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (g->dtype == KWB_F32) {
        switch (shape_order) {
            case 1: return launch_advance<float, 1>(g, sp, in, out, ex, E, B, J, status, s);
            case 2: return launch_advance<float, 2>(g, sp, in, out, ex, E, B, J, status, s);
            case 3: return launch_advance<float, 3>(g, sp, in, out, ex, E, B, J, status, s);
        }
    } else {
        switch (shape_order) {
            case 1: return launch_advance<double, 1>(g, sp, in, out, ex, E, B, J, status, s);
            case 2: return launch_advance<double, 2>(g, sp, in, out, ex, E, B, J, status, s);
            case 3: return launch_advance<double, 3>(g, sp, in, out, ex, E, B, J, status, s);
        }
    }
    kwb_set_error("shape_order must be 1 (CIC), 2 (TSC) or 3 (PCS), got %d", shape_order);
    return KWB_EINVAL;
}

static int shift_grid_blocks() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms * 4;
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
    const int blocks = shift_grid_blocks();
    if (g->dtype == KWB_F32)
        shift_kernel<float><<<blocks, 256, 0, s>>>(store_of<float>(*out), exch_of<float>(*ex), geo, status);
    else
        shift_kernel<double><<<blocks, 256, 0, s>>>(store_of<double>(*out), exch_of<double>(*ex), geo, status);
    return kwb_check_launch("shift_kernel");
}

extern "C" int kwb_store_load(const kwb_grid *g, const kwb_store *st, int64_t n,
                              const int64_t *sc_start, const int32_t *cx, const int32_t *cy,
                              const int32_t *cz, void *const f7[7], int32_t *status,
                              kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(st, "target"))) return rc;
    if (!sc_start || !status || (n > 0 && (!cx || !cy || !cz || !f7))) {
        kwb_set_error("store_load: NULL argument");
        return KWB_EINVAL;
    }
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = shift_grid_blocks() * 2;
    if (g->dtype == KWB_F32) {
        const float *const *f = (const float *const *)f7;
        load_kernel<float><<<blocks, 256, 0, s>>>(geo, store_of<float>(*st), n, sc_start, cx, cy, cz,
                                                  f[0], f[1], f[2], f[3], f[4], f[5], f[6], status);
    } else {
        const double *const *f = (const double *const *)f7;
        load_kernel<double><<<blocks, 256, 0, s>>>(geo, store_of<double>(*st), n, sc_start, cx, cy, cz,
                                                   f[0], f[1], f[2], f[3], f[4], f[5], f[6], status);
    }
    return kwb_check_launch("load_kernel");
}

extern "C" int kwb_store_export(const kwb_grid *g, const kwb_store *st, const int64_t *out_start,
                                int32_t *cx, int32_t *cy, int32_t *cz, void *const f7[7],
                                kwb_stream_t stream) {
    int rc = check_grid(g);
    if (rc) return rc;
    if ((rc = check_store(st, "source"))) return rc;
    if (!out_start || !cx || !cy || !cz || !f7) {
        kwb_set_error("store_export: NULL argument");
        return KWB_EINVAL;
    }
    Geo geo = geo_of(*g);
    cudaStream_t s = (cudaStream_t)stream;
    const int n_sc = g->gx * g->gy * g->gz;
    const int blocks = n_sc < 65535 ? n_sc : 65535;
    if (g->dtype == KWB_F32) {
        float *const *f = (float *const *)f7;
        export_kernel<float><<<blocks, 256, 0, s>>>(geo, store_of<float>(*st), out_start, cx, cy, cz,
                                                    f[0], f[1], f[2], f[3], f[4], f[5], f[6]);
    } else {
        double *const *f = (double *const *)f7;
        export_kernel<double><<<blocks, 256, 0, s>>>(geo, store_of<double>(*st), out_start, cx, cy, cz,
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
    const int n_sc = g->gx * g->gy * g->gz;
    const int blocks = n_sc < 65535 ? n_sc : 65535;
    if (g->dtype == KWB_F32)
        repack_kernel<float><<<blocks, 256, 0, s>>>(geo, store_of<float>(*src), store_of<float>(*dst));
    else
        repack_kernel<double><<<blocks, 256, 0, s>>>(geo, store_of<double>(*src), store_of<double>(*dst));
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
    const int n_sc = g->gx * g->gy * g->gz;
#define KWB_RHO(T, O) rho_kernel<T, O><<<n_sc, kThreads, 0, s>>>(geo, store_of<T>(*st), sp->q_inv_vol, rho)
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
    const int n_sc = g->gx * g->gy * g->gz;
    const int blocks = n_sc < shift_grid_blocks() ? n_sc : shift_grid_blocks();
    if (g->dtype == KWB_F32)
        moments_kernel<float><<<blocks, kThreads, 0, s>>>(geo, store_of<float>(*st), sp->charge, sp->mass, out);
    else
        moments_kernel<double><<<blocks, kThreads, 0, s>>>(geo, store_of<double>(*st), sp->charge, sp->mass, out);
    return kwb_check_launch("moments_kernel");
}
