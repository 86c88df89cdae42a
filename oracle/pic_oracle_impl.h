/* Precision-generic body of the CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * Included twice by pic_oracle.c with FT = float / double and SFX = _f32 /
 * _f64.  Every function restates one compiled reference kernel of
 * kernelweave.pic with the reference's exact rounding recipe (SURVEY.md
 * Appendix A): Numba promotes Python-float constants and int32+float32 to
 * double, keeps F*F / F-F products in the storage type, never contracts to
 * FMA (this file must be built with -ffp-contract=off), and rounds to the
 * storage type only on store.
 *
 * Store layout is the reference SuperCellStore layout (pic/particles.py:21-61):
 * SoA (n_frames, cap) arrays, frame chains head/next_f per super cell, u8 occ.
 * Field arrays are numpy C order (nx, ny, nz), z fastest (pic/fields.py:48-50).
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define ORC(name) CAT(orc_##name, SFX)

/* pic/kernels.py:26-47 `_sample`: trilinear, periodic Python-mod wrap. */
static inline double CAT(sample, SFX)(const FT *a, double px, double py, double pz,
                                      double sx, double sy, double sz,
                                      int64_t nx, int64_t ny, int64_t nz) {
    double tx = px - sx, ty = py - sy, tz = pz - sz;
    int64_t ix = (int64_t)floor(tx), iy = (int64_t)floor(ty), iz = (int64_t)floor(tz);
    double fx = tx - (double)ix, fy = ty - (double)iy, fz = tz - (double)iz;
    int64_t i0 = pymod(ix, nx), i1 = pymod(ix + 1, nx);
    int64_t j0 = pymod(iy, ny), j1 = pymod(iy + 1, ny);
    int64_t k0 = pymod(iz, nz), k1 = pymod(iz + 1, nz);
#define A_(i, j, k) ((double)a[((i) * ny + (j)) * nz + (k)])
    double c00 = A_(i0, j0, k0) * (1.0 - fx) + A_(i1, j0, k0) * fx;
    double c10 = A_(i0, j1, k0) * (1.0 - fx) + A_(i1, j1, k0) * fx;
    double c01 = A_(i0, j0, k1) * (1.0 - fx) + A_(i1, j0, k1) * fx;
    double c11 = A_(i0, j1, k1) * (1.0 - fx) + A_(i1, j1, k1) * fx;
#undef A_
    return (c00 * (1.0 - fy) + c10 * fy) * (1.0 - fz) + (c01 * (1.0 - fy) + c11 * fy) * fz;
}

/* pic/kernels.py:53-77 `_gather` (stagger table pic/kernels.py:50). */
void ORC(gather)(const orc_store *st, const orc_fields *fd, int nthreads) {
    const int64_t nx = fd->nx, ny = fd->ny, nz = fd->nz;
    const FT *F6[6] = {(const FT *)fd->Ex, (const FT *)fd->Ey, (const FT *)fd->Ez,
                       (const FT *)fd->Bx, (const FT *)fd->By, (const FT *)fd->Bz};
    FT *P6[6] = {(FT *)st->epx, (FT *)st->epy, (FT *)st->epz,
                 (FT *)st->bpx, (FT *)st->bpy, (FT *)st->bpz};
    const FT *ox = st->ox, *oy = st->oy, *oz = st->oz;
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
    for (int64_t sc = 0; sc < st->n_sc; ++sc) {
        for (int32_t f = st->head[sc]; f >= 0; f = st->next_f[f]) {
            for (int64_t s = 0; s < st->cap; ++s) {
                int64_t q = (int64_t)f * st->cap + s;
                if (!st->occ[q]) continue;
                double px = (double)st->cx[q] + (double)ox[q];
                double py = (double)st->cy[q] + (double)oy[q];
                double pz = (double)st->cz[q] + (double)oz[q];
                for (int c = 0; c < 6; ++c)
                    P6[c][q] = (FT)CAT(sample, SFX)(F6[c], px, py, pz, ORC_STAGGER[c][0],
                                                    ORC_STAGGER[c][1], ORC_STAGGER[c][2],
                                                    nx, ny, nz);
            }
        }
    }
}

/* pic/kernels.py:80-104 `_push`: relativistic Boris, all arithmetic in double. */
void ORC(push)(const orc_store *st, double qm, int nthreads) {
    FT *ux = st->ux, *uy = st->uy, *uz = st->uz;
    const FT *ex = st->epx, *ey = st->epy, *ez = st->epz;
    const FT *bx = st->bpx, *by = st->bpy, *bz = st->bpz;
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
    for (int64_t sc = 0; sc < st->n_sc; ++sc) {
        for (int32_t f = st->head[sc]; f >= 0; f = st->next_f[f]) {
            for (int64_t s = 0; s < st->cap; ++s) {
                int64_t q = (int64_t)f * st->cap + s;
                if (!st->occ[q]) continue;
                double umx = (double)ux[q] + qm * (double)ex[q];
                double umy = (double)uy[q] + qm * (double)ey[q];
                double umz = (double)uz[q] + qm * (double)ez[q];
                double gam = sqrt(((1.0 + umx * umx) + umy * umy) + umz * umz);
                double tx = (qm * (double)bx[q]) / gam;
                double ty = (qm * (double)by[q]) / gam;
                double tz = (qm * (double)bz[q]) / gam;
                double tsq = (tx * tx + ty * ty) + tz * tz;
                double sx = (2.0 * tx) / (1.0 + tsq);
                double sy = (2.0 * ty) / (1.0 + tsq);
                double sz = (2.0 * tz) / (1.0 + tsq);
                double upx = umx + (umy * tz - umz * ty);
                double upy = umy + (umz * tx - umx * tz);
                double upz = umz + (umx * ty - umy * tx);
                ux[q] = (FT)((umx + (upy * sz - upz * sy)) + qm * (double)ex[q]);
                uy[q] = (FT)((umy + (upz * sx - upx * sz)) + qm * (double)ey[q]);
                uz[q] = (FT)((umz + (upx * sy - upy * sx)) + qm * (double)ez[q]);
            }
        }
    }
}

/* pic/kernels.py:107-135 `_move`: gamma from storage-type squares, floor carry,
 * Python-mod periodic cell wrap; the offset may round to exactly 1.0 in f32. */
void ORC(move)(const orc_store *st, double dtdx, double dtdy, double dtdz,
               int64_t nx, int64_t ny, int64_t nz, int nthreads) {
    FT *ox = st->ox, *oy = st->oy, *oz = st->oz;
    FT *oox = st->oox, *ooy = st->ooy, *ooz = st->ooz;
    const FT *ux = st->ux, *uy = st->uy, *uz = st->uz;
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
    for (int64_t sc = 0; sc < st->n_sc; ++sc) {
        for (int32_t f = st->head[sc]; f >= 0; f = st->next_f[f]) {
            for (int64_t s = 0; s < st->cap; ++s) {
                int64_t q = (int64_t)f * st->cap + s;
                if (!st->occ[q]) continue;
                oox[q] = ox[q]; ooy[q] = oy[q]; ooz[q] = oz[q];
                st->ocx[q] = st->cx[q]; st->ocy[q] = st->cy[q]; st->ocz[q] = st->cz[q];
                FT sxx = ux[q] * ux[q], syy = uy[q] * uy[q], szz = uz[q] * uz[q];
                double gam = sqrt(((1.0 + (double)sxx) + (double)syy) + (double)szz);
                double px = (double)ox[q] + ((double)ux[q] / gam) * dtdx;
                double py = (double)oy[q] + ((double)uy[q] / gam) * dtdy;
                double pz = (double)oz[q] + ((double)uz[q] / gam) * dtdz;
                int64_t dxi = (int64_t)floor(px), dyi = (int64_t)floor(py), dzi = (int64_t)floor(pz);
                ox[q] = (FT)(px - (double)dxi);
                oy[q] = (FT)(py - (double)dyi);
                oz[q] = (FT)(pz - (double)dzi);
                st->cx[q] = (int32_t)pymod((int64_t)st->cx[q] + dxi, nx);
                st->cy[q] = (int32_t)pymod((int64_t)st->cy[q] + dyi, ny);
                st->cz[q] = (int32_t)pymod((int64_t)st->cz[q] + dzi, nz);
            }
        }
    }
}

/* pic/kernels.py:138-150 `_shape5_into` generalised to the shape order
 * (1 CIC, 2 TSC, 3 PCS): out[idx] = (FT) W(|x - centre(idx)|) with
 * centre(idx) = (idx - H) + 0.5, H = 2 (5-point arrays) or 3 (7-point, PCS).
 * Order 2 is the reference's TSC bit for bit. */
static inline void CAT(shape_into, SFX)(double x, int order, FT *out) {
    const int np = (order == 3) ? 7 : 5, H = (order == 3) ? 3 : 2;
    for (int idx = 0; idx < np; ++idx) {
        double d = x - ((double)(idx - H) + 0.5);
        if (d < 0) d = -d;
        double v;
        if (order == 2) {
            if (d < 0.5) v = 0.75 - d * d;
            else if (d < 1.5) { double e = 1.5 - d; v = (0.5 * e) * e; }
            else v = 0.0;
        } else if (order == 1) {
            v = (d < 1.0) ? 1.0 - d : 0.0;
        } else {
            if (d < 1.0) v = ((4.0 - (6.0 * d) * d) + ((3.0 * d) * d) * d) / 6.0;
            else if (d < 2.0) { double e = 2.0 - d; v = ((e * e) * e) / 6.0; }
            else v = 0.0;
        }
        out[idx] = (FT)v;
    }
}

/* Transverse factor of the density decomposition, pic/kernels.py:215-218:
 * ((F(a0*b0) + (0.5*da)*b0) + (0.5*a0)*db) + F(da*db)/3.0 */
static inline double CAT(transverse, SFX)(FT a0, FT da, FT b0, FT db) {
    FT p00 = a0 * b0, pdd = da * db;
    return (((double)p00 + (0.5 * (double)da) * (double)b0) + (0.5 * (double)a0) * (double)db)
           + (double)pdd / 3.0;
}

/* pic/kernels.py:153-250 `_deposit_collect` for one super cell into `tile`
 * (3, tnx, tny, tnz), halo hw = 2 (CIC/TSC) or 3 (PCS).  Returns the count of
 * particles that moved a full cell or more (reference: ContractViolation). */
static int64_t CAT(deposit_sc, SFX)(const orc_store *st, int64_t sc, int order,
                                    const double fac[3], int64_t nx, int64_t ny, int64_t nz,
                                    int64_t orgx, int64_t orgy, int64_t orgz,
                                    int64_t tnx, int64_t tny, int64_t tnz, FT *tile) {
    const int np = (order == 3) ? 7 : 5;
    const int top = np - 2;           /* running-sum end / hi for dc == 0 */
    FT s0x[7], s0y[7], s0z[7], s1x[7], s1y[7], s1z[7];
    const FT *ox = st->ox, *oy = st->oy, *oz = st->oz;
    const FT *oox = st->oox, *ooy = st->ooy, *ooz = st->ooz, *w = st->w;
    int64_t errors = 0;
    const int64_t tplane = tnx * tny * tnz;
#define T_(c, i, j, k) tile[(c) * tplane + ((i) * tny + (j)) * tnz + (k)]
    /* orc_reverse_slots: walk each frame's slots backwards -- another valid
     * particle order of the same super cell (the reference's order depends on
     * its migration history), used only to measure the reference's own
     * f32 accumulation-order spread (tests/parity_util.py order_spread). */
    for (int32_t f = st->head[sc]; f >= 0; f = st->next_f[f]) {
        for (int64_t s_ = 0; s_ < st->cap; ++s_) {
            const int64_t s = orc_reverse_slots ? st->cap - 1 - s_ : s_;
            int64_t q = (int64_t)f * st->cap + s;
            if (!st->occ[q]) continue;
            int64_t dcx = (int64_t)st->cx[q] - st->ocx[q];
            if (dcx > 1) dcx -= nx; else if (dcx < -1) dcx += nx;
            int64_t dcy = (int64_t)st->cy[q] - st->ocy[q];
            if (dcy > 1) dcy -= ny; else if (dcy < -1) dcy += ny;
            int64_t dcz = (int64_t)st->cz[q] - st->ocz[q];
            if (dcz > 1) dcz -= nz; else if (dcz < -1) dcz += nz;
            if (dcx > 1 || dcx < -1 || dcy > 1 || dcy < -1 || dcz > 1 || dcz < -1) {
                ++errors;
                continue;
            }
            CAT(shape_into, SFX)((double)oox[q], order, s0x);
            CAT(shape_into, SFX)((double)ooy[q], order, s0y);
            CAT(shape_into, SFX)((double)ooz[q], order, s0z);
            CAT(shape_into, SFX)((double)dcx + (double)ox[q], order, s1x);
            CAT(shape_into, SFX)((double)dcy + (double)oy[q], order, s1y);
            CAT(shape_into, SFX)((double)dcz + (double)oz[q], order, s1z);
            int64_t lx = st->ocx[q] - orgx, ly = st->ocy[q] - orgy, lz = st->ocz[q] - orgz;
            double ww = (double)w[q];
            int64_t lox = 1 + (dcx < 0 ? dcx : 0), hix = top + (dcx > 0 ? dcx : 0);
            int64_t loy = 1 + (dcy < 0 ? dcy : 0), hiy = top + (dcy > 0 ? dcy : 0);
            int64_t loz = 1 + (dcz < 0 ? dcz : 0), hiz = top + (dcz > 0 ? dcz : 0);
            int64_t ex = hix < top ? hix : top, ey = hiy < top ? hiy : top, ez = hiz < top ? hiz : top;
            /* x currents: running sum of DSx against the (y, z) transverse factor */
            for (int64_t j1 = loy; j1 <= hiy; ++j1) {
                FT dsy = s1y[j1] - s0y[j1];
                for (int64_t j2 = loz; j2 <= hiz; ++j2) {
                    FT dsz = s1z[j2] - s0z[j2];
                    double tr = (CAT(transverse, SFX)(s0y[j1], dsy, s0z[j2], dsz) * fac[0]) * ww;
                    double acc = 0.0;
                    for (int64_t ja = lox; ja <= ex; ++ja) {
                        FT d = s1x[ja] - s0x[ja];
                        acc += (double)d * tr;
                        FT *t = &T_(0, lx + ja, ly + j1, lz + j2);
                        *t = (FT)((double)*t + acc);
                    }
                }
            }
            /* y currents: (z, x) transverse factor */
            for (int64_t j1 = loz; j1 <= hiz; ++j1) {
                FT dsz = s1z[j1] - s0z[j1];
                for (int64_t j2 = lox; j2 <= hix; ++j2) {
                    FT dsx = s1x[j2] - s0x[j2];
                    double tr = (CAT(transverse, SFX)(s0z[j1], dsz, s0x[j2], dsx) * fac[1]) * ww;
                    double acc = 0.0;
                    for (int64_t ja = loy; ja <= ey; ++ja) {
                        FT d = s1y[ja] - s0y[ja];
                        acc += (double)d * tr;
                        FT *t = &T_(1, lx + j2, ly + ja, lz + j1);
                        *t = (FT)((double)*t + acc);
                    }
                }
            }
            /* z currents: (x, y) transverse factor */
            for (int64_t j1 = lox; j1 <= hix; ++j1) {
                FT dsx = s1x[j1] - s0x[j1];
                for (int64_t j2 = loy; j2 <= hiy; ++j2) {
                    FT dsy = s1y[j2] - s0y[j2];
                    double tr = (CAT(transverse, SFX)(s0x[j1], dsx, s0y[j2], dsy) * fac[2]) * ww;
                    double acc = 0.0;
                    for (int64_t ja = loz; ja <= ez; ++ja) {
                        FT d = s1z[ja] - s0z[ja];
                        acc += (double)d * tr;
                        FT *t = &T_(2, lx + j1, ly + j2, lz + ja);
                        *t = (FT)((double)*t + acc);
                    }
                }
            }
        }
    }
#undef T_
    return errors;
}

/* DepositKernel (pic/kernels.py:379-412): per-super-cell tiles (computed in
 * parallel), then the J += tile merge through the wrapped maps
 * (kw/atomics.py:147-163, sim.py:88-94) in ascending super-cell order, in the
 * storage type -- identical to the Serial back-end's order.
 * `tiles` is caller scratch of n_sc * 3 * tnx*tny*tnz elements. */
int64_t ORC(deposit)(const orc_store *st, const orc_fields *fd, int order, const double fac[3],
                     int64_t scx, int64_t scy, int64_t scz, void *tiles_v, int nthreads) {
    const int64_t nx = fd->nx, ny = fd->ny, nz = fd->nz;
    const int64_t hw = (order == 3) ? 3 : 2;
    const int64_t tnx = scx + 2 * hw, tny = scy + 2 * hw, tnz = scz + 2 * hw;
    const int64_t tsize = 3 * tnx * tny * tnz;
    const int64_t gx = nx / scx, gy = ny / scy;
    FT *tiles = (FT *)tiles_v;
    int64_t errors = 0;
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads) reduction(+ : errors)
    for (int64_t sc = 0; sc < st->n_sc; ++sc) {
        FT *tile = tiles + sc * tsize;
        memset(tile, 0, sizeof(FT) * tsize);
        int64_t bx = sc % gx, by = (sc / gx) % gy, bz = sc / (gx * gy);
        errors += CAT(deposit_sc, SFX)(st, sc, order, fac, nx, ny, nz, bx * scx, by * scy,
                                       bz * scz, tnx, tny, tnz, tile);
    }
    if (errors) return errors;
    FT *J3[3] = {(FT *)fd->Jx, (FT *)fd->Jy, (FT *)fd->Jz};
    /* merge order: ascending (the Serial back-end, the bit-authoritative
     * order) or, for orc_merge_seed != 0, a seeded random permutation -- the
     * BlockPool back-end merges tiles in worker-completion order
     * (kw/backends.py:115-139), which is how the reference's own J spread
     * is measured (tests/parity_util.py order_spread). */
    int64_t *perm = NULL;
    if (orc_merge_seed) {
        perm = (int64_t *)malloc(sizeof(int64_t) * st->n_sc);
        uint64_t rs = orc_merge_seed;
        for (int64_t i = 0; i < st->n_sc; ++i) perm[i] = i;
        for (int64_t i = st->n_sc - 1; i > 0; --i) {
            int64_t j = (int64_t)(orc_rng_next(&rs) % (uint64_t)(i + 1));
            int64_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
        }
    }
    for (int64_t si = 0; si < st->n_sc; ++si) {
        const int64_t sc = perm ? perm[si] : si;
        const FT *tile = tiles + sc * tsize;
        int64_t bx = sc % gx, by = (sc / gx) % gy, bz = sc / (gx * gy);
        for (int c = 0; c < 3; ++c) {
            const FT *tc = tile + c * tnx * tny * tnz;
            FT *J = J3[c];
            for (int64_t i = 0; i < tnx; ++i) {
                int64_t mi = pymod(bx * scx - hw + i, nx);
                for (int64_t j = 0; j < tny; ++j) {
                    int64_t mj = pymod(by * scy - hw + j, ny);
                    for (int64_t k = 0; k < tnz; ++k) {
                        int64_t mk = pymod(bz * scz - hw + k, nz);
                        FT *t = &J[(mi * ny + mj) * nz + mk];
                        *t = *t + tc[(i * tny + j) * tnz + k];
                    }
                }
            }
        }
    }
    free(perm);
    return 0;
}

/* pic/kernels.py:253-269 `_faraday`: B -= half_dt * curl E (forward diffs). */
void ORC(faraday)(const orc_fields *fd, double half_dt, int nthreads) {
    const int64_t nx = fd->nx, ny = fd->ny, nz = fd->nz;
    const double dx = fd->dx, dy = fd->dy, dz = fd->dz;
    const FT *Ex = fd->Ex, *Ey = fd->Ey, *Ez = fd->Ez;
    FT *Bx = fd->Bx, *By = fd->By, *Bz = fd->Bz;
#define I_(i, j, k) (((i) * ny + (j)) * nz + (k))
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t i = 0; i < nx; ++i) {
        int64_t ip = (i + 1) % nx;
        for (int64_t j = 0; j < ny; ++j) {
            int64_t jp = (j + 1) % ny;
            for (int64_t k = 0; k < nz; ++k) {
                int64_t kp = (k + 1) % nz, c = I_(i, j, k);
                FT a = Ez[I_(i, jp, k)] - Ez[c], b = Ey[I_(i, j, kp)] - Ey[c];
                Bx[c] = (FT)((double)Bx[c] - half_dt * ((double)a / dy - (double)b / dz));
                a = Ex[I_(i, j, kp)] - Ex[c]; b = Ez[I_(ip, j, k)] - Ez[c];
                By[c] = (FT)((double)By[c] - half_dt * ((double)a / dz - (double)b / dx));
                a = Ey[I_(ip, j, k)] - Ey[c]; b = Ex[I_(i, jp, k)] - Ex[c];
                Bz[c] = (FT)((double)Bz[c] - half_dt * ((double)a / dx - (double)b / dy));
            }
        }
    }
}

/* pic/kernels.py:272-288 `_ampere`: E += dt * (curl B - J) (backward diffs). */
void ORC(ampere)(const orc_fields *fd, double dt, int nthreads) {
    const int64_t nx = fd->nx, ny = fd->ny, nz = fd->nz;
    const double dx = fd->dx, dy = fd->dy, dz = fd->dz;
    FT *Ex = fd->Ex, *Ey = fd->Ey, *Ez = fd->Ez;
    const FT *Bx = fd->Bx, *By = fd->By, *Bz = fd->Bz;
    const FT *Jx = fd->Jx, *Jy = fd->Jy, *Jz = fd->Jz;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t i = 0; i < nx; ++i) {
        int64_t im = (i - 1 + nx) % nx;
        for (int64_t j = 0; j < ny; ++j) {
            int64_t jm = (j - 1 + ny) % ny;
            for (int64_t k = 0; k < nz; ++k) {
                int64_t km = (k - 1 + nz) % nz, c = I_(i, j, k);
                FT a = Bz[c] - Bz[I_(i, jm, k)], b = By[c] - By[I_(i, j, km)];
                Ex[c] = (FT)((double)Ex[c] + dt * (((double)a / dy - (double)b / dz) - (double)Jx[c]));
                a = Bx[c] - Bx[I_(i, j, km)]; b = Bz[c] - Bz[I_(im, j, k)];
                Ey[c] = (FT)((double)Ey[c] + dt * (((double)a / dz - (double)b / dx) - (double)Jy[c]));
                a = By[c] - By[I_(im, j, k)]; b = Bx[c] - Bx[I_(i, jm, k)];
                Ez[c] = (FT)((double)Ez[c] + dt * (((double)a / dx - (double)b / dy) - (double)Jz[c]));
            }
        }
    }
#undef I_
}

/* pic/kernels.py:291-326 `_rho_tsc` (order 2, pool order, f64 accumulation);
 * orders 1 and 3 use the matching shape arrays (SURVEY.md §8c extension):
 * rho[c - H + idx] += ((qw * Sx) * Sy) * Sz over the support. */
void ORC(rho)(const orc_store *st, int64_t n_frames, const int32_t *owner, int order,
              double q_inv_vol, double *rho, int64_t nx, int64_t ny, int64_t nz) {
    const FT *ox = st->ox, *oy = st->oy, *oz = st->oz, *w = st->w;
    for (int64_t f = 0; f < n_frames; ++f) {
        if (owner[f] < 0) continue;
        for (int64_t s = 0; s < st->cap; ++s) {
            int64_t q = f * st->cap + s;
            if (!st->occ[q]) continue;
            int64_t cx = st->cx[q], cy = st->cy[q], cz = st->cz[q];
            double qw = q_inv_vol * (double)w[q];
            if (order == 2) {
                double o, wx[3], wy[3], wz[3], l, r;
                o = (double)ox[q] - 0.5; l = 0.5 * ((0.5 - o) * (0.5 - o)); r = 0.5 * ((0.5 + o) * (0.5 + o));
                wx[0] = l; wx[1] = (1.0 - l) - r; wx[2] = r;
                o = (double)oy[q] - 0.5; l = 0.5 * ((0.5 - o) * (0.5 - o)); r = 0.5 * ((0.5 + o) * (0.5 + o));
                wy[0] = l; wy[1] = (1.0 - l) - r; wy[2] = r;
                o = (double)oz[q] - 0.5; l = 0.5 * ((0.5 - o) * (0.5 - o)); r = 0.5 * ((0.5 + o) * (0.5 + o));
                wz[0] = l; wz[1] = (1.0 - l) - r; wz[2] = r;
                int64_t kk[3] = {pymod(cz - 1, nz), pymod(cz, nz), pymod(cz + 1, nz)};
                for (int a = 0; a < 3; ++a) {
                    int64_t ia = pymod(cx - 1 + a, nx);
                    for (int b = 0; b < 3; ++b) {
                        int64_t jb = pymod(cy - 1 + b, ny);
                        for (int c = 0; c < 3; ++c)
                            rho[(ia * ny + jb) * nz + kk[c]] += ((qw * wx[a]) * wy[b]) * wz[c];
                    }
                }
            } else {
                FT sx[7], sy[7], sz[7];
                const int np = (order == 3) ? 7 : 5, H = (order == 3) ? 3 : 2;
                CAT(shape_into, SFX)((double)ox[q], order, sx);
                CAT(shape_into, SFX)((double)oy[q], order, sy);
                CAT(shape_into, SFX)((double)oz[q], order, sz);
                for (int a = 0; a < np; ++a) {
                    if (sx[a] == 0) continue;
                    int64_t ia = pymod(cx - H + a, nx);
                    for (int b = 0; b < np; ++b) {
                        if (sy[b] == 0) continue;
                        int64_t jb = pymod(cy - H + b, ny);
                        for (int c = 0; c < np; ++c) {
                            if (sz[c] == 0) continue;
                            rho[(ia * ny + jb) * nz + pymod(cz - H + c, nz)] +=
                                ((qw * (double)sx[a]) * (double)sy[b]) * (double)sz[c];
                        }
                    }
                }
            }
        }
    }
}

/* pic/particles.py:238-287 `_apply_migration`: storage-typed record copy. */
void ORC(apply_migration)(const orc_store *st, orc_pool *pl, int64_t count,
                          const int32_t *mov_f, const int32_t *mov_s, const int32_t *mov_dest) {
    FT *A7[7] = {(FT *)st->ox, (FT *)st->oy, (FT *)st->oz, (FT *)st->ux, (FT *)st->uy,
                 (FT *)st->uz, (FT *)st->w};
    int32_t *C3[3] = {st->cx, st->cy, st->cz};
    const int64_t cap = st->cap;
    for (int64_t i = 0; i < count; ++i) {
        int64_t src = (int64_t)mov_f[i] * cap + mov_s[i];
        int32_t dsc = mov_dest[i];
        int32_t t = pl->tail[dsc];
        int64_t slot = -1;
        if (t >= 0 && pl->nfilled[t] < cap) {
            for (int64_t cand = 0; cand < cap; ++cand)
                if (st->occ[(int64_t)t * cap + cand] == 0) { slot = cand; break; }
        } else {
            pl->free_top[0] -= 1;
            t = pl->free_stack[pl->free_top[0]];
            pl->owner[t] = dsc;
            pl->next_f[t] = -1;
            pl->nfilled[t] = 0;
            int32_t old_tail = pl->tail[dsc];
            pl->prev_f[t] = old_tail;
            if (old_tail >= 0) pl->next_f[old_tail] = t;
            else pl->head[dsc] = t;
            pl->tail[dsc] = t;
            slot = 0;
        }
        int64_t dst = (int64_t)t * cap + slot;
        st->occ[dst] = 1;
        pl->nfilled[t] += 1;
        for (int a = 0; a < 7; ++a) A7[a][dst] = A7[a][src];
        for (int a = 0; a < 3; ++a) C3[a][dst] = C3[a][src];
        st->occ[src] = 0;
        pl->nfilled[mov_f[i]] -= 1;
    }
}

#undef ORC
