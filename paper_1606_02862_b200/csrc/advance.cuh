// The fused particle advance: gather -> Boris push -> move -> Esirkepov
// deposit -> in-super-cell shift, one CTA per super cell, one thread per
// cell.  Included by particles.cu inside namespace kwb.
//
// Reference arithmetic: pic/kernels.py:26-135 (gather, push, move) is
// reproduced bit for bit in float64 with no FMA contraction (the library is
// built with --fmad=false), so particle state matches the reference exactly.
// pic/kernels.py:153-250 (deposit) is the same density decomposition in the
// storage precision: J is compared within tolerance, as the reference's own
// J depends on its (thread-pool) accumulation order.
//
// Per-CTA shared memory:
//   ebd   6 x (scx+2)(scy+2)(scz+2) float64  E/B + 1 guard cell, pre-widened
//                                             (no per-particle F->D converts;
//                                             float for float32 PCS, AdvCfg)
//   jt    3 x (scx+2H)(scy+2H)(scz+2H) F      J tile incl. the shape halo; the
//                                             register window of every cell is
//                                             swept in, the queued remainder
//                                             added with CAS
//   queue kWarps x kWarpQ crossing records    (per warp: the out-of-window part
//                                             of crossing particles, every
//                                             particle for PCS; deposited after
//                                             the main loop)
//   arr   V int                               in-super-cell arrivals per cell
//   pf    2 x 7 x 256 F                       next-particle records, cp.async
//                                             (no registers held between rounds)
//   wrap  periodic index tables for staging and the J flush

struct FieldPtrs {
    const void *E[3], *B[3];
    void *J[3];
    // optional [3][nz] base of every J z-plane (x fastest, nx*ny values):
    // z-slab guard planes point into the neighbour's halo buffer (peer /
    // IPC-mapped memory), so the J flush is also the halo exchange.  NULL:
    // plane z of J[c].
    void *const *jpl;
};

constexpr int kMaxCells = 256;            // super-cell volume limit = CTA size limit
constexpr int kWarps = kMaxCells / 32;
// KWB_WIN_SMEM: the float32 window's edge +1 (27 accumulators per thread)
// lives in per-thread shared memory (7 float4 per thread, conflict-free)
// instead of registers, so the kernel keeps 128 registers and 2 CTAs per SM
// (C2 advance: 4.38 ms vs 4.80 ms with the spilling 81-register window and
// 5.26 ms at one CTA per SM without spills; tools/gpurun/r02b.sh).
// KWB_WIN_REGS=1 selects the all-register window.
#if !defined(KWB_WIN_REGS) && !defined(KWB_WIN_SMEM)
#define KWB_WIN_SMEM 1
#endif
#ifndef KWB_WARPQ
#ifdef KWB_WIN_SMEM
#define KWB_WARPQ 96
#else
#define KWB_WARPQ 160
#endif
#endif
constexpr int kWarpQ = KWB_WARPQ;         // crossing-particle queue entries per warp
#ifndef KWB_WARPQ_PCS
#define KWB_WARPQ_PCS 32   // 64 with the closing-edge boxes is 116 KB: 1 CTA per SM
#endif
#ifndef KWB_MIN_BLOCKS
#define KWB_MIN_BLOCKS 2
#endif
#ifndef KWB_MIN_BLOCKS_PCS
#define KWB_MIN_BLOCKS_PCS 2
#endif

// Per-instance configuration.  The E/B tile is staged in float64 (no
// per-particle converts in the gather) except for float32 PCS, which stages
// the float fields as they are (the widening at the load is exact).  PCS
// queues every particle, so its queue is a 64-record ring drained 32 at a
// time (every lane busy) instead of 160 records: 70 KB instead of 108 KB of
// shared memory, 3 CTAs per SM instead of 2 -- more warps to hide its
// serial CAS chains (C4 PCS advance 45.1 -> 37.1 ms, ring 37.1 -> 35.4 ms).
// In the (8,8,4) instance the stayers then left the queue for the
// atomic-free warp boxes (kBoxX; +40 KB, back to 2 CTAs per SM):
// 35.4 -> 25.4 ms.
template <typename F, int ORDER>
struct AdvCfg {
    static constexpr bool kNarrowEB = ORDER == 3 && sizeof(F) == 4;
    using EB = std::conditional_t<kNarrowEB, float, double>;
    static constexpr int kQ = ORDER == 3 ? KWB_WARPQ_PCS : kWarpQ;
    static constexpr int kMinBlocks =
        sizeof(F) == 4 ? (ORDER == 3 ? KWB_MIN_BLOCKS_PCS : KWB_MIN_BLOCKS) : 1;
};

// a / 6 correctly rounded (the PCS weights' division) by
// div_rcp with r = RN(1/6): three fp64 operations instead of a division.
__device__ __forceinline__ double div6(double a) {
    return div_rcp(a, 6.0, 0.16666666666666666);
}

// ---- shape weights, bit for bit the reference's -------------------------
// pic/kernels.py:138-150 `_shape5_into`: weight (F) W(|x - centre|) with x
// and the distance in double, no contraction (the library is built with
// --fmad=false); CIC/PCS per the SURVEY.md §8c extension.  Rounding the
// weights to F only at the end is what keeps J within the reference's
// tolerance: the f32-evaluated weights of round 1 differ by an ulp, and
// ds = s1 - s0 turns that into ~1e-6 of J (profiles/r02_parity.md).
template <int ORDER>
__device__ __forceinline__ double wref(double d) {
    if (ORDER == 2) {
        const double e = 1.5 - d;
        return d < 0.5 ? 0.75 - d * d : (d < 1.5 ? (0.5 * e) * e : 0.0);
    } else if (ORDER == 1) {
        return d < 1.0 ? 1.0 - d : 0.0;
    } else {
        const double e = 2.0 - d;
        return d < 1.0 ? div6((4.0 - (6.0 * d) * d) + ((3.0 * d) * d) * d)
                       : (d < 2.0 ? div6((e * e) * e) : 0.0);
    }
}

// TSC/CIC weights at the three support points c-1, c, c+1 of a particle at
// x in [c, c+1] (x = old offset with c = 0, or x = dc + new offset with
// c = dc, exactly the reference's `(double)dc + (double)o`).  The distances
// x - (c - 0.5), x - (c + 0.5), (c + 1.5) - x are the reference's |x -
// centre| (signs known), and on these ranges the reference's branches
// reduce to the three formulas below (the boundary cases d = 0.5 / 1.5 give
// the same values), so each weight is the reference's bit for bit.
template <int ORDER, typename F>
__device__ __forceinline__ void wref3(double x, double c, F (&s)[3]) {
    const double dl = x - (c - 0.5), dm = x - (c + 0.5), dh = (c + 1.5) - x;
    if (ORDER == 2) {
        const double el = 1.5 - dl, eh = 1.5 - dh;
        s[0] = (F)((0.5 * el) * el);
        s[1] = (F)(0.75 - dm * dm);
        s[2] = (F)((0.5 * eh) * eh);
    } else {
        s[0] = (F)(dl < 1.0 ? 1.0 - dl : 0.0);
        s[1] = (F)(1.0 - fabs(dm));
        s[2] = (F)(dh < 1.0 ? 1.0 - dh : 0.0);
    }
}

// Weight (F) at anchor-relative support index i (0-based) of the old and
// the new position of one axis: the anchor is the old cell + m (m = -1 when
// dc < 0), so index i is own-relative point i + 1 - H + m, centre + 0.5.
template <int ORDER, typename F>
__device__ __forceinline__ void wpair(F oo, F no, int dc, int m, int i, F &s0, F &s1) {
    constexpr int H = Shape<ORDER>::H;
    const double ctr = (double)(i + 1 - H + m) + 0.5;
    const double xo = (double)oo, xn = (double)dc + (double)no;
    s0 = (F)wref<ORDER>(fabs(xo - ctr));
    s1 = (F)wref<ORDER>(fabs(xn - ctr));
}

// Yee staggers in cell units, pic/fields.py:24-31 (Ex Ey Ez Bx By Bz).
__host__ __device__ constexpr double stagger(int c, int a) {
    return (c == 0) ? (a == 0 ? 1.0 : 0.5)
         : (c == 1) ? (a == 1 ? 1.0 : 0.5)
         : (c == 2) ? (a == 2 ? 1.0 : 0.5)
         : (c == 3) ? (a == 0 ? 0.5 : 1.0)
         : (c == 4) ? (a == 1 ? 0.5 : 1.0)
                    : (a == 2 ? 0.5 : 1.0);
}

// 4/8-byte asynchronous global -> shared copy (LDGSTS), bypassing registers.
template <typename F>
__device__ __forceinline__ void cp_async_elem(F *dst, const F *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(d), "l"(src),
                 "n"((int)sizeof(F)));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// PCS stayers (particles that keep their cell, ~95 % at C4) are deposited
// without atomics into a warp-private box per J component: a warp of the
// (8,8,4) super cell is 8 x 4 cells of one z plane, and its stayers'
// footprints (edges -2..2 along the component -- the last the closing
// entry --, points -2..2 across) span Jx, Jy, Jz 12x8x5 entries each.  All lanes run the same entry
// sequence; an instruction group only varies the entry's z offset, and
// cells of one warp share z, so the lanes of a group never hit the same
// entry (plain read-add-write, 4-5 independent per group); __syncwarp
// orders consecutive groups.  The boxes are added into the J tile after
// the loop (CAS, ~40 per thread).
constexpr int kBoxX = 1440;          // 3 x 480 floats per warp
constexpr int kBoxFloats = kBoxX;
template <typename F, int ORDER>
__host__ __device__ inline bool pcs_box_layout(int scx, int scy, int scz) {
    return ORDER == 3 && sizeof(F) == 4 && scx == 8 && scy == 8 && scz == 4;
}

struct AdvLayout {
    int tx, ty, tz, TV, jx, jy, jz, JV;
    size_t off_jt, off_qf, off_qi, off_arr, off_pf, off_wrap, off_wb, off_ws, bytes;
};

// per-particle values prefetched into shared memory: the 7 input arrays, or
// (split path) 3 old offsets, 3 new offsets, 3 new momenta, weight, carries
template <bool SPLIT>
constexpr int kPf = SPLIT ? 11 : 7;

template <typename F, int ORDER, int NS = 1, bool SPLIT = false>
__host__ __device__ inline AdvLayout adv_layout(int scx, int scy, int scz) {
    constexpr int H = Shape<ORDER>::H;
    AdvLayout L;
    L.tx = scx + 2; L.ty = scy + 2; L.tz = scz + 2; L.TV = L.tx * L.ty * L.tz;
    L.jx = scx + 2 * H; L.jy = scy + 2 * H; L.jz = scz + 2 * H; L.JV = L.jx * L.jy * L.jz;
    using C = AdvCfg<F, ORDER>;
    size_t o = SPLIT ? 0 : (size_t)6 * L.TV * sizeof(typename C::EB);   // split: no E/B tile
    o = (o + 127) & ~size_t(127);   // TMA source/destination: 128-byte aligned
    L.off_jt = o;
    o += (size_t)3 * L.JV * sizeof(F);
    o = (o + 127) & ~size_t(127);
    L.off_qf = o;
    o += (size_t)7 * kWarps * C::kQ * sizeof(F);
    L.off_qi = o;
    o += (size_t)kWarps * C::kQ * sizeof(int);
    L.off_arr = o;
    o += (size_t)NS * kMaxCells * sizeof(int);   // in-super-cell arrivals per species
    L.off_pf = o;
    o += (size_t)2 * kPf<SPLIT> * kMaxCells * sizeof(F);   // double-buffered next-particle records
    L.off_wrap = o;
    o += (size_t)(L.tx + L.ty + L.tz + L.jx + L.jy + L.jz) * sizeof(int);
    o = (o + 15) & ~size_t(15);
    L.off_wb = o;
    if (pcs_box_layout<F, ORDER>(scx, scy, scz)) o += (size_t)kWarps * kBoxFloats * sizeof(F);
    o = (o + 15) & ~size_t(15);
    L.off_ws = o;
#ifdef KWB_WIN_SMEM
    if (sizeof(F) == 4 && ORDER != 3) o += (size_t)7 * kMaxCells * sizeof(float4);
#endif
    L.bytes = (o + 15) & ~size_t(15);
    return L;
}

// Trilinear sample of one staged (float64) component, pic/kernels.py:26-47.
// Tile origin = super-cell origin - 1.  The floor/fraction of an axis is
// shared by every component with the same stagger on that axis (CSE).
// All eight corner loads are issued before the arithmetic (measured: the
// compiler then overlaps them with the other components' math).
// Floor-free form of the same sample, bit for bit: the particle sits in
// cell c with px = RN(c + o), o in [0, 1], so t = px - s (s = 1/2 or 1) lies
// in [c - 1, c + 1) and floor(t) = (t >= c ? c : c - 1) -- one compare and a
// select of the precomputed doubles c, c - 1 replace F2I/I2F, and the tile
// index is the lane's base plus the 0/1 carries.  f = t - floor(t) is the
// reference's exact difference.  Computed once per (axis, stagger) pair and
// shared by the components.
struct AxFrac {
    double f;
    int h;
};
__device__ __forceinline__ AxFrac ax_frac(double p, double s, double c, double cm1) {
    const double t = p - s;
    const bool h = t >= c;
    return AxFrac{t - (h ? c : cm1), h ? 1 : 0};
}
template <int C, typename TT>
__device__ __forceinline__ double sample_sel(const TT *__restrict__ T, const AxFrac (&ax)[3][2],
                                             int base, int tx, int txy, int TV) {
    const AxFrac &X = ax[0][stagger(C, 0) == 1.0], &Y = ax[1][stagger(C, 1) == 1.0],
                 &Z = ax[2][stagger(C, 2) == 1.0];
    const double fx = X.f, fy = Y.f, fz = Z.f;
    const int i00 = base + Z.h * txy + Y.h * tx + X.h;
#ifdef KWB_CHECKS
    // the tile holds (sc + 2)^3 points per component; the far corner is
    // i00 + txy + tx + 1 (T points at component C's tile)
    if (!KWB_IN(i00 >= 0 && i00 + txy + tx + 1 < TV)) return 0.0;
#else
    (void)TV;
#endif
    const TT *r00 = T + i00, *r10 = r00 + tx, *r01 = r00 + txy,
             *r11 = r01 + tx;
    const double a00 = r00[0], b00 = r00[1], a10 = r10[0], b10 = r10[1];   // (x, x+1) corners
    const double a01 = r01[0], b01 = r01[1], a11 = r11[0], b11 = r11[1];
    const double gx = 1.0 - fx;
    const double c00 = a00 * gx + b00 * fx;
    const double c10 = a10 * gx + b10 * fx;
    const double c01 = a01 * gx + b01 * fx;
    const double c11 = a11 * gx + b11 * fx;
    return (c00 * (1.0 - fy) + c10 * fy) * (1.0 - fz) + (c01 * (1.0 - fy) + c11 * fy) * fz;
}

// The six gathered components of one particle from the staged float64 tile
// (pic/kernels.py:53-77): floor-free trilinear samples, rounded to F.
template <typename F, typename EB>
__device__ __forceinline__ void gather6(const EB *__restrict__ ebd, int TV, int tx, int txy,
                                        int tbase, double px, double py, double pz, double cxd,
                                        double cyd, double czd, F &e0, F &e1, F &e2, F &b0, F &b1,
                                        F &b2) {
    const AxFrac ax[3][2] = {{ax_frac(px, 0.5, cxd, cxd - 1.0), ax_frac(px, 1.0, cxd, cxd - 1.0)},
                             {ax_frac(py, 0.5, cyd, cyd - 1.0), ax_frac(py, 1.0, cyd, cyd - 1.0)},
                             {ax_frac(pz, 0.5, czd, czd - 1.0), ax_frac(pz, 1.0, czd, czd - 1.0)}};
    e0 = (F)sample_sel<0>(ebd, ax, tbase, tx, txy, TV);
    e1 = (F)sample_sel<1>(ebd + TV, ax, tbase, tx, txy, TV);
    e2 = (F)sample_sel<2>(ebd + 2 * TV, ax, tbase, tx, txy, TV);
    b0 = (F)sample_sel<3>(ebd + 3 * TV, ax, tbase, tx, txy, TV);
    b1 = (F)sample_sel<4>(ebd + 4 * TV, ax, tbase, tx, txy, TV);
    b2 = (F)sample_sel<5>(ebd + 5 * TV, ax, tbase, tx, txy, TV);
}

// Carries of the move packed for the split path's deposit kernel (4 bits
// each, biased by 8; a carry outside -8..7 is clamped -- any |carry| > 1 is
// a ContractViolation there).
__device__ __forceinline__ int pack_carries(int dx, int dy, int dz) {
    dx = min(max(dx, -8), 7);
    dy = min(max(dy, -8), 7);
    dz = min(max(dz, -8), 7);
    return (dx + 8) | ((dy + 8) << 4) | ((dz + 8) << 8);
}
__device__ __forceinline__ void unpack_carries(int code, int &dx, int &dy, int &dz) {
    dx = (code & 15) - 8;
    dy = ((code >> 4) & 15) - 8;
    dz = ((code >> 8) & 15) - 8;
}

// Boris push (pic/kernels.py:80-104) and move (:107-135) of one particle,
// bit for bit the reference: float64 without contraction, the three
// quotients by one divisor through one reciprocal (div_rcp), gamma of the
// move from storage-type squares, offsets rounded to F (1.0 kept).  Returns
// the new momentum, the new offsets and the floor carries of the move.
template <typename F>
__device__ __forceinline__ void push_move(double qm, const double (&dt_d)[3], F e0, F e1, F e2,
                                          F b0, F b1, F b2, F ox, F oy, F oz, F ux, F uy, F uz,
                                          F &nux, F &nuy, F &nuz, F &nox, F &noy, F &noz,
                                          int &dxi, int &dyi, int &dzi) {
    const double qe0 = qm * (double)e0, qe1 = qm * (double)e1, qe2 = qm * (double)e2;
    const double umx = (double)ux + qe0;
    const double umy = (double)uy + qe1;
    const double umz = (double)uz + qe2;
    const double gm = sqrt(((1.0 + umx * umx) + umy * umy) + umz * umz);
    const double rgm = 1.0 / gm;
    const double ttx = div_rcp(qm * (double)b0, gm, rgm);
    const double tty = div_rcp(qm * (double)b1, gm, rgm);
    const double ttz = div_rcp(qm * (double)b2, gm, rgm);
    const double tsq1 = 1.0 + ((ttx * ttx + tty * tty) + ttz * ttz);
    const double rts = 1.0 / tsq1;
    const double ssx = div_rcp(2.0 * ttx, tsq1, rts);
    const double ssy = div_rcp(2.0 * tty, tsq1, rts);
    const double ssz = div_rcp(2.0 * ttz, tsq1, rts);
    const double upx = umx + (umy * ttz - umz * tty);
    const double upy = umy + (umz * ttx - umx * ttz);
    const double upz = umz + (umx * tty - umy * ttx);
    nux = (F)((umx + (upy * ssz - upz * ssy)) + qe0);
    nuy = (F)((umy + (upz * ssx - upx * ssz)) + qe1);
    nuz = (F)((umz + (upx * ssy - upy * ssx)) + qe2);
    // move: gamma from F squares
    const F sxx = nux * nux, syy = nuy * nuy, szz = nuz * nuz;
    const double gv = sqrt(((1.0 + (double)sxx) + (double)syy) + (double)szz);
    const double rgv = 1.0 / gv;
    const double mpx = (double)ox + div_rcp((double)nux, gv, rgv) * dt_d[0];
    const double mpy = (double)oy + div_rcp((double)nuy, gv, rgv) * dt_d[1];
    const double mpz = (double)oz + div_rcp((double)nuz, gv, rgv) * dt_d[2];
    dxi = (int)floor(mpx);
    dyi = (int)floor(mpy);
    dzi = (int)floor(mpz);
    nox = (F)(mpx - (double)dxi);
    noy = (F)(mpy - (double)dyi);
    noz = (F)(mpz - (double)dzi);
}

template <int C, typename TT>
__device__ __forceinline__ double sample_tile(const TT *__restrict__ T, double px, double py,
                                              double pz, int ox0, int oy0, int oz0, int tx,
                                              int txy) {
    const double ttx = px - stagger(C, 0), tty = py - stagger(C, 1), ttz = pz - stagger(C, 2);
    const int ix = (int)floor(ttx), iy = (int)floor(tty), iz = (int)floor(ttz);
    const double fx = ttx - (double)ix, fy = tty - (double)iy, fz = ttz - (double)iz;
    const int i00 = (iz - oz0) * txy + (iy - oy0) * tx + (ix - ox0);
    const TT *r00 = T + i00, *r10 = r00 + tx, *r01 = r00 + txy, *r11 = r01 + tx;
    const double a00 = r00[0], b00 = r00[1], a10 = r10[0], b10 = r10[1];   // (x, x+1) corners
    const double a01 = r01[0], b01 = r01[1], a11 = r11[0], b11 = r11[1];
    const double gx = 1.0 - fx;
    const double c00 = a00 * gx + b00 * fx;
    const double c10 = a10 * gx + b10 * fx;
    const double c01 = a01 * gx + b01 * fx;
    const double c11 = a11 * gx + b11 * fx;
    return (c00 * (1.0 - fy) + c10 * fy) * (1.0 - fz) + (c01 * (1.0 - fy) + c11 * fy) * fz;
}

// Deposit of a queued PCS particle into the shared J tile (PCS queues every
// particle: 300 entries do not fit registers).  Per axis the anchor is
// min(old cell, new cell), so old and new positions lie in [0, 2] and every
// support fits indices 1..NS; the along-axis running sum runs from the
// reference's lo to its min(hi, NP - 2) -- NA entries, NA + 1 when the
// particle moved down (pic/kernels.py:204-209, 221): its last entry is the
// "closing" sum(s1) - sum(s0) unless the particle moved up, and it is kept
// (a rounding residue of the F weights, but the reference deposits it and
// without it f32 J misses the 1e-6 bar).  The running sums are exact
// (double) so the residue is too.  Same density decomposition and
// transverse factor as pic/kernels.py:210-248
// (factorised: T = (s0 + ds/2)_1 s0_2 + (s0/2 + ds/3)_1 ds_2); shared float
// atomics are CAS loops on sm_100a.  The component and transverse-row loops are NOT unrolled
// -- the per-axis register arrays are rotated instead, so every index stays
// a compile-time constant (no local memory) while the code is ~NS x NA CAS
// sites instead of 3 x NS x NS x NA (the unrolled PCS routine is ~90 KB of
// SASS and stalls on instruction fetch).  Same arithmetic and order.
template <typename F, int ORDER>
__device__ __noinline__ void deposit_cross_compact(F *__restrict__ jt, int jx, int jy, int JV,
                                                   int lx, int ly, int lz, int dcx, int dcy,
                                                   int dcz, F oox, F ooy, F ooz, F nox, F noy,
                                                   F noz, F w, double fac0, double fac1,
                                                   double fac2) {
    using CT = F;
    constexpr int NP = Shape<ORDER>::NP, NS = NP - 1, NA = NP - 2;
    const int dc[3] = {dcx, dcy, dcz};
    const F oo[3] = {oox, ooy, ooz}, no[3] = {nox, noy, noz};
    const double fac[3] = {fac0, fac1, fac2};
    CT s0[3][NS], ds[3][NS], P[3][NS];
    int nt[3], na[3], st[3] = {1, jx, jx * jy};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int m = dc[a] < 0 ? -1 : 0;
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            CT s1;
            wpair<ORDER, CT>(oo[a], no[a], dc[a], m, i, s0[a][i], s1);
            ds[a][i] = s1 - s0[a][i];
        }
        nt[a] = dc[a] != 0 ? NS : NS - 1;
        na[a] = NA - m;
        const double fw = fac[a] * (double)w;
        double run = 0.0;
#pragma unroll
        for (int i = 0; i < NS; ++i) { run += (double)ds[a][i]; P[a][i] = (CT)(fw * run); }
    }
    const int ax = lx + min(dcx, 0), ay = ly + min(dcy, 0), az = lz + min(dcz, 0);
    F *Jc = jt + (az * jy + ay) * jx + ax;
    // invariant: slot 0 = the component's axis, 1 = first transverse, 2 = second
#pragma unroll 1
    for (int c = 0; c < 3; ++c) {
        CT u1[NS], v1[NS];
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            u1[j] = s0[1][j] + CT(0.5) * ds[1][j];
            v1[j] = CT(0.5) * s0[1][j] + ds[1][j] * CT(1.0 / 3.0);
        }
        const int sa = st[0], s1_ = st[1], s2_ = st[2], nt1 = nt[1], nt2 = nt[2], nac = na[0];
        F *row = Jc + s1_;
#pragma unroll 1
        for (int j1 = 0; j1 < nt1; ++j1) {
            const CT uu = u1[0], vv = v1[0];
#pragma unroll
            for (int j2 = 0; j2 < NS; ++j2) {
                if (j2 < nt2) {
                    const CT T = uu * s0[2][j2] + vv * ds[2][j2];
                    if (T != CT(0)) {
                        F *q = row + (j2 + 1) * s2_;
#pragma unroll
                        for (int ja = 0; ja < NS; ++ja) {
                            const CT val = P[0][ja] * T;
                            F *dst = q + (ja + 1) * sa;
                            if (ja < nac && val != CT(0) && KWB_IN(dst >= jt && dst < jt + 3 * JV))
                                atomicAdd(dst, (F)val);
                        }
                    }
                }
            }
#pragma unroll
            for (int j = 0; j + 1 < NS; ++j) { u1[j] = u1[j + 1]; v1[j] = v1[j + 1]; }
            row += s1_;
        }
        Jc += JV;
        // rotate the axes: (c, c+1, c+2) -> (c+1, c+2, c+3)
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            const CT a0 = s0[0][j], b0 = ds[0][j], p0 = P[0][j];
            s0[0][j] = s0[1][j]; s0[1][j] = s0[2][j]; s0[2][j] = a0;
            ds[0][j] = ds[1][j]; ds[1][j] = ds[2][j]; ds[2][j] = b0;
            P[0][j] = P[1][j]; P[1][j] = P[2][j]; P[2][j] = p0;
        }
        { const int t0 = nt[0]; nt[0] = nt[1]; nt[1] = nt[2]; nt[2] = t0; }
        { const int t0 = na[0]; na[0] = na[1]; na[1] = na[2]; na[2] = t0; }
        { const int t0 = st[0]; st[0] = st[1]; st[1] = st[2]; st[2] = t0; }
    }
}

// Warp-cooperative form of deposit_cross, for the rare particles that cross
// faces on more than one axis in the register-deposit kernels: all 32
// lanes take the same record.  Lanes 0..3*NS-1 evaluate one support point
// (axis a, index i) each -- s0, ds, the transverse factors u, v and the
// along-axis running sum P (segmented shuffle scan) -- and the footprint
// entries (component c, along ja, transverse j1, j2) are then dealt out 32
// per pass, each lane fetching its operands by shuffle and issuing one CAS.
// Distinct lanes hit distinct entries, the code is a few hundred bytes (the
// fully unrolled per-lane PCS routine is ~90 KB and thrashes the instruction
// cache) and every lane is busy.  Same arithmetic as deposit_cross_compact
// up to the summation order of P (J is compared within tolerance).
// Entries inside the owner's register window (deposit_window: own-relative
// edges -1..+1 for float32; -1..0, and +1 where it is the closing residue,
// for float64) are skipped.
template <typename F, int ORDER>
__device__ __noinline__ void deposit_warp(F *__restrict__ jt, int jx, int jy, int JV, int lane,
                                          int lx, int ly, int lz, int dcx, int dcy, int dcz,
                                          F oox, F ooy, F ooz, F nox, F noy, F noz, F w,
                                          double fac0, double fac1, double fac2,
                                          bool skip_window) {
    using CT = F;
    constexpr int NP = Shape<ORDER>::NP, NS = NP - 1, NA = NP - 2;
    constexpr bool PLUS = sizeof(F) == 4;
    constexpr unsigned FULL = 0xffffffffu;
    // this lane's support point
    const int a = lane / NS, i = lane - a * NS;
    const int dca = a == 0 ? dcx : a == 1 ? dcy : dcz;
    const F ooa = a == 0 ? oox : a == 1 ? ooy : ooz;
    const F noa = a == 0 ? nox : a == 1 ? noy : noz;
    const double faca = a == 0 ? fac0 : a == 1 ? fac1 : fac2;
    const int m = dca < 0 ? -1 : 0;
    CT s0, s1;
    wpair<ORDER, CT>(ooa, noa, dca, m, i, s0, s1);
    const CT ds = s1 - s0;
    const CT u = s0 + CT(0.5) * ds, v = CT(0.5) * s0 + ds * CT(1.0 / 3.0);
    double run = (double)ds;   // exact, so the closing residue is too
#pragma unroll
    for (int o = 1; o < NS; o <<= 1) {
        const double y = __shfl_up_sync(FULL, run, o);
        if (i >= o) run += y;
    }
    const CT P = (CT)(faca * (double)w * run);
    const int ntx = dcx ? NS : NS - 1, nty = dcy ? NS : NS - 1, ntz = dcz ? NS : NS - 1;
    const int ax = lx + min(dcx, 0), ay = ly + min(dcy, 0), az = lz + min(dcz, 0);
    F *base = jt + (az * jy + ay) * jx + ax;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int a1 = (c + 1) % 3, a2 = (c + 2) % 3;
        const int dcc = c == 0 ? dcx : c == 1 ? dcy : dcz;
        const int nt1 = a1 == 0 ? ntx : a1 == 1 ? nty : ntz;
        const int nt2 = a2 == 0 ? ntx : a2 == 1 ? nty : ntz;
        const int na = dcc < 0 ? NA + 1 : NA;   // up to the reference's min(hi, NP - 2)
        const int per_a = nt1 * nt2, npts = na * per_a;
        // x / d for x < 2^10, d <= 64 (exact): multiply by ceil(2^16 / d)
        const unsigned r_pa = 65536u / per_a + 1u, r_n2 = 65536u / nt2 + 1u;
        const int ehi = (PLUS || dcc <= 0) ? 1 : 0;   // window's top edge
        F *Jc = base + c * JV;
        for (int p0 = 0; p0 < npts; p0 += 32) {   // warp-uniform passes
            const int p = p0 + lane;
            const int ja = (int)(((unsigned)p * r_pa) >> 16);
            const int rem = p - ja * per_a;
            const int j1 = (int)(((unsigned)rem * r_n2) >> 16), j2 = rem - j1 * nt2;
            const CT u1 = __shfl_sync(FULL, u, a1 * NS + j1);
            const CT v1 = __shfl_sync(FULL, v, a1 * NS + j1);
            const CT s02 = __shfl_sync(FULL, s0, a2 * NS + j2);
            const CT ds2 = __shfl_sync(FULL, ds, a2 * NS + j2);
            const CT Pv = __shfl_sync(FULL, P, c * NS + ja);
            // entries of the owner cell's register window (anchor-relative
            // index j <-> own-relative j - 1 + m) were already added by
            // deposit_window
            const int mc = dcc < 0 ? -1 : 0;
            const int m1 = (a1 == 0 ? dcx : a1 == 1 ? dcy : dcz) < 0 ? -1 : 0;
            const int m2 = (a2 == 0 ? dcx : a2 == 1 ? dcy : dcz) < 0 ? -1 : 0;
            const int e = ja - 1 + mc, p1 = j1 - 1 + m1, p2 = j2 - 1 + m2;
            const bool inside = e >= -1 && e <= ehi && p1 >= -1 && p1 <= 1 && p2 >= -1 && p2 <= 1;
            if (p < npts && !(skip_window && inside)) {
                const CT T = u1 * s02 + v1 * ds2;
                const CT val = Pv * T;
                if (T != CT(0) && val != CT(0)) {
                    int o;
                    if (c == 0) o = ((j2 + 1) * jy + (j1 + 1)) * jx + (ja + 1);
                    else if (c == 1) o = ((j1 + 1) * jy + (ja + 1)) * jx + (j2 + 1);
                    else o = ((ja + 1) * jy + (j2 + 1)) * jx + (j1 + 1);
                    if (KWB_IN(Jc + o >= jt && Jc + o < jt + 3 * JV)) atomicAdd(Jc + o, (F)val);
                }
            }
        }
    }
}

// Deposit of a particle that crossed exactly one cell face, along axis k
// (the common case: a two-axis crossing is ~40x rarer) -- the part of its
// footprint OUTSIDE the owner cell's register window (deposit_window adds
// the rest in registers).  Axes are rotated so the crossing axis is A0; with
// the anchor min(old, new) its supports span indices 1..4, the other axes
// 1..3; the full footprint (pic/kernels.py:204-248, closing entries kept) is
//   J_A0: along 1..3 (+k) / 0..3 (-k) x (A1: 1..3) x (A2: 1..3)
//   J_A1: along 1..3 x (A0: 1..4) x (A2: 1..3)  = 36 entries
//   J_A2: along 1..3 x (A0: 1..4) x (A1: 1..3)  = 36 entries
// The float32 window holds own-relative edges -1..+1 x points -1..1, so this
// adds J_A0's edge -2 (-k only) and the A0 point outside the window of
// J_A1 / J_A2 (3 edges x 3): 18 (+k) or 27 (-k) CAS.  The float64 window
// holds edge +1 only as the closing residue (dc <= 0), so for +k J_A0's
// edge +1 (a real entry) comes here too.
// (the transverse factor is symmetric in its two axes, so the reference's
// per-component axis order does not matter).  TSC/CIC only.
template <typename F, int ORDER>
__device__ __noinline__ void deposit_cross1(F *__restrict__ jt, int jx, int jy, int JV, int k,
                                            int lx, int ly, int lz, int dck, F oox, F ooy,
                                            F ooz, F nox, F noy, F noz, F w, double fac0,
                                            double fac1, double fac2) {
    using CT = F;
    constexpr bool PLUS = sizeof(F) == 4;
    const int a1 = k == 2 ? 0 : k + 1, a2 = k == 0 ? 2 : k - 1;
    const F oo[3] = {oox, ooy, ooz}, no[3] = {nox, noy, noz};
    const double fac[3] = {fac0, fac1, fac2};
    const int st[3] = {1, jx, jx * jy};
    const int m = dck < 0 ? -1 : 0;
    CT s0c[4], dsc[4], s0p[3], dsp[3], s0q[3], dsq[3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        CT t1;
        wpair<ORDER, CT>(oo[k], no[k], dck, m, i, s0c[i], t1);
        dsc[i] = t1 - s0c[i];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        CT t1;
        wpair<ORDER, CT>(oo[a1], no[a1], 0, 0, i, s0p[i], t1);
        dsp[i] = t1 - s0p[i];
        wpair<ORDER, CT>(oo[a2], no[a2], 0, 0, i, s0q[i], t1);
        dsq[i] = t1 - s0q[i];
    }
    const int lc[3] = {lx, ly, lz};
    F *base = jt + (lc[2] + (k == 2 ? m : 0)) * st[2] + (lc[1] + (k == 1 ? m : 0)) * st[1] +
              (lc[0] + (k == 0 ? m : 0));
    const int sk = st[k], s1_ = st[a1], s2_ = st[a2];
    // J_k: along k x a1 (1..3) x a2 (1..3), the edge outside the window:
    // -k -> own edge -2 (anchor index 0); +k -> own edge +1 (float64 only)
    if (!PLUS || m != 0) {
        F *J = base + k * JV;
        const CT fw = (CT)(fac[k] * (double)w);
        const int ja = m == 0 ? 2 : 0;
        const CT Pout = m == 0 ? fw * ((dsc[0] + dsc[1]) + dsc[2]) : fw * dsc[0];
#pragma unroll
        for (int j1 = 0; j1 < 3; ++j1) {
            const CT u = s0p[j1] + CT(0.5) * dsp[j1], v = CT(0.5) * s0p[j1] + dsp[j1] * CT(1.0 / 3.0);
#pragma unroll
            for (int j2 = 0; j2 < 3; ++j2) {
                const CT T = u * s0q[j2] + v * dsq[j2];
                F *dst = J + (j1 + 1) * s1_ + (j2 + 1) * s2_ + (ja + 1) * sk;
                if (KWB_IN(dst >= jt && dst < jt + 3 * JV)) atomicAdd(dst, (F)(Pout * T));
            }
        }
    }
    // J_a1: along a1 (1..3) x k (1..4) x a2 (1..3);  J_a2: along a2 (1..3) x k x a1
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int c = h == 0 ? a1 : a2;
        const CT *s0a = h == 0 ? s0p : s0q, *dsa = h == 0 ? dsp : dsq;   // along
        const CT *s0o = h == 0 ? s0q : s0p, *dso = h == 0 ? dsq : dsp;   // the other transverse
        const int sa = h == 0 ? s1_ : s2_, so = h == 0 ? s2_ : s1_;
        F *J = base + c * JV;
        const double fwd = fac[c] * (double)w;
        const CT fw = (CT)fwd;
        const CT P0 = fw * dsa[0], P1 = fw * (dsa[0] + dsa[1]);
        // the closing residue, from the exact sum
        const CT P2 = (CT)(fwd * (((double)dsa[0] + (double)dsa[1]) + (double)dsa[2]));
        // only the point along k outside the owner's window: +k -> 4, -k -> 1
        const int j1 = m == 0 ? 3 : 0;
        const CT s0j = m == 0 ? s0c[3] : s0c[0], dsj = m == 0 ? dsc[3] : dsc[0];
        const CT u = s0j + CT(0.5) * dsj, v = CT(0.5) * s0j + dsj * CT(1.0 / 3.0);
#pragma unroll
        for (int j2 = 0; j2 < 3; ++j2) {
            const CT T = u * s0o[j2] + v * dso[j2];
            F *p = J + (j1 + 1) * sk + (j2 + 1) * so;
            if (KWB_IN(p + sa >= jt && p + 3 * sa < jt + 3 * JV)) {
                atomicAdd(p + sa, (F)(P0 * T));
                atomicAdd(p + 2 * sa, (F)(P1 * T));
                atomicAdd(p + 3 * sa, (F)(P2 * T));
            }
        }
    }
}

// The register window of the owner cell (every particle, crossing or not):
// J accumulators at own-relative edges -1, 0, +1 along a component x points
// -1..1 across it, in registers -- 81 per thread (float32).  Entry (edge e,
// j1, j2) of component a gets P_e T(j1, j2): P_e = fw_a x the running sum
// of ds_a from the reference's lo to point e (pic/kernels.py:204-222), and
// T = (s0 + ds/2)_1 s0_2 + (s0/2 + ds/3)_1 ds_2 (the reference's transverse
// factor :215-218, factorised), in fp32 with FMA -- J is compared within
// tolerance (the reference's own J order is not fixed).  Edge +1 is the
// closing entry sum(s1) - sum(s0) for dc_a <= 0 -- a rounding residue of
// the F weights that the reference deposits, and at thermal speeds ~1e-6 of
// J -- so its running sum is formed exactly in double.  A particle that
// moved dc in {-1,0,1} on an axis has its new shape on points dc-1..dc+1:
// the window sees it shifted (zero filled), and for dc = -1 the running sum
// starts one point earlier (ds at point -2).  The entries of a crosser
// outside the window go through the queue (deposit_cross1 / deposit_warp).
// (edge -1, edge 0) of an entry share T: one packed FFMA2 (__ffma2_rn,
// sm_100) updates both -- the same two round-to-nearest FMAs; edge +1 pairs
// the j1 = 0, 1 entries.
struct RegAcc {
    float2 p[3][3][3];  // [component][j1][j2] = {edge -1, edge 0}
    float2 q[3][3];     // [component][j2] = edge +1 at {j1 = 0, j1 = 1}  (unused with
    float r[3][3];      // [component][j2] = edge +1 at j1 = 2             KWB_WIN_SMEM)
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
#pragma unroll
                for (int d = 0; d < 3; ++d) p[c][b][d] = make_float2(0.f, 0.f);
                q[c][b] = make_float2(0.f, 0.f);
                r[c][b] = 0.f;
            }
    }
    // e: 0, 1, 2 = edge -1, 0, +1
    __device__ __forceinline__ float get(int c, int e, int b, int d) const {
        return e == 0 ? p[c][b][d].x
             : e == 1 ? p[c][b][d].y
             : (b == 0 ? q[c][d].x : b == 1 ? q[c][d].y : r[c][d]);
    }
    __device__ __forceinline__ static float2 pack(float lo, float hi) { return make_float2(lo, hi); }
    __device__ __forceinline__ void fma2(int c, int b, int d, float2 P, float T) {
        p[c][b][d] = __ffma2_rn(P, make_float2(T, T), p[c][b][d]);
    }
};

// Per-thread shared-memory copy of the edge +1 accumulators (KWB_WIN_SMEM):
// float4 k of thread t at ws[k * kMaxCells + t]; component c in float4s
// 2c, 2c+1 (q[c][0..2], r[c][0..1]) and lane c of float4 6 (r[c][2]).
__device__ __forceinline__ void win_load(const float4 *ws, float2 (&q)[3][3], float (&r)[3][3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float4 A = ws[(2 * c) * kMaxCells], B = ws[(2 * c + 1) * kMaxCells];
        q[c][0] = make_float2(A.x, A.y); q[c][1] = make_float2(A.z, A.w);
        q[c][2] = make_float2(B.x, B.y); r[c][0] = B.z; r[c][1] = B.w;
    }
    const float4 C = ws[6 * kMaxCells];
    r[0][2] = C.x; r[1][2] = C.y; r[2][2] = C.z;
}
__device__ __forceinline__ void win_store(float4 *ws, const float2 (&q)[3][3], const float (&r)[3][3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        ws[(2 * c) * kMaxCells] = make_float4(q[c][0].x, q[c][0].y, q[c][1].x, q[c][1].y);
        ws[(2 * c + 1) * kMaxCells] = make_float4(q[c][2].x, q[c][2].y, r[c][0], r[c][1]);
    }
    ws[6 * kMaxCells] = make_float4(r[0][2], r[1][2], r[2][2], 0.0f);
}

// The old position's weights of the three axes (they depend on the
// particle's input offsets only; KWB_EARLY_S0 computes them at the top of
// the loop body, off the push/move dependency chain).
template <int ORDER>
__device__ __forceinline__ void old_weights(float oox, float ooy, float ooz, float (&s0)[3][3]) {
    wref3<ORDER, float>((double)oox, 0.0, s0[0]);
    wref3<ORDER, float>((double)ooy, 0.0, s0[1]);
    wref3<ORDER, float>((double)ooz, 0.0, s0[2]);
}

template <int ORDER>
__device__ __forceinline__ void deposit_window(RegAcc &R, float4 *ws, const float (&s0in)[3][3],
                                               float nox, float noy, float noz,
                                               float fwx, float fwy, float fwz, int dcx, int dcy,
                                               int dcz) {
#ifdef KWB_WIN_SMEM
    float2 Q[3][3];
    float Rr[3][3];
    win_load(ws, Q, Rr);
#else
    float2 (&Q)[3][3] = R.q;
    float (&Rr)[3][3] = R.r;
#endif
    float s0[3][3], ds[3][3], dm2[3], rs[3];
    {
        const float no[3] = {nox, noy, noz};
        const int dc[3] = {dcx, dcy, dcz};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float s1[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) s0[a][k] = s0in[a][k];
            const double c = (double)dc[a];
            wref3<ORDER, float>(c + (double)no[a], c, s1);   // own points dc-1 .. dc+1
            const float w0 = dc[a] == 0 ? s1[0] : (dc[a] > 0 ? 0.0f : s1[1]);
            const float w1 = dc[a] == 0 ? s1[1] : (dc[a] > 0 ? s1[0] : s1[2]);
            const float w2 = dc[a] == 0 ? s1[2] : (dc[a] > 0 ? s1[1] : 0.0f);
            dm2[a] = dc[a] < 0 ? s1[0] : 0.0f;
            ds[a][0] = __fsub_rn(w0, s0[a][0]);
            ds[a][1] = __fsub_rn(w1, s0[a][1]);
            ds[a][2] = __fsub_rn(w2, s0[a][2]);
            rs[a] = (float)((((double)dm2[a] + (double)ds[a][0]) + (double)ds[a][1]) +
                            (double)ds[a][2]);
        }
    }
    const float fw[3] = {fwx, fwy, fwz};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int a1 = (c + 1) % 3, a2 = (c + 2) % 3;  // transverse axes: x:(y,z) y:(z,x) z:(x,y)
        const float r1 = __fadd_rn(dm2[c], ds[c][0]);
        const float p1 = __fmul_rn(fw[c], r1);
        const float p2 = __fmul_rn(fw[c], __fadd_rn(r1, ds[c][1]));
        const float p3 = __fmul_rn(fw[c], rs[c]);
        const auto P12 = RegAcc::pack(p1, p2);
        const auto P33 = RegAcc::pack(p3, p3);
        // T for j1 = 0, 1 as one f32x2 pair (same roundings), j1 = 2 scalar
        const auto U01 = RegAcc::pack(__fmaf_rn(0.5f, ds[a1][0], s0[a1][0]),
                                      __fmaf_rn(0.5f, ds[a1][1], s0[a1][1]));
        const auto V01 = RegAcc::pack(
            __fmaf_rn(1.0f / 3.0f, ds[a1][0], __fmul_rn(0.5f, s0[a1][0])),
            __fmaf_rn(1.0f / 3.0f, ds[a1][1], __fmul_rn(0.5f, s0[a1][1])));
        const float u2 = __fmaf_rn(0.5f, ds[a1][2], s0[a1][2]);
        const float v2 = __fmaf_rn(1.0f / 3.0f, ds[a1][2], __fmul_rn(0.5f, s0[a1][2]));
#pragma unroll
        for (int j2 = 0; j2 < 3; ++j2) {
            const float2 vd = __fmul2_rn(V01, make_float2(ds[a2][j2], ds[a2][j2]));
            const float2 T01 = __ffma2_rn(U01, make_float2(s0[a2][j2], s0[a2][j2]), vd);
            const float T2 = __fmaf_rn(u2, s0[a2][j2], __fmul_rn(v2, ds[a2][j2]));
            R.fma2(c, 0, j2, P12, T01.x);
            R.fma2(c, 1, j2, P12, T01.y);
            R.fma2(c, 2, j2, P12, T2);
            Q[c][j2] = __ffma2_rn(P33, T01, Q[c][j2]);
            Rr[c][j2] = __fmaf_rn(p3, T2, Rr[c][j2]);
        }
    }
#ifdef KWB_WIN_SMEM
    win_store(ws, Q, Rr);
#endif
}

// float64 storage: the same window in double for edges -1 and 0 (108
// registers of accumulators, so these kernels run one CTA per SM) plus the
// closing residue of edge +1 (dc <= 0 only: for dc = +1 edge +1 is a real
// entry and goes through the queue) in float -- it is ~1e-16 of J, so
// float is far more than enough.  J in float64 is compared at 1e-13.
struct RegAccD {
    double a[3][2][3][3];  // [component][edge -1, 0][j1][j2]
    float r[3][3][3];      // [component][j1][j2] closing residue at edge +1
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    a[c][0][b][d] = 0.0;
                    a[c][1][b][d] = 0.0;
                    r[c][b][d] = 0.f;
                }
    }
    __device__ __forceinline__ double get(int c, int e, int b, int d) const {
        return e < 2 ? a[c][e][b][d] : (double)r[c][b][d];
    }
};

template <int ORDER>
__device__ __forceinline__ void deposit_window_d(RegAccD &R, double oox, double ooy, double ooz,
                                                 double nox, double noy, double noz, double fwx,
                                                 double fwy, double fwz, int dcx, int dcy,
                                                 int dcz) {
    double s0[3][3], ds[3][3], dm2[3], rs[3];
    {
        const double oo[3] = {oox, ooy, ooz}, no[3] = {nox, noy, noz};
        const int dc[3] = {dcx, dcy, dcz};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            double s1[3];
            wref3<ORDER, double>(oo[a], 0.0, s0[a]);
            const double c = (double)dc[a];
            wref3<ORDER, double>(c + no[a], c, s1);
            const double w0 = dc[a] == 0 ? s1[0] : (dc[a] > 0 ? 0.0 : s1[1]);
            const double w1 = dc[a] == 0 ? s1[1] : (dc[a] > 0 ? s1[0] : s1[2]);
            const double w2 = dc[a] == 0 ? s1[2] : (dc[a] > 0 ? s1[1] : 0.0);
            dm2[a] = dc[a] < 0 ? s1[0] : 0.0;
            ds[a][0] = w0 - s0[a][0];
            ds[a][1] = w1 - s0[a][1];
            ds[a][2] = w2 - s0[a][2];
            rs[a] = dc[a] <= 0 ? ((dm2[a] + ds[a][0]) + ds[a][1]) + ds[a][2] : 0.0;
        }
    }
    const double fw[3] = {fwx, fwy, fwz};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int a1 = (c + 1) % 3, a2 = (c + 2) % 3;
        const double r1 = dm2[c] + ds[c][0];
        const double p1 = fw[c] * r1;
        const double p2 = fw[c] * (r1 + ds[c][1]);
        const float p3 = (float)(fw[c] * rs[c]);
#pragma unroll
        for (int j1 = 0; j1 < 3; ++j1) {
            const double u = __fma_rn(0.5, ds[a1][j1], s0[a1][j1]);
            const double v = __fma_rn(1.0 / 3.0, ds[a1][j1], 0.5 * s0[a1][j1]);
#pragma unroll
            for (int j2 = 0; j2 < 3; ++j2) {
                const double T = __fma_rn(u, s0[a2][j2], v * ds[a2][j2]);
                R.a[c][0][j1][j2] = __fma_rn(p1, T, R.a[c][0][j1][j2]);
                R.a[c][1][j1][j2] = __fma_rn(p2, T, R.a[c][1][j1][j2]);
                R.r[c][j1][j2] = __fmaf_rn(p3, (float)T, R.r[c][j1][j2]);
            }
        }
    }
}

// Tile offset of accumulator (c, ja, j1, j2) relative to the owner cell.
__device__ __forceinline__ int regacc_offset(int c, int ja, int j1, int j2, int jx, int jy) {
    int ox, oy, oz;
    if (c == 0) { ox = ja; oy = j1; oz = j2; }
    else if (c == 1) { ox = j2; oy = ja; oz = j1; }
    else { ox = j1; oy = j2; oz = ja; }
    return (oz * jy + oy) * jx + ox;
}

// One PCS stayer per lane into the warp's boxes (see kBoxX); every lane of
// the warp calls this together (on = false: the lane adds nothing).  Same
// density decomposition and factors as deposit_cross_compact with dc = 0
// (pic/kernels.py:210-248, SURVEY.md §8c PCS), closing entries included.
// (rx, ry) = cell relative to the warp's 8 x 4 patch.  Box layout: x
// fastest, 12 x 8 x 5 per component at 0 / 480 / 960.
// One group: all loads, then all stores (entries of a group never alias
// across the warp's lanes), so the N read-add-writes overlap.
// entry i of the group gets p * T[i] (one FFMA at the read-modify-write)
template <int N>
__device__ __forceinline__ void box_group(float *b, int stride, float p, const float (&T)[N],
                                          const float *box = nullptr) {
#ifdef KWB_CHECKS
    if (box && !KWB_IN(b >= box && b + (N - 1) * stride < box + kBoxFloats)) return;
#endif
    const unsigned a = (unsigned)__cvta_generic_to_shared(b);
    float o[N];
#pragma unroll
    for (int i = 0; i < N; ++i)
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o[i]) : "r"(a + 4u * i * stride) : "memory");
#pragma unroll
    for (int i = 0; i < N; ++i)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(a + 4u * i * stride),
                     "f"(__fmaf_rn(p, T[i], o[i])) : "memory");
#ifndef KWB_EXP_NO_BOX_SYNCWARP   // negative control of the race test (tools/gpurun/r02f.sh)
    __syncwarp();   // measured: without it lanes lose updates (tests/test_gpu_dense.py)
#endif
}

// PCS weights (the reference's recipe) at own points -2..2
// of a particle at offset x in [0, 1]: the distances are x + 1.5, x + 0.5,
// |x - 0.5|, 1.5 - x, 2.5 - x, so points 0 and +-2 need one branch each.
__device__ __forceinline__ void wref5_pcs(double x, float (&s)[5]) {
    auto outer = [](double d) {   // 1 <= d: (2 - d)^3 / 6, 0 from d = 2
        const double e = 2.0 - d;
        return d < 2.0 ? div6((e * e) * e) : 0.0;
    };
    auto inner = [](double d) { return div6((4.0 - (6.0 * d) * d) + ((3.0 * d) * d) * d); };
    const double d0 = x + 1.5, d1 = x + 0.5, d2 = fabs(x - 0.5), d3 = 1.5 - x, d4 = 2.5 - x;
    s[0] = (float)outer(d0);
    s[1] = (float)(d1 < 1.0 ? inner(d1) : outer(d1));
    s[2] = (float)inner(d2);
    s[3] = (float)(d3 < 1.0 ? inner(d3) : outer(d3));
    s[4] = (float)outer(d4);
}

__device__ __forceinline__ void deposit_pcs_box(float *__restrict__ box, int rx, int ry, bool on,
                                                float oox, float ooy, float ooz, float nox,
                                                float noy, float noz, float w, double fac0,
                                                double fac1, double fac2) {
    float s0[3][5], ds[3][5], P[3][5];
    {
        // an idle lane's records may be stale bit patterns: never let them
        // reach the arithmetic (0 * NaN would poison the box)
        const float oo[3] = {on ? oox : 0.5f, on ? ooy : 0.5f, on ? ooz : 0.5f},
                    no[3] = {on ? nox : 0.5f, on ? noy : 0.5f, on ? noz : 0.5f};
        const double fac[3] = {fac0, fac1, fac2};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float a0[5], a1[5];
            wref5_pcs((double)oo[a], a0);
            wref5_pcs((double)no[a], a1);
            const double fw = on ? fac[a] * (double)w : 0.0;   // w read only when on
            double run = 0.0;
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                s0[a][i] = a0[i];
                ds[a][i] = a1[i] - a0[i];
                run += (double)ds[a][i];
                P[a][i] = (float)(fw * run);   // i = 4: the closing residue, exact
            }
        }
    }
    // Jx (along x; across y = j1, z = j2): groups over z; j1 rolled with
    // rotated copies of the y arrays
    {
        float y0[5], y1[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) { y0[j] = s0[1][j]; y1[j] = ds[1][j]; }
        float *b = box + rx + 12 * ry;
#pragma unroll 1
        for (int j1 = 0; j1 < 5; ++j1) {
            const float uu = y0[0] + 0.5f * y1[0], vv = 0.5f * y0[0] + y1[0] * (1.0f / 3.0f);
            float T[5];
#pragma unroll
            for (int j2 = 0; j2 < 5; ++j2) T[j2] = uu * s0[2][j2] + vv * ds[2][j2];
            float pa[5] = {P[0][0], P[0][1], P[0][2], P[0][3], P[0][4]};
#pragma unroll 1
            for (int ja = 0; ja < 5; ++ja) {
                box_group<5>(b + ja, 96, pa[0], T, box);
                pa[0] = pa[1]; pa[1] = pa[2]; pa[2] = pa[3]; pa[3] = pa[4];
            }
            b += 12;
#pragma unroll
            for (int j = 0; j < 4; ++j) { y0[j] = y0[j + 1]; y1[j] = y1[j + 1]; }
        }
    }
    // Jy (along y; across z = j1, x = j2): groups over z; j2 rolled with
    // rotated copies of the x arrays
    {
        float uz[5], vz[5], x0[5], x1[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            uz[j] = s0[2][j] + 0.5f * ds[2][j];
            vz[j] = 0.5f * s0[2][j] + ds[2][j] * (1.0f / 3.0f);
            x0[j] = s0[0][j]; x1[j] = ds[0][j];
        }
        float *b = box + 480 + rx + 12 * ry;
#pragma unroll 1
        for (int j2 = 0; j2 < 5; ++j2) {
            float T[5];
#pragma unroll
            for (int j1 = 0; j1 < 5; ++j1) T[j1] = uz[j1] * x0[0] + vz[j1] * x1[0];
            float pa[5] = {P[1][0], P[1][1], P[1][2], P[1][3], P[1][4]};
#pragma unroll 1
            for (int ja = 0; ja < 5; ++ja) {
                box_group<5>(b + 12 * ja, 96, pa[0], T, box);
                pa[0] = pa[1]; pa[1] = pa[2]; pa[2] = pa[3]; pa[3] = pa[4];
            }
            b += 1;
#pragma unroll
            for (int j = 0; j < 4; ++j) { x0[j] = x0[j + 1]; x1[j] = x1[j + 1]; }
        }
    }
    // Jz (along z; across x = j1, y = j2): groups over the along-z edges;
    // j1 rolled with rotated copies of the x factors
    {
        float ux[5], vx[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            ux[j] = s0[0][j] + 0.5f * ds[0][j];
            vx[j] = 0.5f * s0[0][j] + ds[0][j] * (1.0f / 3.0f);
        }
        float *b = box + 960 + rx + 12 * ry;
#pragma unroll 1
        for (int j1 = 0; j1 < 5; ++j1) {
            const float uu = ux[0], vv = vx[0];
            float y0[5], y1[5];
#pragma unroll
            for (int j = 0; j < 5; ++j) { y0[j] = s0[1][j]; y1[j] = ds[1][j]; }
#pragma unroll 1
            for (int j2 = 0; j2 < 5; ++j2) {
                const float T = uu * y0[0] + vv * y1[0];
                box_group<5>(b + 12 * j2, 96, T, P[2], box);
#pragma unroll
                for (int j = 0; j < 4; ++j) { y0[j] = y0[j + 1]; y1[j] = y1[j + 1]; }
            }
            b += 1;
#pragma unroll
            for (int j = 0; j < 4; ++j) { ux[j] = ux[j + 1]; vx[j] = vx[j + 1]; }
        }
    }
}

// ---- TMA (tensor memory accelerator) helpers -----------------------------
constexpr int TMA_EB = 1;
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *m, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *m, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *tm, int c0, int c1, int c2,
                                            int c3, uint64_t *m) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(m))
        : "memory");
}
// Lane-level species fusion (NS = 2): one launch advances both species of
// the super cell -- E/B staged once, one register window and J tile for
// both, one flush -- and each thread walks its cell's electron column and
// then its ion column in ONE loop, so a warp's trip count is the longest sum
// of the two columns instead of the sum of the two longest (Poisson
// columns: ~9 % fewer rounds).  The species of a lane's current particle
// selects its pointers and constants from a shared-memory table (a runtime
// index into the kernel parameters would copy them to local memory).
template <typename F>
struct SpeciesB {   // the second species of a fused launch
    StoreT<F> in, out;
    kwb_species sp;
    int32_t *status;
};
template <typename F>
struct SpTab {
    const F *in[7];
    F *out[7];
    int32_t *status;
    double qm, fac[3];
    int K;
};
template <typename F>
__device__ __forceinline__ void fill_tab(SpTab<F> &T, const StoreT<F> &in, const StoreT<F> &out,
                                         const kwb_species &sp, int32_t *status) {
    T.in[0] = in.ox; T.in[1] = in.oy; T.in[2] = in.oz; T.in[3] = in.ux; T.in[4] = in.uy;
    T.in[5] = in.uz; T.in[6] = in.w;
    T.out[0] = out.ox; T.out[1] = out.oy; T.out[2] = out.oz; T.out[3] = out.ux;
    T.out[4] = out.uy; T.out[5] = out.uz; T.out[6] = out.w;
    T.status = status;
    T.qm = sp.qm_half_dt;
    T.fac[0] = sp.fac[0]; T.fac[1] = sp.fac[1]; T.fac[2] = sp.fac[2];
    T.K = in.frames;
}

// SX/SY/SZ: compile-time super cell (0 = runtime, from g).
// SPLIT (NS = 1 only): the gather/push/move already ran in push_kernel
// (csrc/push.cuh), whose workspace store arrives as sb.in; this kernel only
// deposits and shifts.
template <typename F, int ORDER, bool REGACC, int SX, int SY, int SZ, int NS, bool SPLIT = false>
__global__ void __launch_bounds__(kMaxCells, AdvCfg<F, ORDER>::kMinBlocks)
advance_kernel(Geo g, kwb_species sp, StoreT<F> in, StoreT<F> out, ExchT<F> ex, FieldPtrs fp,
               int32_t *__restrict__ status, const __grid_constant__ CUtensorMap tm_eb, int tma,
               SpeciesB<F> sb, int sp0) {
    static_assert(NS == 1 || NS == 2, "one or two species per launch");
    static_assert(!SPLIT || NS == 1, "the split path advances one species per launch");
    constexpr int NPF = kPf<SPLIT>;
    constexpr int H = Shape<ORDER>::H;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ int s_maxcol, s_maxcol1;
    __shared__ __align__(8) uint64_t s_mbar;   // TMA completion of the E/B tile

    const int scx = SX ? SX : g.scx, scy = SY ? SY : g.scy, scz = SZ ? SZ : g.scz;
    const int V = scx * scy * scz;
    const AdvLayout L = adv_layout<F, ORDER, NS, SPLIT>(scx, scy, scz);
    const int K = in.frames;
    __shared__ SpTab<F> tab[NS];
    if (NS == 2) {
        if (threadIdx.x == 0) fill_tab(tab[0], in, out, sp, status);
        if (threadIdx.x == 32) fill_tab(tab[NS - 1], sb.in, sb.out, sb.sp, sb.status);
    }
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const bool owner = t < V;
    const int sc = blockIdx.x;
    const int bx = sc % g.gx, by = (sc / g.gx) % g.gy, bz = sc / (g.gx * g.gy);
    const int orgx = bx * scx, orgy = by * scy, orgz = bz * scz;

    // TMA for super cells whose E/B guard lies inside the grid (no periodic
    // wrap; the seams keep the indexed path): one elected thread loads the
    // 6-lattice E/B box (cp.async.bulk.tensor, completion on an mbarrier)
    // into the still unused queue area, and the CTA widens it into the
    // float64 tile.  kwb_particles_advance builds the tensor map when the
    // lattices are equally spaced (TMA_EB).  The box's x start must be
    // 16-byte aligned on B200 (measured: an unaligned start raises an
    // illegal-instruction fault, tools/probe/tma_probe2.cu), so it starts
    // at origin - 4 (f32) / origin - 2 (f64) instead of origin - 1.  Issued
    // first thing, so its latency overlaps the column-count loads.
    const bool interior = bx >= 1 && bx + 2 <= g.gx && by >= 1 && by + 2 <= g.gy && bz >= 1 &&
                          bz + 2 <= g.gz;
    const bool tma_eb = !SPLIT && REGACC && (tma & TMA_EB) && interior;
    constexpr int kTmaX0 = sizeof(F) == 4 ? 4 : 2;        // box x start = origin - kTmaX0
    const int boxx = (L.tx + kTmaX0 - 1 + (16 / (int)sizeof(F)) - 1) / (16 / (int)sizeof(F)) *
                     (16 / (int)sizeof(F));                // covers origin - 1 .. origin + scx
    void *eb_dst = (void *)(smem_raw + L.off_qf);
    if (tma_eb && t == 0) {
        mbar_init(&s_mbar, 1);
        fence_mbar_init();
        mbar_expect_tx(&s_mbar, (unsigned)(6 * boxx * L.ty * L.tz * sizeof(F)));
        tma_load_4d(eb_dst, &tm_eb, orgx - kTmaX0, orgy - 1, orgz - 1, 0, &s_mbar);
    }

    const int lx = t % scx, ly = (t / scx) % scy, lz = t / (scx * scy);

    using EB = typename AdvCfg<F, ORDER>::EB;
    constexpr int kQ = AdvCfg<F, ORDER>::kQ;
    EB *ebd = reinterpret_cast<EB *>(smem_raw);
    F *jt = reinterpret_cast<F *>(smem_raw + L.off_jt);
    F *q_f = reinterpret_cast<F *>(smem_raw + L.off_qf) + wid * kQ;  // this warp's queue
    int *q_info = reinterpret_cast<int *>(smem_raw + L.off_qi) + wid * kQ;
    constexpr int QS = kWarps * kQ;                                  // column stride
    int *arr = reinterpret_cast<int *>(smem_raw + L.off_arr);
    int *wtx = reinterpret_cast<int *>(smem_raw + L.off_wrap);
    int *wty = wtx + L.tx, *wtz = wty + L.ty, *wjx = wtz + L.tz, *wjy = wjx + L.jx,
        *wjz = wjy + L.jy;

    const int64_t col = (int64_t)sc * V + t;
    const int front_in = owner ? in.front[col] : 0;
    const int back_in = owner ? in.back[col] : 0;
    const int n0 = front_in + back_in;           // this cell's species-0 particles
    const int front1 = (NS == 2 && owner) ? sb.in.front[col] : 0;
    const int back1 = (NS == 2 && owner) ? sb.in.back[col] : 0;
    const int n_t = n0 + front1 + back1;         // the lane's sequence: species 0, then 1
    // empty super cell (e.g. a z-slab guard layer): nothing to stage or deposit
    if (__syncthreads_or(n_t) == 0) {
        if (tma_eb && t == 0) mbar_wait(&s_mbar, 0);   // no exit with the box in flight
        if (owner) {
            out.front[col] = 0; out.back[col] = 0;
            if (NS == 2) { sb.out.front[col] = 0; sb.out.back[col] = 0; }
        }
        return;
    }
    const int K1 = NS == 2 ? sb.in.frames : K;

    // particle i of the lane's sequence: species (i >= n0), frame slot
    auto species_of = [&](int i) -> int { return NS == 2 && i >= n0 ? 1 : 0; };
    auto slot_of = [&](int i) -> int64_t {
        const int s = species_of(i);
        const int j = s ? i - n0 : i, fr = s ? front1 : front_in, bk = s ? back1 : back_in;
        const int Ks = s ? K1 : K;
        const int k = j < fr ? j : Ks - bk + (j - fr);
        return ((int64_t)sc * Ks + k) * V + t;
    };
    // next-particle records are copied global -> shared asynchronously
    // (double buffered, this thread's slots only) and read at their uses,
    // so they occupy no registers between rounds
    F *pf = reinterpret_cast<F *>(smem_raw + L.off_pf) + t;
    auto prefetch = [&](int i) {
        if (i < n_t) {
            const int64_t q = slot_of(i);
            F *d = pf + (i & 1) * NPF * kMaxCells;
            if (SPLIT) {
                const StoreT<F> &ws = sb.in;
                cp_async_elem(d + 0 * kMaxCells, in.ox + q);
                cp_async_elem(d + 1 * kMaxCells, in.oy + q);
                cp_async_elem(d + 2 * kMaxCells, in.oz + q);
                cp_async_elem(d + 3 * kMaxCells, ws.ox + q);
                cp_async_elem(d + 4 * kMaxCells, ws.oy + q);
                cp_async_elem(d + 5 * kMaxCells, ws.oz + q);
                cp_async_elem(d + 6 * kMaxCells, ws.ux + q);
                cp_async_elem(d + 7 * kMaxCells, ws.uy + q);
                cp_async_elem(d + 8 * kMaxCells, ws.uz + q);
                cp_async_elem(d + 9 * kMaxCells, in.w + q);
                cp_async_elem(d + 10 * kMaxCells, ws.w + q);
            } else if (NS == 2) {
                const SpTab<F> &T = tab[species_of(i)];
#pragma unroll
                for (int a = 0; a < 7; ++a) cp_async_elem(d + a * kMaxCells, T.in[a] + q);
            } else {
                cp_async_elem(d + 0 * kMaxCells, in.ox + q);
                cp_async_elem(d + 1 * kMaxCells, in.oy + q);
                cp_async_elem(d + 2 * kMaxCells, in.oz + q);
                cp_async_elem(d + 3 * kMaxCells, in.ux + q);
                cp_async_elem(d + 4 * kMaxCells, in.uy + q);
                cp_async_elem(d + 5 * kMaxCells, in.uz + q);
                cp_async_elem(d + 6 * kMaxCells, in.w + q);
            }
        }
        cp_async_commit();
    };
    prefetch(0);   // issued before the staging: its latency overlaps it

    // ---- periodic index tables, then stage E/B and clear the J tile -------
    for (int i = t; i < L.tx; i += blockDim.x) wtx[i] = pymod(orgx - 1 + i, g.nx);
    for (int i = t; i < L.ty; i += blockDim.x) wty[i] = pymod(orgy - 1 + i, g.ny);
    for (int i = t; i < L.tz; i += blockDim.x) wtz[i] = pymod(orgz - 1 + i, g.nz);
    for (int i = t; i < L.jx; i += blockDim.x) wjx[i] = pymod(orgx - H + i, g.nx);
    for (int i = t; i < L.jy; i += blockDim.x) wjy[i] = pymod(orgy - H + i, g.ny);
    for (int i = t; i < L.jz; i += blockDim.x) wjz[i] = pymod(orgz - H + i, g.nz);
    if (t < kMaxCells)
#pragma unroll
        for (int s_ = 0; s_ < NS; ++s_) arr[s_ * kMaxCells + t] = 0;
    if (t == 0) { s_maxcol = 0; s_maxcol1 = 0; }
    for (int i = t; i < 3 * L.JV; i += blockDim.x) jt[i] = F(0);
    constexpr bool PCSBOX = ORDER == 3 && !REGACC && sizeof(F) == 4 && SX == 8 && SY == 8 && SZ == 4;
    float *wbox = reinterpret_cast<float *>(smem_raw + L.off_wb) + wid * kBoxFloats;
    if constexpr (PCSBOX)
        for (int i = lane; i < kBoxFloats; i += 32) wbox[i] = 0.0f;
    __syncthreads();
    if (tma_eb) {
        mbar_wait(&s_mbar, 0);
        // widen / copy the box (x from origin - kTmaX0) into the tile (x from origin - 1)
        // element i = row * tx + a of the tile, row = (c * tz + d) * ty + b,
        // is element row * boxx + a + kTmaX0 - 1 of the box
        const F *src = reinterpret_cast<const F *>(eb_dst) + kTmaX0 - 1;
        const int total = 6 * L.TV;
        for (int i = t; i < total; i += blockDim.x) {
            const int row = i / L.tx, a = i - row * L.tx;
            ebd[i] = (EB)src[row * boxx + a];
        }
    } else if (!SPLIT) {
        // flat over (component, z, y, x) so every lane works, and batches of
        // kStageB independent loads in flight per thread (one memory latency
        // per batch instead of one per tile row)
        constexpr int kStageB = 16;   // 6 x 600 values / 256 threads: one batch
        const int total = 6 * L.TV, nth = blockDim.x, txy_ = L.tx * L.ty;
        for (int base = t; base < total; base += kStageB * nth) {
            F v[kStageB];
#pragma unroll
            for (int u = 0; u < kStageB; ++u) {
                const int i = base + u * nth;
                if (i < total) {
                    const int c = i / L.TV, r = i - c * L.TV;
                    const int d = r / txy_, r2 = r - d * txy_;
                    const int b = r2 / L.tx, a = r2 - b * L.tx;
                    // select chain, not fp.E[c]: a runtime index into the
                    // parameter struct would copy it to local memory
                    const void *sv = c == 0 ? fp.E[0] : c == 1 ? fp.E[1] : c == 2 ? fp.E[2]
                                   : c == 3 ? fp.B[0] : c == 4 ? fp.B[1] : fp.B[2];
                    const F *src = (const F *)sv;
                    v[u] = __ldg(src + ((int64_t)wtz[d] * g.ny + wty[b]) * g.nx + wtx[a]);
                }
            }
#pragma unroll
            for (int u = 0; u < kStageB; ++u) {
                const int i = base + u * nth;
                if (i < total) ebd[i] = (EB)v[u];
            }
        }
    }

    int n_w = n_t;  // warp-uniform trip count
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_w = max(n_w, __shfl_xor_sync(0xffffffffu, n_w, o));
    __syncthreads();

    std::conditional_t<sizeof(F) == 4, RegAcc, RegAccD> R;
    if (REGACC) R.zero();
    float4 *wsm = reinterpret_cast<float4 *>(smem_raw + L.off_ws) + t;   // KWB_WIN_SMEM
#ifdef KWB_WIN_SMEM
    if (REGACC && sizeof(F) == 4 && owner)
#pragma unroll
        for (int k = 0; k < 7; ++k) wsm[k * kMaxCells] = make_float4(0.f, 0.f, 0.f, 0.f);
#endif
    const double qm0 = sp.qm_half_dt;
    const int cx = orgx + lx, cy = orgy + ly, cz = orgz + lz;
    const double cxd = (double)cx, cyd = (double)cy, czd = (double)cz;
    const int txy = L.tx * L.ty;
    const int tbase = (lz * L.ty + ly) * L.tx + lx;   // tile index of (cell - 1) on each axis
    const EB *EBx = ebd, *EBy = ebd + L.TV, *EBz = ebd + 2 * L.TV, *BBx = ebd + 3 * L.TV,
                 *BBy = ebd + 4 * L.TV, *BBz = ebd + 5 * L.TV;
    int fo = 0;      // stayers written to the front of this column (species 0)
    int fo1 = 0;     // ... species 1 (NS = 2)
    int n_err = 0;
    int wq = 0;      // this warp's queue fill (warp-uniform)
    // PCS: the queue is a ring of kQ (a power of two) records from qh, and
    // every full 32 are drained at once, so the drain's lanes are all busy
    int qh = 0;
    static_assert(REGACC || (kQ & (kQ - 1)) == 0, "PCS queue must be a power of two");
    auto qidx = [&](int k) -> int { return REGACC ? k : (qh + k) & (kQ - 1); };


    // Deposit the queued crossing particles of this warp (lanes take one
    // record each; CAS into the J tile).
    // the record's species (bit 30 of its info word) selects the deposit factors
    auto fac_of = [&](int info, int k) -> double {
        return NS == 2 ? tab[(info >> 30) & 1].fac[k] : sp.fac[k];
    };
    auto drain_queue = [&]() {
        __syncwarp();
        auto warp_record = [&](int j) {   // warp-uniform j
            const int info = q_info[j];
            deposit_warp<F, ORDER>(jt, L.jx, L.jy, L.JV, lane, info & 255, (info >> 8) & 255,
                                   (info >> 16) & 255, ((info >> 24) & 3) - 1,
                                   ((info >> 26) & 3) - 1, ((info >> 28) & 3) - 1,
                                   q_f[0 * QS + j], q_f[1 * QS + j], q_f[2 * QS + j],
                                   q_f[3 * QS + j], q_f[4 * QS + j], q_f[5 * QS + j],
                                   q_f[6 * QS + j], fac_of(info, 0), fac_of(info, 1),
                                   fac_of(info, 2), true);
        };
        if (!REGACC) {
            // PCS: every particle is queued; one record per lane, loop-rolled
            // routine (its unrolled form does not fit the instruction cache)
            for (int k = lane; k < wq; k += 32) {
                const int j = qidx(k);
                const int info = q_info[j];
                deposit_cross_compact<F, ORDER>(
                    jt, L.jx, L.jy, L.JV, info & 255, (info >> 8) & 255, (info >> 16) & 255,
                    ((info >> 24) & 3) - 1, ((info >> 26) & 3) - 1, ((info >> 28) & 3) - 1,
                    q_f[0 * QS + j], q_f[1 * QS + j], q_f[2 * QS + j], q_f[3 * QS + j],
                    q_f[4 * QS + j], q_f[5 * QS + j], q_f[6 * QS + j], fac_of(info, 0),
                    fac_of(info, 1), fac_of(info, 2));
            }
        } else {
            // single-axis crossers (the common case): one record per lane,
            // anchor-shifted fp32 routine; the rare multi-axis ones: one warp
            // per record
            for (int j0 = 0; j0 < wq; j0 += 32) {
                const int j = j0 + lane;
                bool multi = false;
                if (j < wq) {
                    const int info = q_info[j];
                    const int ddx = ((info >> 24) & 3) - 1, ddy = ((info >> 26) & 3) - 1,
                              ddz = ((info >> 28) & 3) - 1;
                    if ((ddx != 0) + (ddy != 0) + (ddz != 0) == 1) {
                        const int k = ddx ? 0 : (ddy ? 1 : 2);
                        deposit_cross1<F, ORDER>(jt, L.jx, L.jy, L.JV, k, info & 255,
                                                 (info >> 8) & 255, (info >> 16) & 255,
                                                 ddx + ddy + ddz, q_f[0 * QS + j],
                                                 q_f[1 * QS + j], q_f[2 * QS + j],
                                                 q_f[3 * QS + j], q_f[4 * QS + j],
                                                 q_f[5 * QS + j], q_f[6 * QS + j],
                                                 fac_of(info, 0), fac_of(info, 1),
                                                 fac_of(info, 2));
                    } else {
                        multi = true;
                    }
                }
                unsigned mm = __ballot_sync(0xffffffffu, multi);
                while (mm) {
                    const int b = __ffs(mm) - 1;
                    mm &= mm - 1u;
                    warp_record(j0 + b);
                }
            }
        }
        __syncwarp();
    };

    for (int i = 0; i < n_w; ++i) {
        const bool active = i < n_t;
        const int sp_i = species_of(i);   // this particle's species (0 unless NS = 2)
        cp_async_wait_all();
        const F *cur = pf + (i & 1) * NPF * kMaxCells;
        prefetch(i + 1);
        // read at their uses, not hoisted into registers (measured: hoisting
        // all seven costs 5 %)
        const F &ox = cur[0 * kMaxCells], &oy = cur[1 * kMaxCells], &oz = cur[2 * kMaxCells],
                &ux = cur[3 * kMaxCells], &uy = cur[4 * kMaxCells], &uz = cur[5 * kMaxCells],
                &w = cur[(SPLIT ? 9 : 6) * kMaxCells];
        bool queue = false, leave = false, mover = false, stay = false, pstay = false;
        F nox = 0, noy = 0, noz = 0, nux = 0, nuy = 0, nuz = 0;
        int dcx = 0, dcy = 0, dcz = 0, ncx = 0, ncy = 0, ncz = 0, dest = 0, nlc = 0;
        if (active) {
#ifdef KWB_EARLY_S0
            float s0w[3][3];
            if constexpr (REGACC && sizeof(F) == 4) old_weights<ORDER>((float)ox, (float)oy, (float)oz, s0w);
#endif
            int dxi, dyi, dzi;
            if constexpr (SPLIT) {
                // push_kernel's results (csrc/push.cuh)
                nox = cur[3 * kMaxCells]; noy = cur[4 * kMaxCells]; noz = cur[5 * kMaxCells];
                nux = cur[6 * kMaxCells]; nuy = cur[7 * kMaxCells]; nuz = cur[8 * kMaxCells];
                unpack_carries((int)cur[10 * kMaxCells], dxi, dyi, dzi);
            } else {
            // -- gather (pic/kernels.py:53-77): f64 compute, F store --------
            const double px = cxd + (double)ox, py = cyd + (double)oy, pz = czd + (double)oz;
            const int ox0 = orgx - 1, oy0 = orgy - 1, oz0 = orgz - 1;
#if defined(KWB_GATHER_FLOOR)
            const F e0 = (F)sample_tile<0>(EBx, px, py, pz, ox0, oy0, oz0, L.tx, txy);
            const F e1 = (F)sample_tile<1>(EBy, px, py, pz, ox0, oy0, oz0, L.tx, txy);
            const F e2 = (F)sample_tile<2>(EBz, px, py, pz, ox0, oy0, oz0, L.tx, txy);
            const F b0 = (F)sample_tile<3>(BBx, px, py, pz, ox0, oy0, oz0, L.tx, txy);
            const F b1 = (F)sample_tile<4>(BBy, px, py, pz, ox0, oy0, oz0, L.tx, txy);
            const F b2 = (F)sample_tile<5>(BBz, px, py, pz, ox0, oy0, oz0, L.tx, txy);
#elif !defined(KWB_EXP_NOGATHER)
            (void)ox0; (void)oy0; (void)oz0;
            const AxFrac ax[3][2] = {{ax_frac(px, 0.5, cxd, cxd - 1.0), ax_frac(px, 1.0, cxd, cxd - 1.0)},
                                     {ax_frac(py, 0.5, cyd, cyd - 1.0), ax_frac(py, 1.0, cyd, cyd - 1.0)},
                                     {ax_frac(pz, 0.5, czd, czd - 1.0), ax_frac(pz, 1.0, czd, czd - 1.0)}};
            const F e0 = (F)sample_sel<0>(EBx, ax, tbase, L.tx, txy, L.TV);
            const F e1 = (F)sample_sel<1>(EBy, ax, tbase, L.tx, txy, L.TV);
            const F e2 = (F)sample_sel<2>(EBz, ax, tbase, L.tx, txy, L.TV);
            const F b0 = (F)sample_sel<3>(BBx, ax, tbase, L.tx, txy, L.TV);
            const F b1 = (F)sample_sel<4>(BBy, ax, tbase, L.tx, txy, L.TV);
            const F b2 = (F)sample_sel<5>(BBz, ax, tbase, L.tx, txy, L.TV);
#else   // timing experiment only: no field gather
            const F e0 = (F)(px * 1e-30), e1 = (F)(py * 1e-30), e2 = (F)(pz * 1e-30);
            const F b0 = e0, b1 = e1, b2 = e2;
#endif

            // -- Boris push + move (pic/kernels.py:80-135), shared with the
            // split path's push_kernel (csrc/push.cuh)
            const double qm = NS == 2 ? tab[sp_i].qm : qm0;
            push_move<F>(qm, sp.dt_d, e0, e1, e2, b0, b1, b2, ox, oy, oz, ux, uy, uz, nux, nuy, nuz,
                         nox, noy, noz, dxi, dyi, dzi);
            }

            // -- cell, membership (pic/particles.py:226-228), deposit route
            const int nlx = lx + dxi, nly = ly + dyi, nlz = lz + dzi;
            const bool small = (unsigned)(dxi + 1) <= 2u && (unsigned)(dyi + 1) <= 2u &&
                               (unsigned)(dzi + 1) <= 2u;
            if (small && (unsigned)nlx < (unsigned)scx && (unsigned)nly < (unsigned)scy &&
                (unsigned)nlz < (unsigned)scz) {
                // still inside this super cell: no periodic wrap involved
                dcx = dxi; dcy = dyi; dcz = dzi;
                nlc = nlx + scx * (nly + scy * nlz);
                if (nlc == t) stay = true; else mover = true;
            } else {
                ncx = pymod(cx + dxi, g.nx);
                ncy = pymod(cy + dyi, g.ny);
                ncz = pymod(cz + dzi, g.nz);
                dcx = ncx - cx; dcy = ncy - cy; dcz = ncz - cz;
                if (dcx > 1) dcx -= g.nx; else if (dcx < -1) dcx += g.nx;
                if (dcy > 1) dcy -= g.ny; else if (dcy < -1) dcy += g.ny;
                if (dcz > 1) dcz -= g.nz; else if (dcz < -1) dcz += g.nz;
                dest = (ncx / scx) + g.gx * ((ncy / scy) + g.gy * (ncz / scz));
                if (dest == sc) {
                    nlc = (ncx - orgx) + scx * ((ncy - orgy) + scy * (ncz - orgz));
                    if (nlc == t) stay = true; else mover = true;
                } else {
                    leave = true;
                }
            }
            if (dcx > 1 || dcx < -1 || dcy > 1 || dcy < -1 || dcz > 1 || dcz < -1) {
                ++n_err;  // pic/kernels.py:188-191: counted, not deposited
            }
#ifdef KWB_EXP_NODEPOSIT   // timing experiment only: no current deposit
            else if (true) { }
#endif
            else if (REGACC) {
                // the owner's register window, for crossers too; what a
                // crosser deposits outside it goes through the queue
                const double ww = (double)w;
                const double f0 = NS == 2 ? tab[sp_i].fac[0] : sp.fac[0];
                const double f1 = NS == 2 ? tab[sp_i].fac[1] : sp.fac[1];
                const double f2 = NS == 2 ? tab[sp_i].fac[2] : sp.fac[2];
                if constexpr (sizeof(F) == 4) {
#ifndef KWB_EARLY_S0
                    float s0w[3][3];
                    old_weights<ORDER>((float)ox, (float)oy, (float)oz, s0w);
#endif
                    deposit_window<ORDER>(R, wsm, s0w, (float)nox,
                                        (float)noy, (float)noz, (float)(f0 * ww),
                                        (float)(f1 * ww), (float)(f2 * ww),
                                        dcx, dcy, dcz);
                }
                else
                    deposit_window_d<ORDER>(R, (double)ox, (double)oy, (double)oz, (double)nox,
                                          (double)noy, (double)noz, f0 * ww,
                                          f1 * ww, f2 * ww, dcx, dcy, dcz);
#ifndef KWB_EXP_NOCROSS   // timing experiment only: skip crossing deposits
                queue = (dcx | dcy | dcz) != 0;
#endif
            } else {
#ifndef KWB_EXP_NOCROSS   // timing experiment only: skip crossing deposits
                if (PCSBOX && stay && (dcx | dcy | dcz) == 0) pstay = true;
                else queue = true;
#endif
            }
        }

        // ---- crossing particles -> this warp's queue (no atomics) ---------
        const unsigned qmask = __ballot_sync(0xffffffffu, queue);
        if (!REGACC && wq + __popc(qmask) > kQ) {   // PCS ring full: drain what it holds
            drain_queue();
            qh = (qh + wq) & (kQ - 1);
            wq = 0;
        }
        if (queue && KWB_IN(qidx(wq + __popc(qmask & ((1u << lane) - 1u))) < kQ)) {
            const int j = qidx(wq + __popc(qmask & ((1u << lane) - 1u)));
            q_f[0 * QS + j] = ox; q_f[1 * QS + j] = oy; q_f[2 * QS + j] = oz;
            q_f[3 * QS + j] = nox; q_f[4 * QS + j] = noy; q_f[5 * QS + j] = noz;
            q_f[6 * QS + j] = w;
            q_info[j] = lx | (ly << 8) | (lz << 16) | ((dcx + 1) << 24) | ((dcy + 1) << 26) |
                        ((dcz + 1) << 28) | (sp_i << 30);
        }
        wq += __popc(qmask);
        if (!REGACC) {
            if (wq >= 32) {   // PCS: one full record per lane
                const int left = wq - 32;
                wq = 32;
                drain_queue();
                qh = (qh + 32) & (kQ - 1);
                wq = left;
            }
        } else if (wq > kQ - 32) {   // rare: the queue is normally drained after the loop
            drain_queue();
            wq = 0;
        }
        if constexpr (PCSBOX) {   // PCS stayers: the warp's boxes, no atomics
            if (__any_sync(0xffffffffu, pstay))
                deposit_pcs_box(wbox, lx, ly - 4 * (wid & 1), pstay, ox, oy, oz, nox, noy, noz, w,
                                NS == 2 ? tab[sp_i].fac[0] : sp.fac[0],
                                NS == 2 ? tab[sp_i].fac[1] : sp.fac[1],
                                NS == 2 ? tab[sp_i].fac[2] : sp.fac[2]);
        }

        // ---- write the particle to its column / the exchange --------------
        {   // one store block for stayers (own column front) and in-super-cell
            // movers (destination column back): less code, fewer reconvergence points
            int frame = -1, cell = t;
            const int Ks = sp_i ? K1 : K;
            if (stay) {
                frame = sp_i ? fo1 : fo;
                fo += sp_i ? 0 : 1;
                fo1 += sp_i;
            } else if (mover) {
                const int slot = atomicAdd(&arr[sp_i * kMaxCells + nlc], 1);
                if (slot < Ks) { frame = Ks - 1 - slot; cell = nlc; }
            }
            if (frame >= 0 && KWB_IN(frame < Ks && cell < V)) {
                const int64_t o = ((int64_t)sc * Ks + frame) * V + cell;
                if (NS == 2) {
                    F *const *op = tab[sp_i].out;
                    op[0][o] = nox; op[1][o] = noy; op[2][o] = noz;
                    op[3][o] = nux; op[4][o] = nuy; op[5][o] = nuz;
                    op[6][o] = w;
                } else {
                    out.ox[o] = nox; out.oy[o] = noy; out.oz[o] = noz;
                    out.ux[o] = nux; out.uy[o] = nuy; out.uz[o] = nuz;
                    out.w[o] = w;
                }
            }
        }
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
                    // fused species: the destination carries the species
                    // (shift_kernel: s = dest / n_sc)
                    ex.dest[k] = dest + (sp0 + sp_i) * (g.gx * g.gy * g.gz);
                } else {
                    atomicAdd(&status[KWB_ST_EXCH_OVERFLOW], 1);
                }
            }
        }
    }
    if (n_err) atomicAdd(&status[KWB_ST_MOVE_ERRORS], n_err);
    __syncthreads();

    // ---- reduce the register accumulators into the J tile ----------------
    // Sweep s adds accumulator s of every cell: the targets cell + offset(s)
    // are distinct across threads, so plain read-modify-writes are race free;
    // the three components go to different arrays and share a sweep (27
    // sweeps: edges -1, 0, +1 x 3 x 3); the barrier orders consecutive sweeps.
    if (REGACC) {
        F *Jb = jt + ((lz * L.jy) + ly) * L.jx + lx;
#ifdef KWB_WIN_SMEM
        if constexpr (sizeof(F) == 4) win_load(wsm, R.q, R.r);
#endif
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    if (owner) {
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            F *p = Jb + c * L.JV + regacc_offset(c, a + 1, b + 1, d + 1, L.jx, L.jy);
                            if (KWB_IN(p >= jt && p < jt + 3 * L.JV)) *p = *p + (F)R.get(c, a, b, d);
                        }
                    }
                    __syncthreads();
                }
    }

    // ---- deposit the crossing particles queued during the loop -----------
    // (after the accumulator sweeps, when nothing else is live, so the
    // out-of-line deposit routines run without spilling the accumulators)
    if (wq > 0) drain_queue();
    if constexpr (PCSBOX) {   // the warp's boxes into the J tile
        __syncwarp();
        const int y0 = 4 * (wid & 1), z0 = wid >> 1;
        for (int e = lane; e < kBoxFloats; e += 32) {
            const float v = wbox[e];
            if (v != 0.0f) {
                const int c = e / 480, r = e - c * 480;
                const int X = r % 12, Y = (r / 12) % 8, Z = r / 96;
                const int o = c * L.JV + ((Z + z0 + 1) * L.jy + (Y + y0 + 1)) * L.jx + (X + 1);
                if (KWB_IN(o >= 0 && o < 3 * L.JV)) atomicAdd(jt + o, v);
            }
        }
    }
    __syncthreads();

    // ---- flush the J tile: coalesced red.global.add of non-zero entries ---
    // (a TMA reduce-add of the tile needs a 16-byte aligned box start, i.e. a
    // halo of 4 in x instead of the shape's 2: the wider tile does not fit
    // the shared-memory budget of 2 CTAs per SM)
    auto jrow = [&](int c, int d, int b) -> F * {   // row (tile z d, tile y b) of J[c]
        if (fp.jpl)
            return (F *)fp.jpl[c * g.nz + wjz[d]] + (int64_t)wjy[b] * g.nx;
        F *dst = (F *)(c == 0 ? fp.J[0] : c == 1 ? fp.J[1] : fp.J[2]);
        return dst + ((int64_t)wjz[d] * g.ny + wjy[b]) * g.nx;
    };
    if (sizeof(F) == 4 && (L.jx & 1) == 0) {
        // x-adjacent pairs with one red.global.add.v2.f32 where the pair is
        // contiguous and 8-byte aligned in J (not across the periodic seam)
        const int total = 3 * L.JV / 2, nth = blockDim.x, jxy = L.jx * L.jy;
        for (int i2 = t; i2 < total; i2 += nth) {
            const int i = 2 * i2;
            const F v0 = jt[i], v1 = jt[i + 1];
            if (v0 != F(0) || v1 != F(0)) {
                const int c = i / L.JV, r = i - c * L.JV;
                const int d = r / jxy, r2 = r - d * jxy;
                const int b = r2 / L.jx, a = r2 - b * L.jx;
                F *row = jrow(c, d, b);
                const int x0 = wjx[a], x1 = wjx[a + 1];
                F *p0 = row + x0;
                if (x1 == x0 + 1 && ((reinterpret_cast<uintptr_t>(p0) & 7) == 0)) {
                    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p0), "f"((float)v0),
                                 "f"((float)v1) : "memory");
                } else {
                    if (v0 != F(0)) atomicAdd(p0, v0);
                    if (v1 != F(0)) atomicAdd(row + x1, v1);
                }
            }
        }
    } else {
        const int total = 3 * L.JV, nth = blockDim.x, jxy = L.jx * L.jy;
        for (int i = t; i < total; i += nth) {
            const F v = jt[i];
            if (v != F(0)) {
                const int c = i / L.JV, r = i - c * L.JV;
                const int d = r / jxy, r2 = r - d * jxy;
                const int b = r2 / L.jx, a = r2 - b * L.jx;
                atomicAdd(jrow(c, d, b) + wjx[a], v);
            }
        }
    }
    if (owner) {
        const int nb = arr[t];
        out.front[col] = fo;
        out.back[col] = nb < K ? nb : K;
        if (fo + nb > K) atomicAdd(&status[KWB_ST_STORE_OVERFLOW], fo + nb - K);
        atomicMax(&s_maxcol, fo + nb);
        if (NS == 2) {
            const int nb1 = arr[kMaxCells + t];
            sb.out.front[col] = fo1;
            sb.out.back[col] = nb1 < K1 ? nb1 : K1;
            if (fo1 + nb1 > K1) atomicAdd(&sb.status[KWB_ST_STORE_OVERFLOW], fo1 + nb1 - K1);
            atomicMax(&s_maxcol1, fo1 + nb1);
        }
    }
    __syncthreads();
    if (t == 0) atomicMax(&status[KWB_ST_MAX_COUNT], s_maxcol);
    if (NS == 2 && t == 32) atomicMax(&sb.status[KWB_ST_MAX_COUNT], s_maxcol1);
}
